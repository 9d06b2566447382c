"""SASS instruction census of the product library (cuobjdump -sass): per kernel, the mnemonics that
prove where the work runs -- UTCHMMA (tcgen05.mma), UTMALDG / UTMASTG (TMA tensor load / store),
UBLKCP (1-D bulk copy), LDTM / STTM (tcgen05.ld / st), legacy HMMA (must be 0), MUFU, and the
memory/atomic instructions.  Usage: python tools/sass_census.py [liblbx.so] > profiles/r2_sass_census.txt"""
import collections
import os
import re
import subprocess
import sys

KEYS = ["UTCHMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM", "HMMA", "MUFU.TANH", "MUFU.EX2",
        "LDG", "STG", "LDS", "STS", "SHFL", "ATOMG", "REDG", "DFMA", "DADD"]


def main():
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    so = sys.argv[1] if len(sys.argv) > 1 else os.path.join(here, "paper_2605_19385_b200", "liblbx.so")
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True, check=True).stdout
    counts = collections.OrderedDict()
    cur = None
    for ln in sass.splitlines():
        m = re.search(r"Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P[T0-9]+\s+)?([A-Z][A-Z0-9_.]+)", ln)
        if not m:
            continue
        op = m.group(1)
        for k in KEYS:
            if op == k or op.startswith(k + "."):
                counts[cur][k] += 1
    names = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
    print("kernel\t" + "\t".join(KEYS))
    for (raw, c), nm in zip(counts.items(), names):
        nm = re.sub(r"\(.*", "", nm.replace("(anonymous namespace)::", ""))
        print(nm + "\t" + "\t".join(str(c.get(k, 0)) for k in KEYS))
    tot = collections.Counter()
    for c in counts.values():
        tot.update(c)
    print("TOTAL\t" + "\t".join(str(tot.get(k, 0)) for k in KEYS))


if __name__ == "__main__":
    main()
