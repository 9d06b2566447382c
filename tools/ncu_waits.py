#!/usr/bin/env python3
"""Summarise an ncu --set full report of gemm_tc_kernel: stall samples at each mbarrier wait, grouped
by barrier (offset from a_full: a_full 0, a_empty 0x80, b_full 0x100, b_empty 0x180, tfull 0x200,
tempty 0x210), plus the sample total per warp role (by SASS address range).  Diagnostic only.

  python tools/ncu_waits.py gpurun_out/prof.ncu-rep
"""
import csv
import io
import re
import subprocess
import sys

NAMES = {0: "a_full", 0x80: "a_empty", 0x100: "b_full", 0x180: "b_empty", 0x200: "tfull", 0x210: "tempty",
         0x220: "a_xform"}


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    data = rows[2:]
    isrc, iall, iex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    tot = sum(float(r[iall] or 0) for r in data)
    print(f"total samples {tot:.0f}")
    agg = {}
    pending = None
    for i, r in enumerate(data):
        s = r[isrc]
        m = re.search(r"SYNCS\.PHASECHK\.TRANS64(?:\.TRYWAIT)? P\d, \[R\d+\+URZ(\+0x([0-9a-f]+))?\]", s)
        samples = float(r[iall] or 0)
        if m:
            off = int(m.group(2), 16) if m.group(2) else 0
            pending = (off, i)
            agg.setdefault(off, [0.0, 0.0])
            agg[off][0] += samples
            agg[off][1] += float(r[iex] or 0)
        elif pending and i - pending[1] <= 3 and ("BRA" in s or "NANOSLEEP" in s):
            agg[pending[0]][0] += samples
    for off, (smp, ex) in sorted(agg.items()):
        print(f"  {NAMES.get(off, hex(off)):>8}: {smp:8.0f} samples ({100 * smp / tot:5.1f}%)  {ex:12.0f} executions")


if __name__ == "__main__":
    main(sys.argv[1])
