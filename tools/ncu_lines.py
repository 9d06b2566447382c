#!/usr/bin/env python3
"""Where a kernel's warps stall, by CUDA source line: from an ncu --set full --import-source report
(compiled with -lineinfo), the lines with the most warp-stall samples, each with its top stall
reasons, plus the sample totals of line ranges you name (e.g. a warp role's code region).

  python tools/ncu_lines.py rep.ncu-rep [--file gemm_tc.cu] [--top 25] [--range xf:431-489 --range epi:495-860]
Diagnostic only; runs here (no GPU needed) or on the box."""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--file", default="gemm_tc.cu")
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("--range", action="append", default=[], help="name:first-last (source lines)")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    # per source file: "File Path", "Function Name", a header starting "Line No", then one row per CUDA line
    # (Address "-", metrics aggregated over its SASS) interleaved with that line's SASS rows
    cur_file, head, lines = None, None, []
    for r in rows:
        if r and r[0] == "File Path":
            cur_file = r[1] if len(r) > 1 else ""
            head = None
            continue
        if r and r[0] == "Line No":
            head = r
            continue
        if not head or not cur_file or a.file not in cur_file or len(r) != len(head):
            continue
        if not r[0].isdigit() or r[2] != "-":
            continue
        d = {}
        for i, k in enumerate(head):
            if k not in d:  # "Source" appears twice (CUDA, SASS): keep the first
                d[k] = r[i]
        try:
            tot = float((d.get("Warp Stall Sampling (All Samples)") or "0").replace(",", "") or 0)
        except ValueError:
            continue
        reasons = {}
        for k, v in d.items():
            if k.startswith("stall_") and "Not Issued" not in k:
                try:
                    reasons[k] = float((v or "0").replace(",", ""))
                except ValueError:
                    pass
        lines.append((int(r[0]), tot, reasons, d.get("Source", "").strip()))
    total = sum(t for _, t, _, _ in lines) or 1.0
    print(f"# {a.rep}: {a.file}, {total:.0f} warp-stall samples")
    for name_rng in a.range:
        name, rng = name_rng.split(":")
        lo, hi = (int(x) for x in rng.split("-"))
        s = sum(t for ln, t, _, _ in lines if lo <= ln <= hi)
        agg = {}
        for ln, _, rs, _ in lines:
            if lo <= ln <= hi:
                for k, v in rs.items():
                    agg[k] = agg.get(k, 0.0) + v
        top = ", ".join(f"{k[6:]} {v / max(s, 1):.0%}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:4])
        print(f"range {name} (lines {lo}-{hi}): {s:.0f} samples = {s / total:.1%}; {top}")
    print("line\tsamples\tshare\ttop stall reasons\tsource")
    for ln, t, rs, src in sorted(lines, key=lambda x: -x[1])[:a.top]:
        top = ", ".join(f"{k[6:]} {v / max(t, 1):.0%}" for k, v in sorted(rs.items(), key=lambda kv: -kv[1])[:3])
        print(f"{ln}\t{t:.0f}\t{t / total:.1%}\t{top}\t{src[:90]}")


if __name__ == "__main__":
    main()
