#!/usr/bin/env python3
"""Per-launch summary of an ncu --set full report (read here, no GPU needed):

  python tools/ncu_summary.py gpurun_out/ncu_all_r2.ncu-rep > profiles/r2_ncu_kernels.tsv

For every captured launch: device time, SM clock, tensor-pipe utilisation, DRAM bytes read/written and
the achieved DRAM bandwidth (against MEASURED_PEAKS.json's copy rate), L2 hit rate, SM / memory
throughput % of peak, registers and grid.  ncu replays each kernel in isolation with a cold-ish cache
and serialised launches: compare shares and utilisations, not absolute times, with the bench."""
import csv
import io
import json
import os
import re
import subprocess
import sys

WANT = {
    "time_ns": ["gpu__time_duration.sum"],
    "sm_hz": ["sm__cycles_elapsed.avg.per_second"],
    "tensor_pct": ["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                   "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
                   "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active"],
    "dram_rd": ["dram__bytes_read.sum"],
    "dram_wr": ["dram__bytes_write.sum"],
    "l2_hit": ["lts__t_sector_hit_rate.pct"],
    "sm_pct": ["sm__throughput.avg.pct_of_peak_sustained_elapsed"],
    "mem_pct": ["gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"],
    "dram_pct": ["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"],
    "regs": ["launch__registers_per_thread"],
    "grid": ["launch__grid_size"],
    "block": ["launch__block_size"],
    "issue_pct": ["sm__inst_issued.avg.pct_of_peak_sustained_active"],
}
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6,
         "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9, "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/second": 1,
         "cycle/nsecond": 1e9, "cycle/usecond": 1e6}


def main():
    rep = sys.argv[1]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    head, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(head)}
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    hbm = 6547.2
    try:
        hbm = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except (OSError, KeyError, ValueError):
        pass
    print("# ncu --set full per launch (cold cache, serialised; see tools/ncu_summary.py); HBM peak "
          f"{hbm} GB/s (MEASURED_PEAKS.json)")
    print("kernel\tus\tsm_MHz\ttensor%\tdram_rd_MB\tdram_wr_MB\tdram_GBps\tdram_frac\tl2_hit%\tsm%\tmem%\tissue%\tregs\tgrid\tblock")

    def get(r, key):
        for name in WANT[key]:
            if name in col:
                v = r[col[name]].replace(",", "")
                try:
                    return float(v) * UNITS.get(units[col[name]], 1)
                except ValueError:
                    return None
        return None

    for r in data:
        name = r[col["Kernel Name"]]
        name = re.sub(r"\(.*", "", name.replace("(anonymous namespace)::", "")).replace("void ", "")
        t = get(r, "time_ns") or 0
        rd, wr = get(r, "dram_rd") or 0, get(r, "dram_wr") or 0
        gbs = (rd + wr) / t if t else 0  # bytes / ns = GB/s
        f = lambda v, d=1: "" if v is None else f"{v:.{d}f}"
        hz = get(r, "sm_hz")
        print("\t".join([name, f(t / 1e3), f(hz / 1e6 if hz else None, 0), f(get(r, "tensor_pct")), f(rd / 1e6),
                         f(wr / 1e6), f(gbs, 0), f(gbs / hbm, 3), f(get(r, "l2_hit")), f(get(r, "sm_pct")),
                         f(get(r, "mem_pct")), f(get(r, "issue_pct")), f(get(r, "regs"), 0), f(get(r, "grid"), 0),
                         f(get(r, "block"), 0)]))


if __name__ == "__main__":
    main()
