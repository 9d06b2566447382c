#!/usr/bin/env python3
"""Turn one evidence run (scripts/gpu_evidence.sh TAG) into the committed summaries under profiles/:
  profiles/<tag>_bench.json          the bench line
  profiles/<tag>_step_profile.tsv    per-kernel-group device time of one eager decode (lbx_profile)
  profiles/<tag>_launches.tsv        ncu launch list of a short bench, grouped by kernel
  profiles/<tag>_ncu_dominant.txt    key counters + mbarrier wait summary of the dominant conv
  profiles/ncu_traffic.json          DRAM bytes per launch of the dominant kernel (read by bench.py)

  python tools/summarize_evidence.py r1b
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def step_profile(tag):
    d = json.load(open(os.path.join(G, f"profile_{tag}.json")))["groups"]
    tot = sum(v["ms"] for v in d.values())
    lines = [f"# per-launch device time of one eager decode (lbx_profile, CUDA events between launches), config2 batch 32",
             f"# total {tot:.1f} ms per step of 32 images",
             "ms\tshare\tlaunches\tTFLOP/s(algo)\tTFLOP/s(exec)\tGB/s(algo bytes)\tname"]
    for k, v in sorted(d.items(), key=lambda kv: -kv[1]["ms"]):
        s = v["ms"] / 1e3
        lines.append(f"{v['ms']:.2f}\t{100 * v['ms'] / tot:.1f}%\t{v['n']}\t{v['algo'] / s / 1e12:.0f}\t"
                     f"{v['flops'] / s / 1e12:.0f}\t{v['bytes'] / s / 1e9:.0f}\t{k}")
    open(os.path.join(P, f"{tag}_step_profile.tsv"), "w").write("\n".join(lines) + "\n")


def launches(tag):
    txt = open(os.path.join(G, f"launches_{tag}.csv")).read()
    txt = "\n".join(l for l in txt.splitlines() if not l.startswith("=="))
    rows = list(csv.DictReader(io.StringIO(txt)))
    agg = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        name = re.sub(r"^void ", "", name)
        name = re.sub(r"\(.*$", "", name).replace("lbx::", "").replace("(int)", "").replace("(bool)", "")
        val = float(r["Metric Value"].replace(",", ""))
        us = val * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r["Metric Unit"]]
        g = agg.setdefault(name, [0, 0.0])
        g[0] += 1
        g[1] += us
    tot = sum(v[1] for v in agg.values())
    n = sum(v[0] for v in agg.values())
    lines = ["# ncu --metrics gpu__time_duration.sum --clock-control none: every launch of a short bench run "
             "(scripts/gpu_round.sh: config 2, batch 32, --steps 1 --warmup 1: 2 decodes + the eager profile)",
             "# cold-cache, serialised: compare SHARES with the step profile, not absolutes",
             f"# launches {n}, total {tot / 1e3:.1f} ms", "share\tlaunches\ttotal_us\tkernel"]
    for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{100 * us / tot:.1f}%\t{c}\t{us:.0f}\t{k}")
    open(os.path.join(P, f"{tag}_launches.tsv"), "w").write("\n".join(lines) + "\n")


def ncu_dom(tag):
    rep = os.path.join(G, f"dom_{tag}.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    want = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "smsp__issue_active.avg.pct_of_peak_sustained_active"]
    vals = {}
    out = [f"# ncu --set full --clock-control none of the dominant kernel (conv3x3 c128->128 + residual + GN "
           f"statistics, 2 images at 1024^2 = one of the decoder's launches of this conv, 2^28 output elements): scripts/op_bench.py conv --b 2 --hw 1024 --c 128 --resid --stats (residual preloaded into TMEM, as in the decoder)"]
    for i, name in enumerate(h):
        if name in want:
            vals[name] = (v[i], u[i])
            out.append(f"{name} {v[i]} {u[i]}")
    wait = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_waits.py"), rep], capture_output=True,
                          text=True).stdout
    out.append("# stall samples at mbarrier waits (tools/ncu_waits.py): tfull = epilogue waiting for the MMA")
    out += wait.strip().splitlines()
    open(os.path.join(P, f"{tag}_ncu_dominant.txt"), "w").write("\n".join(out) + "\n")

    def gb(name):
        val, unit = vals[name]
        f = float(val.replace(",", ""))
        return f * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}[unit]
    traffic = gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum")
    tj = {"resnet.conv2+residual conv3x3 c128->128 @1024x1024": traffic,
          "_source": f"profiles/{tag}_ncu_dominant.txt: ncu --set full of scripts/op_bench.py conv --b 2 --hw 1024 "
                     "--c 128 --resid --stats (the decoder's dominant launch: this conv runs 2 images per "
                     "launch); dram__bytes_read.sum + dram__bytes_write.sum per launch; algorithmic = "
                     "3 x 0.537 GB (input, residual, output)"}
    json.dump(tj, open(os.path.join(P, "ncu_traffic.json"), "w"), indent=1)


def main(tag):
    b = json.load(open(os.path.join(G, f"bench_{tag}.json")))
    json.dump(b, open(os.path.join(P, f"{tag}_bench.json"), "w"), indent=1)
    step_profile(tag)
    launches(tag)
    if os.path.exists(os.path.join(G, f"dom_{tag}.ncu-rep")):
        ncu_dom(tag)
    print("wrote profiles/ for", tag)


if __name__ == "__main__":
    main(sys.argv[1])
