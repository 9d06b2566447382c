#!/bin/bash
# Round evidence: bench line (with CPU baseline), launch list, full ncu capture of the dominant kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv,noheader
lscpu | grep -E "Model name|^CPU\(s\)" | tr -s ' '
timeout -s KILL 1200 python bench.py --steps 10 --warmup 3 --profile-json gpurun_out/profile_final.json > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
tail -c 400 gpurun_out/bench_final.json
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --batch 4 > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/dominant_conv128 python scripts/op_bench.py conv --b 32 --hw 1024 --c 128 --fold --stats --iters 1 > gpurun_out/ncu_dom.log 2>&1
tail -n 1 gpurun_out/ncu_dom.log
