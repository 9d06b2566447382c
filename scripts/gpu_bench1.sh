#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nproc; lscpu | grep "Model name"
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --profile-json gpurun_out/profile_r1.json 2>&1 | tail -5
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --batch 4 > gpurun_out/ncu_bench.log 2>&1
tail -3 gpurun_out/ncu_bench.log
