#!/bin/bash
# ncu of the three PNG kernels (one launch each) on the png_bench workload (batch 32 at 1024^2).
set -x
TAG=${1:-png}
mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:png_ --launch-skip 3 --launch-count 3 \
  -o gpurun_out/ncu_$TAG -f python scripts/png_bench.py --reps 1 --cpu 1 > gpurun_out/ncu_$TAG.log 2>&1
tail -5 gpurun_out/ncu_$TAG.log
