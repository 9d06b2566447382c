#!/bin/bash
# K1 unpack at scale: bench line + ncu DRAM bytes of one unpack launch (4096 latents, mode 1 noise)
cd "$(dirname "$0")/.."
TAG=${1:-unpack}
mkdir -p gpurun_out
timeout -s KILL 300 python scripts/unpack_bench.py --n 4096 > gpurun_out/unpack_bench_$TAG.json 2> gpurun_out/unpack_bench_$TAG.err
cat gpurun_out/unpack_bench_$TAG.json
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:lblp_unpack --launch-skip 2 --launch-count 1 python scripts/unpack_bench.py --n 4096 --reps 1 > gpurun_out/ncu_unpack_$TAG.txt 2>&1
grep -E "lblp|dram__|duration|warps_active" gpurun_out/ncu_unpack_$TAG.txt
