#!/bin/bash
# DRAM bytes per launch of every GEMM of an eager batch-32 decode (is the c128 conv's halo re-read
# excess present inside the decode, as in the op-level capture?).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:gemm_tc --csv --log-file gpurun_out/dram32.csv python scripts/ncu_kernels.py --batch 32 > gpurun_out/dram32.log 2>&1
tail -n 2 gpurun_out/dram32.log; wc -l gpurun_out/dram32.csv
