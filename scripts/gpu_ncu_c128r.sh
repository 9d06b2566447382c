#!/bin/bash
# ncu --set full with source of the dominant kernel's shape: c128 conv2 + residual (rpf) @1024^2, batch 8
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/c128r python scripts/op_bench.py conv --b 8 --hw 1024 --c 128 --resid --stats --iters 1 > gpurun_out/ncu_c128r.log 2>&1
tail -n 2 gpurun_out/ncu_c128r.log
ls -la gpurun_out/*.ncu-rep
