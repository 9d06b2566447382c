#!/bin/bash
# Full ncu capture of the dominant kernel at the bench's launch config (c128 conv2 + residual; the decoder
# launches a c128 @1024^2 conv 2 images at a time: 2^28 output elements per launch).
cd "$(dirname "$0")/.."
TAG=${1:-ev}
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/dom_$TAG python scripts/op_bench.py conv --b 2 --hw 1024 --c 128 --resid --stats --iters 1 > gpurun_out/ncu_dom_$TAG.log 2>&1
tail -n 1 gpurun_out/ncu_dom_$TAG.log
