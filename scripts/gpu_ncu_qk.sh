#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/op_bench.py gemm --b 1 --hw 128 --n 16384 --k 512 --iters 5 --nobias
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/qk python scripts/op_bench.py gemm --b 1 --hw 128 --n 16384 --k 512 --iters 1 --nobias > gpurun_out/ncu_qk.log 2>&1
tail -1 gpurun_out/ncu_qk.log
