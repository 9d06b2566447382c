#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/c128_vsub python scripts/op_bench.py conv --b 16 --hw 1024 --c 128 --fold --stats --iters 1 > gpurun_out/ncu_c128.log 2>&1
tail -n 2 gpurun_out/ncu_c128.log
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/c512_256 python scripts/op_bench.py conv --b 16 --hw 256 --c 512 --fold --stats --iters 1 > gpurun_out/ncu_c512.log 2>&1
tail -n 2 gpurun_out/ncu_c512.log
ls -la gpurun_out/*.ncu-rep
