#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/op_bench.py conv --b 8 --hw 256 --c 512 --stats --iters 5
python scripts/op_bench.py conv --b 8 --hw 256 --c 512 --stats --gnfuse --iters 5
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/conv512_fused python scripts/op_bench.py conv --b 4 --hw 256 --c 512 --stats --gnfuse --iters 1 > gpurun_out/ncu5.log 2>&1
tail -n 1 gpurun_out/ncu5.log
