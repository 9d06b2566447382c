#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/op_bench.py conv --b 4 --hw 1024 --c 128 --resid --stats --iters 5
python scripts/op_bench.py conv --b 4 --hw 1024 --c 128 --iters 5
python scripts/op_bench.py conv --b 4 --hw 256 --c 512 --resid --stats --iters 5
python scripts/op_bench.py conv --b 4 --hw 1024 --c 128 --resid --stats --iters 5 --cg 1
python scripts/op_bench.py gn --b 4 --hw 1024 --c 128 --iters 5
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/conv128 python scripts/op_bench.py conv --b 2 --hw 1024 --c 128 --resid --stats --iters 1 > gpurun_out/ncu1.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:gn_apply -s 1 -c 1 -o gpurun_out/gnapply python scripts/op_bench.py gn --b 2 --hw 1024 --c 128 --iters 1 > gpurun_out/ncu2.log 2>&1
tail -2 gpurun_out/ncu1.log gpurun_out/ncu2.log
