#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_gemm.py -q -p no:cacheprovider -k gn_stats 2>&1 | tail -1
python scripts/op_bench.py gn --b 4 --hw 1024 --c 128 --iters 5
python scripts/op_bench.py gn --b 4 --hw 512 --c 256 --iters 5
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/conv128_halo python scripts/op_bench.py conv --b 4 --hw 1024 --c 128 --resid --stats --iters 1 > gpurun_out/ncu3.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:gn_apply -s 1 -c 1 -o gpurun_out/gnapply2 python scripts/op_bench.py gn --b 4 --hw 1024 --c 128 --iters 1 > gpurun_out/ncu4.log 2>&1
tail -n 2 gpurun_out/ncu3.log; tail -n 2 gpurun_out/ncu4.log
