#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_decode.py -q -s -p no:cacheprovider 2>&1 | grep -E "passed|failed|\[" | tail -6
for a in "conv --hw 1024 --c 128 --resid --stats" "conv --hw 1024 --c 128" "conv --hw 512 --c 256 --resid --stats" "conv --hw 256 --c 512 --resid --stats" "conv --hw 128 --c 512 --resid --stats" "subpix --hw 512 --c 256 --stats" "subpix --hw 256 --c 512 --stats"; do
  python scripts/op_bench.py $a --b 4 --iters 5
done
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/profile_r1d.json 2>&1 | tail -1 | cut -c1-400
