#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_decode.py tests/test_gpu_unpack.py -q -s -p no:cacheprovider 2>&1 | grep -E "passed|failed|Error|\[|FAIL" | tail -12
python scripts/op_bench.py gn --b 4 --hw 1024 --c 128 --iters 5
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/profile_r1c.json 2>&1 | tail -1 | cut -c1-700
