#!/bin/bash
cd "$(dirname "$0")/.."
timeout -s KILL 600 python -m pytest tests/test_gpu_unpack.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout -s KILL 600 python bench.py --steps 2 --warmup 3 --no-configs --no-latency --no-cpu-baseline --no-e2e > gpurun_out/bench_r2d_codec.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bench_r2d_codec.json')); print(d['kernels']['unpack_entropy'])"
timeout -s KILL 900 python scripts/ab_decode.py --bits 1 536870913 1025 --batch 32 --rounds 3 --steps 2 --profile --grep "c128->128"
