#!/bin/bash
cd "$(dirname "$0")/.."
timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_decode.py -q -x -p no:cacheprovider --timeout=120 2>&1 | tail -1
timeout -s KILL 600 python bench.py --batch 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_b1b.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench_b1b.json')); print('b1', d['ms_per_step'], d['e2e']['value'])"
timeout -s KILL 600 python scripts/ab_decode.py --bits 1 --batch 32 --rounds 3 --steps 2 --profile --grep gn_
