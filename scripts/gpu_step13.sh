#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_gemm.py -q -p no:cacheprovider --timeout=120 -k "fused_groupnorm" 2>&1 | tail -4
timeout -s KILL 600 python -m pytest tests/test_gpu_decode.py -q -s -p no:cacheprovider --timeout=300 2>&1 | grep -E "passed|failed|\[" | tail -6
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/profile_r1g.json 2>&1 | tail -1 > gpurun_out/bench_r1g.json
python -c "import json;d=json.load(open('gpurun_out/bench_r1g.json'));print(d['value'],d['e2e']['value'],d['clocks'],d['step_roofline'])"
