#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_decode.py -q -s -p no:cacheprovider 2>&1 | grep -E "passed|failed|\[|Error" | tail -12
for a in "conv --hw 1024 --c 128 --stats" "conv --hw 1024 --c 128 --fold --stats" "conv --hw 1024 --c 256 --n 128 --stats" "gn --hw 1024 --c 128"; do
  python scripts/op_bench.py $a --b 4 --iters 5
done
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/profile_r1f.json 2>&1 | tail -1 > gpurun_out/bench_r1f.json
python -c "import json;d=json.load(open('gpurun_out/bench_r1f.json'));print(d['value'],d['e2e']['value'],d['clocks'],d['step_roofline'])"
