#!/bin/bash
# Bench with the pipelined e2e leg, then the XF (fused GroupNorm+SiLU A operand) ncu captures.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=r2f
timeout -s KILL 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"; tail -3 gpurun_out/bench_$TAG.err
python - <<PY
import json
d=json.load(open('gpurun_out/bench_$TAG.json'))
print('bench', round(d['value'],2), 'e2e', d['e2e'], d['clocks'])
for k,v in (d.get('configs') or {}).items(): print(k, {a:b for a,b in v.items() if a not in ('clocks','workload')})
PY
bash scripts/gpu_ncu_xf.sh
