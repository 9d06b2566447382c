#!/bin/bash
# Round check on one B200: GPU tests (decode stats printed), smoke, then the driver's default bench
# command (all legs) with its wall time.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-full}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv,noheader
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider --timeout=400 2>&1 | grep -E "^\[|passed|failed|Error|error" | tail -40
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
T0=$(date +%s)
timeout -s KILL 1200 python bench.py --gpus 1 --steps 20 --warmup 5 --profile-json gpurun_out/profile_$TAG.json > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$? wall=$(( $(date +%s) - T0 ))s"
tail -3 gpurun_out/bench_$TAG.err
python - <<PY
import json
d=json.load(open('gpurun_out/bench_$TAG.json'))
print('bench', round(d['value'],2), round(d['ms_per_step'],1), 'e2e', round(d['e2e']['value'],2), d['clocks'])
print('roof', d['roofline']['kernel'], round(d['roofline']['frac'],3), 'step', {k: round(v,3) for k,v in d['step_roofline'].items() if isinstance(v,float)})
for k,v in (d.get('configs') or {}).items(): print(k, {a:b for a,b in v.items() if a!='clocks'}, v.get('clocks',{}).get('sm_mhz'))
print('batcher', d.get('batcher_service'))
print('latency', d.get('latency'))
print('cpu', d.get('cpu_baseline'))
PY
