#!/bin/bash
# Round evidence on one B200: GPU tests, smoke, the driver's default bench command, the N=2 code
# path on a shared GPU (diagnostics), and the ncu launch list of a short bench.
cd "$(dirname "$0")/.."
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv,noheader
lscpu | grep -E "Model name|^CPU\(s\)" | tr -s ' '
timeout -s KILL 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider --timeout=400 2>&1 | grep -E "^\[|passed|failed|Error" > gpurun_out/tests_$TAG.txt; tail -3 gpurun_out/tests_$TAG.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
T0=$(date +%s)
timeout -s KILL 1200 python bench.py --gpus 1 --steps 20 --warmup 5 --profile-json gpurun_out/profile_$TAG.json > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$? wall=$(( $(date +%s) - T0 ))s"
python - <<PY
import json
d=json.load(open('gpurun_out/bench_$TAG.json'))
print('bench', round(d['value'],2), round(d['ms_per_step'],1), 'e2e', round(d['e2e']['value'],2), d['clocks'])
print('roof', d['roofline']['kernel'], round(d['roofline']['frac'],3))
for k,v in (d.get('configs') or {}).items(): print(k, {a:b for a,b in v.items() if a not in ('clocks','workload')})
print('batcher', d.get('batcher_service'))
print('latency', {k: d['latency'].get(k) for k in ('decode_p50_ms','decode_p99_ms','decodes_per_s')})
PY
LBX_BENCH_SHARE_GPU=1 timeout -s KILL 900 python bench.py --gpus 2 --steps 3 --warmup 3 --batch 8 --no-latency > gpurun_out/bench_${TAG}_n2shared.json 2> gpurun_out/bench_${TAG}_n2shared.err
echo "n2 shared rc=$?"; tail -c 600 gpurun_out/bench_${TAG}_n2shared.json; tail -3 gpurun_out/bench_${TAG}_n2shared.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-configs --no-kernels --no-latency > /dev/null 2>&1
wc -l gpurun_out/launches_$TAG.csv
