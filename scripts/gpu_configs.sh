#!/bin/bash
# Config 4 bench line, reference arm, config-5 live replays (measured batch service curve).
cd "$(dirname "$0")/.."
TAG=${1:-cfg}
mkdir -p gpurun_out
timeout -s KILL 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_$TAG.json 2> gpurun_out/bench_c4_$TAG.err
python -c "import json; d=json.load(open('gpurun_out/bench_c4_$TAG.json')); print('c4', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), d['clocks'])"
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>&1; tail -c 300 gpurun_out/bench_ref_$TAG.json
for sc in 10 25 35; do
  timeout -s KILL 600 ./tools/c5_replay live --scale $sc --devices 1 --gpus 1 --json gpurun_out/c5_live_1gpu_${sc}x_$TAG.json > gpurun_out/c5_live_${sc}x_$TAG.log 2>&1
  tail -n 3 gpurun_out/c5_live_${sc}x_$TAG.log
done
