#!/bin/bash
# Config-5 live replays (1 GPU): measured batch service curve + 20 s wall-clock windows through lbx_batcher.
cd "$(dirname "$0")/.."
TAG=${1:-c5}
mkdir -p gpurun_out
for sc in ${SCALES:-10 25}; do
  timeout -s KILL 600 ./tools/c5_replay live --scale $sc --devices 1 --gpus 1 --json gpurun_out/c5_live_1gpu_${sc}x_$TAG.json --dump gpurun_out/c5_dump_${sc}x_$TAG.txt > gpurun_out/c5_live_${sc}x_$TAG.log 2>&1
  python -c "import json; d=json.load(open('gpurun_out/c5_live_1gpu_${sc}x_$TAG.json')); print($sc, d['service_ms'], d['live'])"
done
