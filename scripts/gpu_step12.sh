#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_batcher.py -q -p no:cacheprovider 2>&1 | tail -1
for s in 10 25 35; do
  timeout -s KILL 400 ./tools/c5_replay live --scale $s --devices 1 --window-s 20 --json gpurun_out/c5_live_${s}x.json 2>gpurun_out/c5_live_${s}x.err >/dev/null
  python -c "import json;d=json.load(open('gpurun_out/c5_live_${s}x.json'));print($s, 'sim', d['sim']['decode_p50_ms'], d['sim']['decode_p99_ms'], 'live', d['live'])"
done
