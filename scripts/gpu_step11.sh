#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout=300 2>&1 | tail -3
timeout -s KILL 400 ./tools/c5_replay live --scale 10 --devices 1 --window-s 20 --json gpurun_out/c5_live_10x.json 2>gpurun_out/c5_live_10x.err | cut -c1-2000
timeout -s KILL 400 ./tools/c5_replay live --scale 25 --devices 1 --window-s 20 --json gpurun_out/c5_live_25x.json 2>gpurun_out/c5_live_25x.err | tail -c 600
cat gpurun_out/c5_live_10x.err | head -8
