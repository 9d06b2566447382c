#!/bin/bash
# Full GPU check: tests (decode stats printed), smoke, bench with per-launch profile.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-chk}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv,noheader
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider --timeout=300 2>&1 | grep -E "^\[|passed|failed|Error" | tail -30
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 900 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/profile_$TAG.json > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python -c "import json; d=json.load(open('gpurun_out/bench_$TAG.json')); print('bench', round(d['value'],2), round(d['ms_per_step'],1), 'e2e', round(d['e2e']['value'],2), d['clocks'], d['roofline']['kernel'], round(d['roofline']['frac'],3))"
