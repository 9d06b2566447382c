#!/bin/bash
# Re-entry check: GPU tests, smoke, short bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv,noheader
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout=300 2>&1 | tail -5
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/profile_r1b.json > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err
tail -c 600 gpurun_out/bench_r1b.json
