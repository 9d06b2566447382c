#!/bin/bash
# Round evidence: GPU tests, smoke, bench line (with CPU baseline + per-launch profile), ncu launch
# list of a short bench, full ncu capture of the dominant kernel at the bench's launch config.
cd "$(dirname "$0")/.."
TAG=${1:-ev}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv,noheader
lscpu | grep -E "Model name|^CPU\(s\)" | tr -s ' '
timeout -s KILL 900 python -m pytest tests -m gpu -q -s -p no:cacheprovider --timeout=300 2>&1 | grep -E "^\[|passed|failed" > gpurun_out/tests_$TAG.txt; tail -3 gpurun_out/tests_$TAG.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 1200 python bench.py --steps 10 --warmup 3 --profile-json gpurun_out/profile_$TAG.json > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python -c "import json; d=json.load(open('gpurun_out/bench_$TAG.json')); print('bench', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), d['clocks'], d['roofline']['kernel'], round(d['roofline']['frac'],3), 'cpu', d['cpu_baseline'])"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --batch 4 > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/dom_$TAG python scripts/op_bench.py conv --b 32 --hw 1024 --c 128 --resid --stats --iters 1 > gpurun_out/ncu_dom_$TAG.log 2>&1
tail -n 1 gpurun_out/ncu_dom_$TAG.log
