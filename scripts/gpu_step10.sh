#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests/test_gpu_gemm.py -v -p no:cacheprovider --timeout=120 2>&1 | grep -E "PASS|FAIL|ERROR|Timeout|passed|failed" | tail -45
