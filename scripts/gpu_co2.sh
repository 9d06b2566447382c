#!/bin/bash
cd "$(dirname "$0")/.."
timeout -s KILL 300 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider --timeout=120 -k "conv_out" 2>&1 | tail -1
bash scripts/gpu_ncu_co.sh 2>&1 | grep conv_out
