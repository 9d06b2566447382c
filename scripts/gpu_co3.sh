#!/bin/bash
cd "$(dirname "$0")/.."
timeout -s KILL 300 python -m pytest tests/test_gpu_gemm.py -q -x -s -p no:cacheprovider --timeout=120 -k "conv_out" 2>&1 | grep -E "^\[|passed|failed|Error"
timeout -s KILL 300 python -m pytest tests/test_gpu_decode.py -q -x -s -p no:cacheprovider --timeout=120 2>&1 | grep -E "^\[|passed|failed|Error"
bash scripts/gpu_ncu_co.sh 2>&1 | grep conv_out
timeout -s KILL 600 python scripts/ab_decode.py --bits 1 17 --batch 32 --rounds 3 --steps 2 --profile --grep conv_out
