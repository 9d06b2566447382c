#!/bin/bash
cd "$(dirname "$0")/.."
timeout -s KILL 300 python -m pytest tests/test_gpu_gemm.py -q -s -x -p no:cacheprovider --timeout=120 -k "conv_out" 2>&1 | grep -E "^\[|passed|failed|Error|error" | head -20
echo "== decode (TC tail, fp32 SiLU)"; timeout -s KILL 600 python -m pytest tests/test_gpu_decode.py -q -s -p no:cacheprovider --timeout=300 2>&1 | grep -E "^\[|passed|failed"
echo "== decode (TC tail, half2 SiLU)"; LBX_GEMM_DEBUG=9,0 timeout -s KILL 600 python -m pytest tests/test_gpu_decode.py -q -s -p no:cacheprovider --timeout=300 2>&1 | grep -E "^\[|passed|failed"
timeout -s KILL 600 python scripts/ab_decode.py --bits 17 1 9 --batch 32 --rounds 4 --steps 2 --profile
