#!/bin/bash
cd "$(dirname "$0")/.."
echo "== fp32 SiLU"; timeout -s KILL 600 python -m pytest tests/test_gpu_decode.py -q -s -p no:cacheprovider --timeout=300 2>&1 | grep -E "^\[|passed|failed"
echo "== half2 SiLU"; LBX_GEMM_DEBUG=9,0 timeout -s KILL 600 python -m pytest tests/test_gpu_decode.py -q -s -p no:cacheprovider --timeout=300 2>&1 | grep -E "^\[|passed|failed"
timeout -s KILL 600 python scripts/ab_decode.py --bits 1 9 --batch 32 --rounds 5 --steps 2 --profile
