#!/bin/bash
# Quick regression: GEMM + decode parity tests, one A/B decode timing with per-kernel profile.
cd "$(dirname "$0")/.."
timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_decode.py -q -x -p no:cacheprovider --timeout=120 2>&1 | tail -1
timeout -s KILL 600 python scripts/ab_decode.py --bits ${BITS:-1} --batch 32 --rounds 3 --steps 2 --profile --grep "${GREP:-attn}"
