#!/bin/bash
cd "$(dirname "$0")/.."
timeout -s KILL 300 python -m pytest tests/test_gpu_gemm.py -q -p no:cacheprovider --timeout=120 -k "mn_major" 2>&1 | tail -3
timeout -s KILL 600 python -m pytest tests/test_gpu_decode.py -q -x -s -p no:cacheprovider --timeout=120 2>&1 | grep -E "^\[|passed|failed"
timeout -s KILL 600 python scripts/ab_decode.py --bits 513 1 --batch 32 --rounds 3 --steps 2 --profile --grep attn
