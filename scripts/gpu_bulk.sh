#!/bin/bash
cd "$(dirname "$0")/.."
timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_decode.py -q -x -p no:cacheprovider --timeout=120 2>&1 | tail -2
timeout -s KILL 600 python scripts/ab_decode.py --bits 257 1 --batch 32 --rounds 4 --steps 2 --profile --grep gn_apply
