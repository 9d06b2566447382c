#!/bin/bash
cd "$(dirname "$0")/.."
timeout -s KILL 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_decode.py -q -x -p no:cacheprovider --timeout=400 2>&1 | tail -2
timeout -s KILL 900 python scripts/ab_decode.py --bits 1 268435457 134217729 --batch 32 --rounds 3 --steps 2 --profile --grep c128
for r in 1 2; do
  LBX_LIB=ab/liblbx_a.so timeout -s KILL 300 python scripts/ab_lib.py --steps 6
  timeout -s KILL 300 python scripts/ab_lib.py --steps 6
done
