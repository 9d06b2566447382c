#!/bin/bash
cd "$(dirname "$0")/.."
timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider -k "resid or fold" 2>&1 | tail -1
LBX_GEMM_DEBUG=268435457,0 timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider -k "resid" 2>&1 | tail -1
timeout -s KILL 900 python scripts/ab_decode.py --bits 1 268435457 --batch 32 --rounds 4 --steps 2 --profile --grep "c128->128"
for r in 1 2; do
  LBX_LIB=ab/liblbx_a.so timeout -s KILL 300 python scripts/ab_lib.py --steps 6
  timeout -s KILL 300 python scripts/ab_lib.py --steps 6
done
