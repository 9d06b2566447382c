#!/bin/bash
cd "$(dirname "$0")/.."
for cfg in "1,0" "1,1" "0,0"; do
  echo "== LBX_GEMM_DEBUG=$cfg"
  LBX_GEMM_DEBUG=$cfg timeout -s KILL 300 python -m pytest tests/test_gpu_gemm.py -q -p no:cacheprovider -k "conv3x3 or subpixel" 2>&1 | tail -2
done
