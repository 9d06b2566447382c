#!/bin/bash
# rbuf (debug bit 24): extra K segments through their own buffer between halo taps; c128 identity
# residual folded into K instead of preloaded.  Op tests, decode parity under the bit, A/B timing.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv,noheader
timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider --timeout=120 -k "folded" 2>&1 | tail -3
LBX_GEMM_DEBUG="16777217,0" timeout -s KILL 900 python -m pytest tests/test_gpu_decode.py -q -x -p no:cacheprovider --timeout=300 2>&1 | tail -3
timeout -s KILL 900 python scripts/ab_decode.py --bits 1 16777217 16777345 --batch 32 --rounds 4 --steps 2 --profile --grep "conv2"
