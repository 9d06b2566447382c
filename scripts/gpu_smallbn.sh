#!/bin/bash
# 128-wide tiles for small grids (default) vs always 256-wide (LBX_SMALL_BN=0): batch-1 profiles,
# config-1 / batch-1 graph latency, and the parity / batch-invariance tests.
cd "$(dirname "$0")/.."
timeout -s KILL 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_batcher.py -q -x -s -p no:cacheprovider --timeout=300 2>&1 | grep -E "^\[|passed|failed|Error|assert" | tail -30
for r in 1 2; do
  for v in 1 0; do echo "SMALL_BN=$v"; LBX_SMALL_BN=$v timeout 300 python scripts/prof_b1.py | grep -E "graph|eager|@64x64|attn.pv|attn.out"; done
done
