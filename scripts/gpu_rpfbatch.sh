#!/bin/bash
# Residual preload with batched loads (LBX_RPF_BATCH 1: per sub-tile, 2: both sub-tiles in flight)
# vs the per-chunk loads (0): c128 conv2 + residual sustained at the cap, then the decode.
cd "$(dirname "$0")/.."
for r in 1 2; do
  for v in 0 1 2; do
    echo "RPF_BATCH=$v"; LBX_RPF_BATCH=$v timeout 120 python scripts/op_bench.py conv --b 32 --hw 1024 --c 128 --resid --stats --sustain 4
  done
done
for r in 1 2 3; do
  for v in 0 1 2; do
    echo -n "RPF_BATCH=$v "; LBX_RPF_BATCH=$v timeout -s KILL 300 python scripts/ab_lib.py --steps 6
  done
done
