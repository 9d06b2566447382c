#!/bin/bash
# What the residual preload costs the c128 conv2 at the power cap: normal (0), zeros without loads
# (1), and the same L2-resident rows for every tile (2) -- diagnostics, wrong results for 1 / 2.
cd "$(dirname "$0")/.."
for r in 1 2; do
  for v in 0 1 2; do
    echo -n "RESID_DIAG=$v "; LBX_RESID_DIAG=$v timeout 120 python scripts/op_bench.py conv --b 32 --hw 1024 --c 128 --resid --stats --sustain 4
  done
done
echo -n "no residual "; timeout 120 python scripts/op_bench.py conv --b 32 --hw 1024 --c 128 --stats --sustain 4
