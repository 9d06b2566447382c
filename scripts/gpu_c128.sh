#!/bin/bash
# c128@1024^2 conv at op level (batch 8): plain, residual preload, folded identity (A ring), folded
# identity through rbuf (bit 24); burst and sustained (power-capped) rates.
cd "$(dirname "$0")/.."
S="--b 8 --hw 1024 --c 128 --stats"
for r in 1 2; do
  python scripts/op_bench.py conv $S --iters 10
  python scripts/op_bench.py conv $S --resid --iters 10
  python scripts/op_bench.py conv $S --fold --iters 10
  python scripts/op_bench.py conv $S --fold --bits 16777217 --iters 10
done
python scripts/op_bench.py conv $S --sustain 3
python scripts/op_bench.py conv $S --resid --sustain 3
python scripts/op_bench.py conv $S --fold --sustain 3
python scripts/op_bench.py conv $S --fold --bits 16777217 --sustain 3
