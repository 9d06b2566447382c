#!/bin/bash
cd "$(dirname "$0")/.."
for hw_c in "1024 128" "512 256" "256 512" "128 512"; do
  set -- $hw_c
  timeout -s KILL 120 python scripts/op_bench.py conv --b 32 --hw $1 --c $2 --fold --stats --iters 4
  timeout -s KILL 120 python scripts/op_bench.py conv --b 32 --hw $1 --c $2 --resid --stats --iters 4
  timeout -s KILL 120 python scripts/op_bench.py conv --b 32 --hw $1 --c $2 --stats --iters 4
done
