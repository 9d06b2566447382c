#!/bin/bash
cd "$(dirname "$0")/.."
for n in 128 256; do
  timeout -s KILL 120 python scripts/op_bench.py conv --b 16 --hw 1024 --c 128 --n $n --stats --iters 4
  timeout -s KILL 120 python scripts/op_bench.py conv --b 16 --hw 1024 --c 128 --n $n --iters 4
done
timeout -s KILL 120 python scripts/op_bench.py conv --b 16 --hw 1024 --c 128 --n 128 --iters 4 --bits 3
timeout -s KILL 120 python scripts/op_bench.py conv --b 16 --hw 512 --c 256 --n 128 --iters 4
timeout -s KILL 120 python scripts/op_bench.py conv --b 16 --hw 512 --c 256 --n 256 --iters 4
