#!/bin/bash
cd "$(dirname "$0")/.."
for bits in 1 65537 131073 16385; do
  echo "bits $bits"
  python scripts/op_bench.py conv --b 32 --hw 1024 --c 128 --stats --iters 4 --bits $bits
  python scripts/op_bench.py conv --b 32 --hw 256 --c 512 --stats --iters 4 --bits $bits
  python scripts/op_bench.py gemm --b 1 --hw 128 --n 16384 --k 512 --iters 5 --nobias --bits $bits
done
