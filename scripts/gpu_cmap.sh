#!/bin/bash
cd "$(dirname "$0")/.."
timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_decode.py -q -x -p no:cacheprovider --timeout=120 2>&1 | tail -1
for r in 1 2; do for bits in 1 524289; do
  echo "bits $bits"
  python scripts/op_bench.py conv --b 32 --hw 1024 --c 128 --stats --resid --iters 4 --bits $bits
  python scripts/op_bench.py subpix --b 32 --hw 512 --c 256 --stats --iters 4 --bits $bits
  python scripts/op_bench.py gemm --b 1 --hw 128 --n 16384 --k 512 --iters 5 --nobias --bits $bits
done; done
timeout -s KILL 600 python scripts/ab_decode.py --bits 524289 1 --batch 32 --rounds 4 --steps 2
