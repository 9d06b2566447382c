#!/bin/bash
cd "$(dirname "$0")/.."
timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_decode.py -q -x -p no:cacheprovider --timeout=120 2>&1 | tail -2
for bits in 33 65 97; do
  LBX_GEMM_DEBUG=$bits,0 timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider --timeout=120 -k "conv3x3" 2>&1 | tail -1
done
for bits in 1 33 65 97; do
  echo "bits $bits"
  timeout -s KILL 120 python scripts/op_bench.py conv --b 32 --hw 1024 --c 128 --fold --stats --iters 3 --bits $bits
  timeout -s KILL 120 python scripts/op_bench.py conv --b 32 --hw 512 --c 256 --fold --stats --iters 3 --bits $bits
  timeout -s KILL 120 python scripts/op_bench.py conv --b 32 --hw 256 --c 512 --fold --stats --iters 3 --bits $bits
  timeout -s KILL 120 python scripts/op_bench.py subpix --b 32 --hw 512 --c 256 --stats --iters 3 --bits $bits
done
timeout -s KILL 600 python scripts/ab_decode.py --bits 97 1 --batch 32 --rounds 4 --steps 2 --profile
