#!/bin/bash
cd "$(dirname "$0")/.."
timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider --timeout=120 -k "fused or folded or conv3x3" 2>&1 | tail -2
for hc in "1024 128" "512 256" "256 512"; do
  set -- $hc
  timeout -s KILL 120 python scripts/op_bench.py conv --b 32 --hw $1 --c $2 --fold --stats --iters 4
  timeout -s KILL 120 python scripts/op_bench.py conv --b 32 --hw $1 --c $2 --fold --stats --gnfuse --iters 4
  timeout -s KILL 120 python scripts/op_bench.py conv --b 32 --hw $1 --c $2 --stats --iters 4
  timeout -s KILL 120 python scripts/op_bench.py conv --b 32 --hw $1 --c $2 --stats --gnfuse --iters 4
done
LBX_GEMM_DEBUG=5,0 timeout -s KILL 600 python -m pytest tests/test_gpu_decode.py -q -s -p no:cacheprovider --timeout=300 2>&1 | grep -E "^\[|passed|failed"
timeout -s KILL 600 python scripts/ab_decode.py --bits 1 5 --batch 32 --rounds 4 --steps 2 --profile
