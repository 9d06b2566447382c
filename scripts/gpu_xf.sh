#!/bin/bash
# Fused GroupNorm+SiLU A-operand (XF) experiment: correctness, op-level timing against conv + apply,
# and the full decode A/B (bit 2 = XF in the decoder).
cd "$(dirname "$0")/.."
timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider -k "fused or gn_stats" 2>&1 | tail -2
for shp in "--b 8 --hw 1024 --c 128" "--b 8 --hw 512 --c 256" "--b 8 --hw 256 --c 512"; do
  timeout -s KILL 120 python scripts/op_bench.py conv $shp --stats --iters 5
  timeout -s KILL 120 python scripts/op_bench.py conv $shp --stats --gnfuse --iters 5
  timeout -s KILL 120 python scripts/op_bench.py gn $shp --iters 5
done
timeout -s KILL 900 python scripts/ab_decode.py --bits 1 5 --batch 32 --rounds 3 --steps 2 --profile --grep conv1
