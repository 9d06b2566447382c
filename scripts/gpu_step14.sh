#!/bin/bash
cd "$(dirname "$0")/.."
timeout -s KILL 300 python -m pytest tests/test_gpu_gemm.py -q -p no:cacheprovider --timeout=120 -k "fused_groupnorm" 2>&1 | tail -2
python scripts/op_bench.py conv --b 8 --hw 256 --c 512 --stats --iters 5
python scripts/op_bench.py conv --b 8 --hw 256 --c 512 --stats --gnfuse --iters 5
python scripts/op_bench.py conv --b 8 --hw 512 --c 256 --stats --iters 5
python scripts/op_bench.py conv --b 8 --hw 512 --c 256 --stats --gnfuse --iters 5
python scripts/op_bench.py gn --b 8 --hw 256 --c 512 --iters 5
