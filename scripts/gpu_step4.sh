#!/bin/bash
cd "$(dirname "$0")/.."
timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py -q -p no:cacheprovider 2>&1 | tail -2
python scripts/op_bench.py conv --b 4 --hw 1024 --c 128 --resid --stats --iters 5
python scripts/op_bench.py conv --b 4 --hw 1024 --c 128 --iters 5
python scripts/op_bench.py conv --b 4 --hw 512 --c 256 --resid --stats --iters 5
python scripts/op_bench.py conv --b 4 --hw 256 --c 512 --resid --stats --iters 5
python scripts/op_bench.py subpix --b 4 --hw 512 --c 256 --stats --iters 5
