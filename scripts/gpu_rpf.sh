#!/bin/bash
cd "$(dirname "$0")/.."
timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_decode.py -q -x -p no:cacheprovider --timeout=120 2>&1 | tail -2
python scripts/op_bench.py conv --b 32 --hw 1024 --c 128 --resid --stats --sustain 4
python scripts/op_bench.py conv --b 32 --hw 1024 --c 128 --fold --stats --sustain 4
python scripts/op_bench.py conv --b 32 --hw 512 --c 256 --resid --stats --sustain 4
python scripts/op_bench.py conv --b 32 --hw 256 --c 512 --resid --stats --sustain 4
timeout -s KILL 600 python scripts/ab_decode.py --bits 1025 1 --batch 32 --rounds 3 --steps 2 --profile --grep conv2
