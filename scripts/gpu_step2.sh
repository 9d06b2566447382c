#!/bin/bash
cd "$(dirname "$0")/.."
timeout -s KILL 300 python -m pytest tests/test_gpu_gemm.py -q -p no:cacheprovider -k subpixel 2>&1 | tail -5
timeout -s KILL 900 python -m pytest tests/test_gpu_unpack.py tests/test_gpu_decode.py -q -s -p no:cacheprovider 2>&1 | grep -vE "^\s*$" | tail -80
