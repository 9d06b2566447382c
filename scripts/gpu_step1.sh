#!/bin/bash
# First GPU bring-up: kernel-level parity, then the decoder end to end.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout -s KILL 120 python -m pytest tests/test_gpu_gemm.py -x -q -k "test_plain_gemm and 1-128 and 256-256-64" 2>&1 | tail -15
timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py -q -p no:cacheprovider 2>&1 | tail -40
timeout -s KILL 600 python -m pytest tests/test_gpu_unpack.py tests/test_gpu_decode.py -q -s -p no:cacheprovider 2>&1 | tail -60
