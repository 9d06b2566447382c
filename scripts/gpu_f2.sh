#!/bin/bash
# Packed fp32 (FFMA2/FADD2/FMUL2) + small-image tiles: op/decode tests, decode A/B vs ab/liblbx_a.so,
# config-1 latency with and without the small-image tile policy (bit 3 clears it).
cd "$(dirname "$0")/.."
timeout -s KILL 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_decode.py -q -x -p no:cacheprovider --timeout=300 2>&1 | tail -2
for r in 1 2 3; do
  LBX_LIB=$PWD/ab/liblbx_a.so timeout -s KILL 300 python scripts/ab_lib.py --steps 6
  timeout -s KILL 300 python scripts/ab_lib.py --steps 6
done
S="--b 8 --hw 1024 --c 128 --stats"
for lib in ab/liblbx_a.so paper_2605_19385_b200/liblbx.so; do
  echo "== $lib"
  LBX_LIB=$PWD/$lib python scripts/op_bench.py conv $S --resid --iters 10
  LBX_LIB=$PWD/$lib python scripts/op_bench.py conv $S --resid --sustain 3
  LBX_LIB=$PWD/$lib python scripts/op_bench.py tail --b 32 --hw 1024 --iters 10
done
for b in 1 9 1 9; do python scripts/prof_c1.py $b | grep -E "bits|64x64|graph"; done
