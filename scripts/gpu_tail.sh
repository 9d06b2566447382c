#!/bin/bash
# conv_out_tc A/B: two transform groups (new) vs one (liblbx_old.so); tail op tests; decode A/B.
cd "$(dirname "$0")/.."
timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider --timeout=120 -k "conv_out" 2>&1 | tail -2
for r in 1 2 3; do
  for lib in paper_2605_19385_b200/liblbx_old.so paper_2605_19385_b200/liblbx.so; do
    echo -n "$(basename $lib): "; LBX_LIB=$PWD/$lib timeout -s KILL 120 python scripts/op_bench.py tail --b 32 --hw 1024 --iters 10
  done
done
for lib in paper_2605_19385_b200/liblbx_old.so paper_2605_19385_b200/liblbx.so; do
  echo -n "$(basename $lib): "; LBX_LIB=$PWD/$lib timeout -s KILL 120 python scripts/op_bench.py tail --b 32 --hw 1024 --sustain 3
done
A=paper_2605_19385_b200/liblbx_old.so bash scripts/gpu_ab_lib.sh --profile conv_out
