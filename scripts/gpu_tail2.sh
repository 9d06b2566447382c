#!/bin/bash
# conv_out_tc variants (transform groups x chunks in flight), op level at batch 32, interleaved.
cd "$(dirname "$0")/.."
timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider --timeout=120 -k "conv_out" 2>&1 | tail -1
for r in 1 2 3; do
  for lib in ab/liblbx_co33.so ab/liblbx_co32.so ab/liblbx_co31.so ab/liblbx_co23.so ab/liblbx_co22.so; do
    echo -n "$(basename $lib): "; LBX_LIB=$PWD/$lib timeout -s KILL 120 python scripts/op_bench.py tail --b 32 --hw 1024 --iters 10
  done
done
