#!/bin/bash
# L2 evict_last hint on the conv halo loads (LBX_A_HINT=1) vs none: DRAM bytes per launch (ncu),
# sustained energy per TFLOP, and the decode.
cd "$(dirname "$0")/.."
for v in 0 1; do
  for cfg in "--hw 512 --c 256" "--hw 1024 --c 128 --resid"; do
    LBX_A_HINT=$v timeout -s KILL 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:gemm_tc -s 1 -c 1 python scripts/op_bench.py conv --b 32 $cfg --stats --iters 1 2>&1 | grep -E "dram__|duration" | sed "s/^/A_HINT=$v $cfg /"
  done
done
for r in 1 2; do
  for v in 0 1; do
    echo "A_HINT=$v"
    LBX_A_HINT=$v timeout 120 python scripts/op_bench.py conv --b 32 --hw 512 --c 256 --stats --sustain 4
    LBX_A_HINT=$v timeout 120 python scripts/op_bench.py conv --b 32 --hw 1024 --c 128 --resid --stats --sustain 4
  done
done
for r in 1 2 3; do
  for v in 0 1; do echo -n "A_HINT=$v "; LBX_A_HINT=$v timeout -s KILL 300 python scripts/ab_lib.py --steps 6; done
done
