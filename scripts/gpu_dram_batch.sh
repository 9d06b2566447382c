#!/bin/bash
# DRAM read bytes of one c256 @512^2 conv (and c128 @1024^2 + residual) vs batch size: does the halo
# re-read excess grow with the launch length?
cd "$(dirname "$0")/.."
for b in 4 8 16 32; do
  for cfg in "--hw 512 --c 256" "--hw 1024 --c 128 --resid"; do
    timeout -s KILL 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none \
      -k regex:gemm_tc -s 1 -c 1 python scripts/op_bench.py conv --b $b $cfg --stats --iters 1 2>&1 | grep -E "dram__|duration" | sed "s/^/b$b $cfg /"
  done
done
