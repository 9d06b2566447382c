#!/bin/bash
# Shared-memory / pipe counters of the plain vs fused-GroupNorm (XF) conv (is the smem port the
# XF bottleneck?).  Raw-page CSVs of one launch each, batch 8.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for shp in "256 512" "1024 128"; do
  set -- $shp
  for f in "" "--gnfuse"; do
    tag=smem_${1}_${2}${f:+_fused}
    timeout -s KILL 600 ncu --set full --clock-control none -k regex:gemm_tc_kernel -s 1 -c 1 \
      -o gpurun_out/$tag python scripts/op_bench.py conv --b 8 --hw $1 --c $2 --stats $f --iters 1 > /dev/null 2>&1
    ncu -i gpurun_out/$tag.ncu-rep --page raw --csv > gpurun_out/$tag.csv 2>/dev/null
    rm -f gpurun_out/$tag.ncu-rep
  done
done
ls -la gpurun_out/smem_*.csv
