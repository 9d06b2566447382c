#!/bin/bash
# ncu --set full (with source) of the fused GroupNorm+SiLU A-operand (XF) conv kernel and the plain
# conv it replaces, at c128@1024^2 and c512@256^2 (batch 8); summarised on the box.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
OUT=gpurun_out/ncu_xf_r2.txt
: > $OUT
for shp in "1024 128" "256 512"; do
  set -- $shp
  for f in "" "--gnfuse"; do
    tag=xf_${1}_${2}${f:+_fused}
    timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1 -c 1 \
      -o gpurun_out/$tag python scripts/op_bench.py conv --b 8 --hw $1 --c $2 --stats $f --iters 1 > /dev/null 2>&1
    echo "=== $tag (op_bench conv --b 8 --hw $1 --c $2 --stats $f)" >> $OUT
    python tools/ncu_summary.py gpurun_out/$tag.ncu-rep | tail -n +2 >> $OUT
    python tools/ncu_lines.py gpurun_out/$tag.ncu-rep --top 12 --range producers:267-522 --range xf_transform:524-602 \
      --range epilogue:603-912 >> $OUT
    python tools/ncu_waits.py gpurun_out/$tag.ncu-rep >> $OUT
    rm -f gpurun_out/$tag.ncu-rep
  done
done
wc -l $OUT
