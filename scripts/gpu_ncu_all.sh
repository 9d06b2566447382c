#!/bin/bash
# ncu --set full of one launch of every kernel class (scripts/ncu_kernels.py): the eager decode's
# launches (second profile call) plus pack / unpack / PNG.  Summarise here with tools/ncu_summary.py.
cd "$(dirname "$0")/.."
TAG=${1:-r2}
mkdir -p gpurun_out
N=$(timeout -s KILL 300 python scripts/ncu_kernels.py --batch 8 | grep "launches per decode" | awk '{print $4}')
echo "launches per decode: $N"
timeout -s KILL 2400 ncu --set full --clock-control none -s $N \
  -k regex:'gemm_tc|gn_apply|softmax|attn_|conv_out|latent_prep|gn_finalize|lblp|png_' \
  -o gpurun_out/ncu_all_$TAG python scripts/ncu_kernels.py --batch 8 > gpurun_out/ncu_all_$TAG.log 2>&1
tail -n 3 gpurun_out/ncu_all_$TAG.log
ls -la gpurun_out/ncu_all_$TAG.ncu-rep
# summarise on the box (the full report is ~200 MB, above gpurun's copy-back limit)
python tools/ncu_summary.py gpurun_out/ncu_all_$TAG.ncu-rep > gpurun_out/ncu_kernels_$TAG.tsv && rm -f gpurun_out/ncu_all_$TAG.ncu-rep
wc -l gpurun_out/ncu_kernels_$TAG.tsv
