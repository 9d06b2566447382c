#!/bin/bash
# Old build (ab/liblbx_a.so, before the fused-exp attention) vs the in-tree build: with bits 9 the new
# build runs the two-pass attention, so the difference is the conv epilogue's extra branches; with
# bits 1 it is the whole change.
cd "$(dirname "$0")/.."
bash scripts/gpu_ab_lib.sh --bits 9
echo "---- bits 1"
A=ab/liblbx_a.so
for r in 1 2 3; do
  LBX_LIB=$A timeout -s KILL 300 python scripts/ab_lib.py --steps 6 --bits 1
  LBX_LIB=paper_2605_19385_b200/liblbx.so timeout -s KILL 300 python scripts/ab_lib.py --steps 6 --bits 1
done
