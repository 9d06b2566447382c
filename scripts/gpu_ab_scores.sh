#!/bin/bash
# A/B of two builds (ab/liblbx_a.so vs in-tree) with the attention rows of the eager profile.
cd "$(dirname "$0")/.."
A=${A:-ab/liblbx_a.so}
for r in 1 2 3; do
  LBX_LIB=$A timeout -s KILL 300 python scripts/ab_lib.py --steps 6
  LBX_LIB=paper_2605_19385_b200/liblbx.so timeout -s KILL 300 python scripts/ab_lib.py --steps 6
done
LBX_LIB=$A timeout -s KILL 300 python scripts/ab_lib.py --steps 2 --profile attn
LBX_LIB=paper_2605_19385_b200/liblbx.so timeout -s KILL 300 python scripts/ab_lib.py --steps 2 --profile attn
