#!/bin/bash
# A/B two builds of liblbx.so on one GPU, alternating processes: ab/liblbx_a.so vs the in-tree build.
cd "$(dirname "$0")/.."
A=${A:-ab/liblbx_a.so}
B=paper_2605_19385_b200/liblbx.so
for r in 1 2 3; do
  LBX_LIB=$A timeout -s KILL 300 python scripts/ab_lib.py --steps 6 "$@"
  LBX_LIB=$B timeout -s KILL 300 python scripts/ab_lib.py --steps 6 "$@"
done
LBX_LIB=$A timeout -s KILL 300 python scripts/ab_lib.py --steps 2 --profile conv "$@"
LBX_LIB=$B timeout -s KILL 300 python scripts/ab_lib.py --steps 2 --profile conv "$@"
