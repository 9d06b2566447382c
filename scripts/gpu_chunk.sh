#!/bin/bash
# Conv launches split into whole-image chunks (LBX_CONV_CHUNK=4 / 8) vs one launch per batch (0):
# decode time interleaved, rgb checksum (bit-identical expected), per-conv eager profile.
cd "$(dirname "$0")/.."
for r in 1 2 3; do
  for v in 0 8 4; do echo -n "CHUNK=$v "; LBX_CONV_CHUNK=$v timeout -s KILL 300 python scripts/ab_lib.py --steps 6; done
done
for v in 0 8; do echo "CHUNK=$v"; LBX_CONV_CHUNK=$v timeout -s KILL 300 python scripts/ab_lib.py --steps 2 --profile conv; done
