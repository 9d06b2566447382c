#!/bin/bash
# Fused GroupNorm+SiLU A operand (bit 2) only at the 128-input-channel convs (LBX_FUSE_C=128):
# decode A/B against the default (separate apply passes), same box, interleaved.
cd "$(dirname "$0")/.."
LBX_FUSE_C=128 timeout -s KILL 900 python scripts/ab_decode.py --bits 1 5 --batch 32 --rounds 5 --steps 2 --profile --grep c128
