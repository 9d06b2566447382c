#!/bin/bash
# Fused-exp attention scores: parity tests (incl. the peaked-score fallback), the decode A/B against
# the two-pass softmax (bit 3), and the bench's roofline leg.
cd "$(dirname "$0")/.."
timeout -s KILL 900 python -m pytest tests/test_gpu_decode.py -q -x -s -p no:cacheprovider --timeout=300 -k "attention or config1 or batch_invariance" 2>&1 | grep -E "^\[|passed|failed|Error|assert" | tail -40
timeout -s KILL 600 python scripts/ab_decode.py --bits 1 9 --batch 32 --rounds 4 --steps 2 --profile --grep attn
