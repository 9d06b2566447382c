#!/bin/bash
# Fused-exp attention scores: parity tests (incl. the peaked-score fallback and its counter).
cd "$(dirname "$0")/.."
timeout -s KILL 900 python -m pytest tests/test_gpu_decode.py -q -x -s -p no:cacheprovider --timeout=300 -k "attention or config1 or batch_invariance" 2>&1 | grep -E "^\[|passed|failed|Error|assert" | tail -40
