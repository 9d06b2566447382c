#!/bin/bash
# Interleaved decode A/B of environment settings (each arm a fresh process): "NAME=VALUE ..." per arm.
cd "$(dirname "$0")/.."
ARMS=("$@")
for r in 1 2 3; do
  for arm in "${ARMS[@]}"; do echo -n "[$arm] "; env $arm timeout -s KILL 300 python scripts/ab_lib.py --steps 6; done
done
