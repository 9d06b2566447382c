#!/bin/bash
# Energy / time of the operand traffic: debug bits 27 (no B loads after a CTA's first tile) and 28
# (no A loads), sustained at the power cap (op_bench --sustain), per conv width.
cd "$(dirname "$0")/.."
S=${S:-4}
run() { echo "$(date +%T) $*"; timeout 90 python scripts/op_bench.py "$@" || echo "rc=$?"; }
python -c "import torch; print(torch.cuda.get_device_name())"
for bits in ${BITS:-134217729 1 268435457 402653185}; do
  echo "bits $bits"
  run conv --b 32 --hw 512 --c 256 --stats --sustain $S --bits $bits
  run conv --b 32 --hw 256 --c 512 --stats --sustain $S --bits $bits
  run conv --b 32 --hw 1024 --c 128 --resid --stats --sustain $S --bits $bits
  run conv --b 32 --hw 1024 --c 128 --stats --sustain $S --bits $bits
done
