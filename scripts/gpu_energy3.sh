#!/bin/bash
cd "$(dirname "$0")/.."
S=4
python scripts/op_bench.py conv --b 32 --hw 1024 --c 128 --fold --stats --gnfuse --sustain $S --bits 5
python scripts/op_bench.py conv --b 32 --hw 1024 --c 128 --stats --gnfuse --sustain $S --bits 5
python scripts/op_bench.py conv --b 32 --hw 512 --c 256 --resid --stats --gnfuse --sustain $S --bits 5
python scripts/op_bench.py conv --b 32 --hw 256 --c 512 --resid --stats --gnfuse --sustain $S --bits 5
timeout -s KILL 600 python scripts/ab_decode.py --bits 1 --batch 32 --rounds 3 --steps 3 --profile --grep gn_apply
