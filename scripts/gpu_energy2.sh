#!/bin/bash
cd "$(dirname "$0")/.."
S=4
python scripts/op_bench.py conv --b 32 --hw 1024 --c 128 --fold --stats --sustain $S
python scripts/op_bench.py conv --b 32 --hw 1024 --c 128 --resid --stats --sustain $S
python scripts/op_bench.py conv --b 32 --hw 1024 --c 128 --sustain $S
python scripts/op_bench.py conv --b 32 --hw 1024 --c 128 --stats --sustain $S --bits 65
python scripts/op_bench.py conv --b 32 --hw 1024 --c 128 --stats --sustain $S --bits 3
python scripts/op_bench.py conv --b 32 --hw 1024 --c 128 --n 256 --stats --sustain $S
