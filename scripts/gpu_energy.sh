#!/bin/bash
# Sustained (power-capped) rate and power per kernel type: where the energy of a decode goes.
cd "$(dirname "$0")/.."
S=4
python scripts/op_bench.py conv --b 32 --hw 1024 --c 128 --fold --stats --sustain $S
python scripts/op_bench.py conv --b 32 --hw 1024 --c 128 --stats --sustain $S
python scripts/op_bench.py conv --b 32 --hw 512 --c 256 --resid --stats --sustain $S
python scripts/op_bench.py conv --b 32 --hw 256 --c 512 --resid --stats --sustain $S
python scripts/op_bench.py conv --b 32 --hw 256 --c 512 --stats --sustain $S
python scripts/op_bench.py subpix --b 32 --hw 512 --c 256 --stats --sustain $S
python scripts/op_bench.py gemm --b 1 --hw 128 --n 16384 --k 512 --sustain $S
python scripts/op_bench.py gn --b 32 --hw 1024 --c 128 --sustain $S
