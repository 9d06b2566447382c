#!/bin/bash
cd "$(dirname "$0")/.."
for c_hw in "256 512" "256 1024" "128 1024" "512 256"; do
  set -- $c_hw
  for bits in 1 2049 257; do
    for ip in "" "--inplace"; do
      echo -n "c$1 hw$2 bits$bits $ip: "; python scripts/op_bench.py gn --b 32 --hw $2 --c $1 --iters 5 --bits $bits $ip | awk '{print $(NF-3), $(NF-2), $(NF-1), $NF}'
    done
  done
done
