#!/bin/bash
# f16x2 exponent for the fused-exp score GEMM (debug bit 30): parity vs the oracle, decode A/B.
cd "$(dirname "$0")/.."
timeout -s KILL 600 python - <<'PY'
import sys; sys.path[:0] = ["oracle", "."]
import numpy as np, vae_ref, weights_ref, paper_2605_19385_b200 as lbx
for fam, n, seed in (("sd15", 1, 1), ("sd3", 2, 5)):
    z = weights_ref.make_latents(fam, n, 64, 64, seed=seed)
    ref = vae_ref.decode(z, weights_ref.make_weights(fam, 0), fam)
    for bits in (1, 1 | (1 << 30)):
        lbx.check(lbx.lib().lbx_op_set_debug(bits, 0))
        got = lbx.Decoder(fam, (64, 64), seed=0, max_batch=n).reconstruct_latents(z)
        print(fam, bits, vae_ref.pixel_stats(got, ref))
PY
timeout -s KILL 600 python scripts/ab_decode.py --bits 1 1073741825 --batch 32 --rounds 4 --steps 2 --profile --grep scores
