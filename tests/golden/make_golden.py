"""Generate the committed golden fixtures under tests/golden/ from the CPU oracle.

  decode_sd15_64_seed1.npz   config 1: sd15 4x64x64 latent (seed 1) -> 512^2 uint8, weights seed 0
  decode_sd3_128_seed3.npz   configs 3/4 shape: sd3 16x128x128 latent (seed 3) -> 1024^2 uint8, weights seed 0
  lblp_kat.json              LBLP v1 known-answer vectors (oracle encoder), modes 0/1/2

The reference has no decoder or codec to run; these vectors pin the product to the
oracle restatement across machines (the GPU box does not have /root/reference).
Usage: python tests/golden/make_golden.py  (about a minute on 8 cores)
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))

import lblp  # noqa: E402
import vae_ref  # noqa: E402
import weights_ref  # noqa: E402


def decode_fixture(family, h, seed, wseed, name):
    z = weights_ref.make_latents(family, 1, h, h, seed=seed)
    img = vae_ref.decode_float(z, weights_ref.make_weights(family, wseed), family)
    rgb = vae_ref.to_uint8(img)
    np.savez_compressed(os.path.join(HERE, name), latents=z, rgb=rgb, weight_seed=np.int64(wseed),
                        family=np.array(family))
    print(name, rgb.shape, hashlib.sha256(rgb.tobytes()).hexdigest()[:16])


def kat():
    special = np.array([0x0000, 0x8000, 0x0001, 0x8001, 0x03FF, 0x83FF, 0x0400, 0x7BFF, 0xFBFF, 0x7C00, 0xFC00,
                        0x7E00, 0x7C01, 0xFE01, 0x3C00, 0xBC00], dtype=np.uint16)
    rng = np.random.default_rng(1234)
    cases = []
    # 2 x 2 x 64: row 0 = specials, row 1 = smooth ramp, row 2 = constant, row 3 = random bits
    x = np.zeros((2, 2, 64), dtype=np.uint16)
    x[0, 0] = np.resize(special, 64)
    x[0, 1] = np.linspace(-2, 2, 64).astype(np.float16).view(np.uint16)
    x[1, 0] = 0x3C00
    x[1, 1] = rng.integers(0, 65536, 64, dtype=np.uint16)
    y = rng.standard_normal((2, 4, 32)).astype(np.float16).view(np.uint16)
    for name, arr in (("mixed_2x2x64", x), ("normal_2x4x32", y)):
        for mode in (0, 1, 2, 3):
            if mode == 2 and name == "mixed_2x2x64":
                continue  # q8 of inf/NaN is saturating by design; KAT uses finite data
            blob = lblp.encode(arr.view(np.float16), mode)
            dec = lblp.decode(blob, *arr.shape).view(np.uint16)
            cases.append({"name": name, "mode": mode, "shape": list(arr.shape),
                          "values_hex": arr.tobytes().hex(), "blob_hex": blob.hex(),
                          "decoded_hex": dec.tobytes().hex()})
    with open(os.path.join(HERE, "lblp_kat.json"), "w") as f:
        json.dump({"format": "LBLP v1 (include/lbx/lblp.h)", "cases": cases}, f, indent=1)
    print("lblp_kat.json", len(cases), "cases")


if __name__ == "__main__":
    kat()
    decode_fixture("sd15", 64, 1, 0, "decode_sd15_64_seed1.npz")
    decode_fixture("sd3", 128, 3, 0, "decode_sd3_128_seed3.npz")
