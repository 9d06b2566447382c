"""CPU tests: the oracle pinned against its golden vectors, and the product's host-side code
(weight generator, LBLP packer) checked bit-for-bit against the independent oracle restatements.
No GPU needed."""
import json
import os

import numpy as np
import pytest

import lblp
import weights_ref

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_param_counts_match_paper():
    # 49.49 M (SD1.5, 4-ch), 49.55 M (SD3.5 / FLUX, 16-ch)
    assert weights_ref.param_count("sd15") == 49_490_199
    assert weights_ref.param_count("sd3") == 49_545_475
    assert weights_ref.param_count("flux") == 49_545_475


def test_product_param_count_and_generator_match_oracle(lbx):
    for fam in ("sd15", "sd3", "flux"):
        assert lbx.param_count(fam) == weights_ref.param_count(fam)
    for fam, seed in (("sd15", 0), ("sd3", 7)):
        got = lbx.generate_params(fam, seed)
        ref = np.concatenate([v.ravel() for v in weights_ref.make_weights(fam, seed).values()])
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), fam


def test_weights_are_fp16_representable():
    w = weights_ref.make_weights("sd15", 0)
    x = w["decoder.up_blocks.3.resnets.2.conv2.weight"]
    assert np.array_equal(x, x.astype(np.float16).astype(np.float32))


def test_lblp_known_answer_vectors():
    kat = json.load(open(os.path.join(GOLD, "lblp_kat.json")))
    assert len(kat["cases"]) >= 5
    for c in kat["cases"]:
        vals = np.frombuffer(bytes.fromhex(c["values_hex"]), dtype=np.uint16).reshape(c["shape"])
        blob = bytes.fromhex(c["blob_hex"])
        assert lblp.encode(vals.view(np.float16), c["mode"]) == blob, c["name"]
        dec = lblp.decode(blob, *c["shape"]).view(np.uint16)
        assert dec.tobytes().hex() == c["decoded_hex"], c["name"]
        if c["mode"] in (0, 1, 3):
            assert np.array_equal(dec, vals)
    assert {c["mode"] for c in kat["cases"]} == {0, 1, 2, 3}


@pytest.mark.parametrize("mode", [0, 1, 2, 3])
@pytest.mark.parametrize("shape,smooth", [((4, 64, 64), False), ((16, 128, 128), True), ((2, 3, 32), False)])
def test_product_packer_bytes_equal_oracle_encoder(lbx, mode, shape, smooth):
    c, h, w = shape
    rng = np.random.default_rng(c * h + mode)
    if smooth:
        z = weights_ref.make_latents("sd3", 1, h, w, seed=3, smooth=True)[0][:c]
    else:
        z = rng.standard_normal(shape).astype(np.float16)
    assert lbx.pack(z, mode) == lblp.encode(z, mode)


def test_product_packer_special_values(lbx):
    special = np.array([0x0000, 0x8000, 0x0001, 0x8001, 0x03FF, 0x83FF, 0x0400, 0x7BFF, 0xFBFF, 0x7C00, 0xFC00,
                        0x7E00, 0x7C01, 0xFE01, 0x3C00, 0xBC00], dtype=np.uint16)
    z = np.resize(special, (3, 4, 64)).astype(np.uint16)
    z[1] = np.random.default_rng(5).integers(0, 65536, (4, 64), dtype=np.uint16)  # arbitrary bit patterns
    for mode in (0, 1, 3):
        b = lbx.pack(z.view(np.float16), mode)
        assert b == lblp.encode(z.view(np.float16), mode)
        assert np.array_equal(lblp.decode(b, 3, 4, 64).view(np.uint16), z)
    const = np.full((2, 8, 32), 0x3C00, dtype=np.uint16)  # one bin, zero-cost symbols, no renormalisation
    b = lbx.pack(const.view(np.float16), 3)
    assert b == lblp.encode(const.view(np.float16), 3)
    assert np.array_equal(lblp.decode(b, 2, 8, 32).view(np.uint16), const)


def test_packer_rejects_bad_arguments(lbx):
    with pytest.raises(lbx.LbxError) as e:
        lbx.pack(np.zeros((2, 4, 48), dtype=np.float16), 1)  # W % 32 != 0 in mode 1
    assert e.value.status == lbx.E_CONFIG
    with pytest.raises(lbx.LbxError):
        lbx.pack(np.zeros((2, 4, 64), dtype=np.float16), 7)
    with pytest.raises(lbx.LbxError):
        lbx.pack(np.zeros((1, 4, 48), dtype=np.float16), 3)  # mode 3: W % 32 != 0
    with pytest.raises(lbx.LbxError):
        lbx.pack(np.zeros((1, 256, 128), dtype=np.float16), 3)  # mode 3: plane > 16384 values


def test_oracle_decoder_reproduces_config1_golden():
    """The committed config-1 fixture is what the oracle produces (guards oracle drift)."""
    import vae_ref
    g = np.load(os.path.join(GOLD, "decode_sd15_64_seed1.npz"))
    ref = vae_ref.decode(g["latents"], weights_ref.make_weights("sd15", int(g["weight_seed"])), "sd15")
    assert np.array_equal(ref, g["rgb"])


def test_oracle_lossless_roundtrip_and_ratio():
    z = weights_ref.make_latents("sd3", 1, 128, 128, seed=3)[0]
    b = lblp.encode(z, 1)
    assert np.array_equal(lblp.decode(b, 16, 128, 128).view(np.uint16), z.view(np.uint16))
    q = lblp.encode(z, 2)
    assert len(q) == 32 + 8 * 16 + z.size  # q8: 1 byte per value
    err = np.abs(lblp.decode(q, 16, 128, 128).astype(np.float32) - z.astype(np.float32))
    assert err.max() < 0.05


@pytest.mark.parametrize("fixture", ["pin_cheers_sd15_64_seed1.npz", "pin_cheers_sd3_32_seed5.npz",
                                     "pin_cheers_flux_32_seed6.npz"])
def test_oracle_pinned_to_independent_decoder(fixture):
    """The oracle against outputs of an independent implementation of the same decoder (vllm 0.22's
    CheersVAEDecoder, the CompVis/LDM Decoder; generated by tests/golden/pin_vllm_cheers.py with the
    same seeded weights and latents).  Bar: uint8 max |diff| <= 1 with >= 99.99% identical (the
    remaining pixels sit on a rounding boundary, fp32 noise ~4e-6), float output within 2e-5."""
    import vae_ref
    g = np.load(os.path.join(GOLD, fixture))
    fam = str(g["family"])
    w = weights_ref.make_weights(fam, int(g["weight_seed"]))
    img = vae_ref.decode_float(g["latents"], w, fam)
    st = vae_ref.pixel_stats(vae_ref.to_uint8(img), g["rgb"])
    assert st["max_abs"] <= 1 and st["frac_exact"] >= 0.9999, st
    if "float_out" in g:
        assert float(np.abs(img.numpy() - g["float_out"]).max()) <= 2e-5
    rep = json.load(open(os.path.join(GOLD, "pin_cheers.json")))
    case = next(c for c in rep["cases"] if c["fixture"] == fixture)
    assert case["cheers_params"] == case["oracle_params"] and case["max_abs_float_diff"] <= 2e-5


@pytest.mark.parametrize("smooth", [False, True])
def test_entropy_mode_roundtrip_and_ratio(lbx, smooth):
    """LBLP mode 3 (binned rANS, the pcodec algorithm class): lossless, and smaller than mode 1 --
    16x128x128 N(0,1) latents at < 0.9 of raw fp16 (order-0 entropy 0.84), smooth ones < 0.8."""
    z = weights_ref.make_latents("sd3", 1, 128, 128, seed=3, smooth=smooth)[0]
    b = lbx.pack(z, 3)
    assert b == lblp.encode(z, 3)
    assert np.array_equal(lblp.decode(b, 16, 128, 128).view(np.uint16), z.view(np.uint16))
    assert len(b) < len(lbx.pack(z, 1))
    assert len(b) / z.nbytes < (0.80 if smooth else 0.90)
