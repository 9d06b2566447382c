"""ORACLE (test infrastructure only) -- deterministic decoder weights, numpy restatement.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import this module.
The product generates the same weights in C++ (paper_2605_19385_b200/csrc/weights.cpp); the two
implementations are written independently and must agree bit-for-bit (tests/test_oracle_cpu.py).

Architecture: AutoencoderKL decoder as pinned by PAPER.md:386-391 (49.49 M / 49.55 M params) and
SURVEY.md Appendix A (block_out_channels (128,256,512,512), 3 resnets per up block, GroupNorm-32,
1-head mid attention, nearest-2x upsample in the first three up blocks).  The reference repository
has no decoder at all (decode is the constant proj/src/sim.cpp:414), so parameter
*names* follow the diffusers AutoencoderKL state-dict convention (third-party, not vendored).

Generator (the contract, restated in DESIGN.md section 3):
  counter-based splitmix64 over (seed, tensor_id, element) -- same finalizer as the reference's
  ring hash mix64 (proj/src/router.cpp:30-37):
      z  = (seed + 1) * 0x9E3779B97F4A7C15  ^  (tensor_id + 1) * 0xC2B2AE3D27D4EB4F
      z += (element + 1) * 0xD1B54A32D192ED03            (all mod 2^64)
      z  = mix64(z);  u = (z >> 11) * 2^-53              (u in [0,1), exact in double)
  conv / linear weight:  (2u-1) / sqrt(fan_in)  -> rounded to fp32 -> rounded to fp16
                         (the decoder is an fp16 model; the oracle computes in
                         fp32/fp64 with these fp16-valued weights)
  conv / linear bias:    (2u-1) / sqrt(fan_in)  -> fp32
  GroupNorm gamma:       1 + 0.25 (2u-1)        -> fp32
  GroupNorm beta:        0.25 (2u-1)            -> fp32
"""
from __future__ import annotations

import numpy as np

FAMILIES = {
    # name: (latent_channels, scaling_factor, shift_factor, post_quant_conv)
    "sd15": (4, 0.18215, 0.0, True),
    "sd3": (16, 1.5305, 0.0609, False),
    "flux": (16, 0.3611, 0.1159, False),
}

BLOCK_OUT = (128, 256, 512, 512)
LAYERS_PER_BLOCK = 2
GROUPS = 32
EPS = 1e-6


def param_specs(latent_channels: int, post_quant: bool):
    """Canonical parameter order: list of (name, shape, kind, fan_in); tensor_id = list index."""
    specs = []

    def conv(name, cin, cout, k):
        fan = cin * k * k
        specs.append((name + ".weight", (cout, cin, k, k), "w", fan))
        specs.append((name + ".bias", (cout,), "b", fan))

    def linear(name, cin, cout):
        specs.append((name + ".weight", (cout, cin), "w", cin))
        specs.append((name + ".bias", (cout,), "b", cin))

    def norm(name, c):
        specs.append((name + ".weight", (c,), "gamma", 0))
        specs.append((name + ".bias", (c,), "beta", 0))

    def resnet(name, cin, cout):
        norm(name + ".norm1", cin)
        conv(name + ".conv1", cin, cout, 3)
        norm(name + ".norm2", cout)
        conv(name + ".conv2", cout, cout, 3)
        if cin != cout:
            conv(name + ".conv_shortcut", cin, cout, 1)

    top = BLOCK_OUT[-1]
    if post_quant:
        conv("post_quant_conv", latent_channels, latent_channels, 1)
    conv("decoder.conv_in", latent_channels, top, 3)
    resnet("decoder.mid_block.resnets.0", top, top)
    a = "decoder.mid_block.attentions.0"
    norm(a + ".group_norm", top)
    linear(a + ".to_q", top, top)
    linear(a + ".to_k", top, top)
    linear(a + ".to_v", top, top)
    linear(a + ".to_out.0", top, top)
    resnet("decoder.mid_block.resnets.1", top, top)
    prev = top
    rev = list(reversed(BLOCK_OUT))
    for i, out in enumerate(rev):
        for j in range(LAYERS_PER_BLOCK + 1):
            resnet(f"decoder.up_blocks.{i}.resnets.{j}", prev if j == 0 else out, out)
        if i < len(rev) - 1:
            conv(f"decoder.up_blocks.{i}.upsamplers.0.conv", out, out, 3)
        prev = out
    norm("decoder.conv_norm_out", BLOCK_OUT[0])
    conv("decoder.conv_out", BLOCK_OUT[0], 3, 3)
    return specs


_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _uniform(seed: int, tensor_id: int, n: int) -> np.ndarray:
    """u in [0,1) as float64, one per element (splitmix64 counter hash)."""
    with np.errstate(over="ignore"):
        base = (np.uint64((seed + 1) & 0xFFFFFFFFFFFFFFFF) * np.uint64(0x9E3779B97F4A7C15)) ^ (
            np.uint64(tensor_id + 1) * np.uint64(0xC2B2AE3D27D4EB4F))
        idx = np.arange(1, n + 1, dtype=np.uint64)
        z = base + idx * np.uint64(0xD1B54A32D192ED03)
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def make_weights(family: str = "sd15", seed: int = 0) -> dict:
    """name -> np.ndarray (float32; conv/linear weights hold fp16-representable values)."""
    cl, _, _, pq = FAMILIES[family]
    out = {}
    for tid, (name, shape, kind, fan) in enumerate(param_specs(cl, pq)):
        n = int(np.prod(shape))
        s = 2.0 * _uniform(seed, tid, n) - 1.0
        if kind == "w":
            v = (s / np.sqrt(float(fan))).astype(np.float32).astype(np.float16).astype(np.float32)
        elif kind == "b":
            v = (s / np.sqrt(float(fan))).astype(np.float32)
        elif kind == "gamma":
            v = (1.0 + 0.25 * s).astype(np.float32)
        else:
            v = (0.25 * s).astype(np.float32)
        out[name] = v.reshape(shape)
    return out


def param_count(family: str) -> int:
    cl, _, _, pq = FAMILIES[family]
    return sum(int(np.prod(s)) for _, s, _, _ in param_specs(cl, pq))


def make_latents(family: str, n: int, h: int, w: int, seed: int, smooth: bool = False) -> np.ndarray:
    """Synthetic latents, fp16 NCHW.  i.i.d. N(0,1), or (smooth=True) a bilinear-upsampled 16x16
    noise field plus small noise -- closer to real latents for codec-ratio realism."""
    cl = FAMILIES[family][0]
    rng = np.random.default_rng(seed)
    if not smooth:
        return rng.standard_normal((n, cl, h, w), dtype=np.float32).astype(np.float16)
    coarse = rng.standard_normal((n, cl, 16, 16), dtype=np.float32)
    ys = (np.arange(h) + 0.5) * 16 / h - 0.5
    xs = (np.arange(w) + 0.5) * 16 / w - 0.5
    y0 = np.clip(np.floor(ys).astype(int), 0, 15)
    x0 = np.clip(np.floor(xs).astype(int), 0, 15)
    y1 = np.clip(y0 + 1, 0, 15)
    x1 = np.clip(x0 + 1, 0, 15)
    fy = np.clip(ys - y0, 0, 1)[:, None]
    fx = np.clip(xs - x0, 0, 1)[None, :]
    c = coarse
    top = c[:, :, y0][:, :, :, x0] * (1 - fx) + c[:, :, y0][:, :, :, x1] * fx
    bot = c[:, :, y1][:, :, :, x0] * (1 - fx) + c[:, :, y1][:, :, :, x1] * fx
    field = top * (1 - fy) + bot * fy
    field += 0.05 * rng.standard_normal(field.shape, dtype=np.float32)
    return field.astype(np.float16)
