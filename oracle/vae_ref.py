"""ORACLE (test infrastructure only) -- CPU restatement of the decode-on-miss reconstruction.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module; the product path (paper_2605_19385_b200) never does.

What it restates.  The reference models decode as a constant 40 ms service time
(proj/src/sim.cpp:409-442, proj/include/latentbox/sim.hpp:19) and explicitly scopes the real decoder
out.  The decoder is pinned by the paper instead: "a deterministic feed-forward neural
network" x = D(z), an AutoencoderKL decoder of 49.49 M / 49.55 M parameters
(PAPER.md:386-391), fp16.  Layer order:
  [post_quant_conv 1x1] -> conv_in 3x3 -> mid(Res, Attn, Res) -> 4 up blocks (3 Res each, nearest-2x
  upsample + conv3x3 after the first three) -> GroupNorm -> SiLU -> conv_out 3x3 -> RGB.
Res(x) = x' + conv2(SiLU(GN2(conv1(SiLU(GN1(x))))))  with x' = x or conv_shortcut_1x1(x).
Attn(x) = x + out(softmax(Q K^T / sqrt(512)) V),  Q,K,V = Linear(GN(x)) over h*w tokens, 1 head.
Latent pre-scale z/scaling + shift; post-process (x/2 + 0.5).clamp(0,1) * 255, round-half-even.

Parity status: the decoder has no reference implementation to run -- the oracle is
pinned only by the paper's parameter counts (checked in tests) and by this restatement; see
DESIGN.md "parity unpinned" note.
"""
from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F

from weights_ref import BLOCK_OUT, EPS, FAMILIES, GROUPS, LAYERS_PER_BLOCK


def _t(w, name, dtype):
    return torch.from_numpy(np.ascontiguousarray(w[name])).to(dtype)


def _gn(x, w, name, dtype):
    return F.group_norm(x, GROUPS, _t(w, name + ".weight", dtype), _t(w, name + ".bias", dtype), EPS)


def _conv(x, w, name, dtype, pad):
    return F.conv2d(x, _t(w, name + ".weight", dtype), _t(w, name + ".bias", dtype), padding=pad)


def _resnet(x, w, name, dtype):
    h = _conv(F.silu(_gn(x, w, name + ".norm1", dtype)), w, name + ".conv1", dtype, 1)
    h = _conv(F.silu(_gn(h, w, name + ".norm2", dtype)), w, name + ".conv2", dtype, 1)
    if name + ".conv_shortcut.weight" in w:
        x = _conv(x, w, name + ".conv_shortcut", dtype, 0)
    return x + h


def _attention(x, w, name, dtype):
    b, c, hh, ww = x.shape
    h = _gn(x, w, name + ".group_norm", dtype).reshape(b, c, hh * ww).transpose(1, 2)
    q = F.linear(h, _t(w, name + ".to_q.weight", dtype), _t(w, name + ".to_q.bias", dtype))
    k = F.linear(h, _t(w, name + ".to_k.weight", dtype), _t(w, name + ".to_k.bias", dtype))
    v = F.linear(h, _t(w, name + ".to_v.weight", dtype), _t(w, name + ".to_v.bias", dtype))
    outs = []
    for i in range(b):  # one image at a time bounds the L x L score matrix
        s = (q[i] @ k[i].transpose(0, 1)) * (1.0 / math.sqrt(c))
        p = torch.softmax(s, dim=-1)
        outs.append(p @ v[i])
    o = torch.stack(outs)
    o = F.linear(o, _t(w, name + ".to_out.0.weight", dtype), _t(w, name + ".to_out.0.bias", dtype))
    return x + o.transpose(1, 2).reshape(b, c, hh, ww)


def decode_float(latents: np.ndarray, weights: dict, family: str, dtype=torch.float32,
                 threads: int | None = None) -> torch.Tensor:
    """fp16 NCHW latents -> float image in [-1,1]-ish, NCHW (before the uint8 post-process)."""
    if threads:
        torch.set_num_threads(threads)
    cl, scaling, shift, pq = FAMILIES[family]
    assert latents.shape[1] == cl, (latents.shape, cl)
    with torch.no_grad():
        z = torch.from_numpy(latents.astype(np.float32)).to(dtype)
        z = z / scaling + shift
        if pq:
            z = _conv(z, weights, "post_quant_conv", dtype, 0)
        x = _conv(z, weights, "decoder.conv_in", dtype, 1)
        x = _resnet(x, weights, "decoder.mid_block.resnets.0", dtype)
        x = _attention(x, weights, "decoder.mid_block.attentions.0", dtype)
        x = _resnet(x, weights, "decoder.mid_block.resnets.1", dtype)
        nblk = len(BLOCK_OUT)
        for i in range(nblk):
            for j in range(LAYERS_PER_BLOCK + 1):
                x = _resnet(x, weights, f"decoder.up_blocks.{i}.resnets.{j}", dtype)
            if i < nblk - 1:
                x = F.interpolate(x, scale_factor=2.0, mode="nearest")
                x = _conv(x, weights, f"decoder.up_blocks.{i}.upsamplers.0.conv", dtype, 1)
        x = F.silu(_gn(x, weights, "decoder.conv_norm_out", dtype))
        x = _conv(x, weights, "decoder.conv_out", dtype, 1)
    return x


def to_uint8(img: torch.Tensor) -> np.ndarray:
    """(x/2+0.5).clamp(0,1)*255 -> round-half-even -> uint8, NHWC (numpy .round() convention)."""
    y = (img.to(torch.float64) / 2 + 0.5).clamp(0, 1) * 255.0
    y = torch.round(y)  # torch.round is round-half-even
    return y.to(torch.uint8).permute(0, 2, 3, 1).contiguous().numpy()


def decode(latents: np.ndarray, weights: dict, family: str, dtype=torch.float32,
           threads: int | None = None) -> np.ndarray:
    """fp16 NCHW latents -> uint8 RGB NHWC."""
    return to_uint8(decode_float(latents, weights, family, dtype, threads))


def pixel_stats(got: np.ndarray, ref: np.ndarray) -> dict:
    """Per-config agreement statistics: max |diff| (LSB), fraction within +-1 LSB, PSNR (dB)."""
    d = got.astype(np.int32) - ref.astype(np.int32)
    mse = float(np.mean(d.astype(np.float64) ** 2))
    psnr = float("inf") if mse == 0 else 10.0 * math.log10(255.0 ** 2 / mse)
    return {
        "max_abs": int(np.abs(d).max()),
        "frac_exact": float(np.mean(d == 0)),
        "frac_le1": float(np.mean(np.abs(d) <= 1)),
        "psnr_db": psnr,
    }
