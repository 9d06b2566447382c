"""Pin the decoder oracle (oracle/vae_ref.py) against an independent implementation of the same
network, and commit what it produced as fixtures.

The reference repository has no decoder (decode is the constant proj/src/sim.cpp:414),
so SURVEY.md 8(c) calls decoder parity "unpinned".  This image does ship a third-party
implementation of exactly this decoder: vllm 0.22's `CheersVAEDecoder`
(vllm/model_executor/models/cheers.py), the CompVis/LDM `Decoder` that diffusers' AutoencoderKL
restates -- ch 128, ch_mult (1,2,4,4), 2+1 resnets per level, GroupNorm-32 eps 1e-6, swish, mid
block with one 1x1-conv attention head (SDPA, scale 1/sqrt(512)), nearest-2x upsample + conv3x3,
norm_out -> swish -> conv_out.  With z_channels = 4 it has 49,490,199 parameters, the paper's
49.49 M.  It is written independently of this repo (module names, 1x1 convs
instead of linears, SDPA instead of an explicit softmax), so agreement pins the restatement.

What this script does (CPU, fp32, ~1 min plus ~30 s for importing vllm):
  1. loads the seeded weights (oracle/weights_ref.py) into CheersVAEDecoder by a name map
     (families without post_quant_conv get an exact identity 1x1 conv);
  2. decodes the same pre-scaled latents (z / scaling + shift) with both;
  3. records max |float diff| and uint8 agreement in pin_cheers.json, and saves Cheers' outputs
     (pin_cheers_*.npz) so tests/test_oracle_cpu.py can re-check the oracle against them without
     importing vllm.
Usage: python tests/golden/pin_vllm_cheers.py
"""
import hashlib
import json
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))

import vae_ref  # noqa: E402
import weights_ref  # noqa: E402

CASES = [  # (family, latent h = w, latent seed, weight seed, save float output)
    ("sd15", 64, 1, 0, False),   # config 1 (BASELINE configs[0]); same latents as decode_sd15_64_seed1.npz
    ("sd3", 32, 5, 0, True),     # 16-channel family, small enough to keep the float output
    ("flux", 32, 6, 0, False),
]


def cheers_state(w: dict, family: str) -> dict:
    cl, _, _, pq = weights_ref.FAMILIES[family]
    out = {}

    def put(dst, src, conv1x1=False):
        for s in ("weight", "bias"):
            t = torch.from_numpy(np.ascontiguousarray(w[f"{src}.{s}"]))
            if conv1x1 and s == "weight" and t.dim() == 2:
                t = t[:, :, None, None]
            out[f"{dst}.{s}"] = t

    if pq:
        put("post_quant_conv", "post_quant_conv")
    else:  # exact identity: y = 1.0 * x + 0
        out["post_quant_conv.weight"] = torch.eye(cl)[:, :, None, None].contiguous()
        out["post_quant_conv.bias"] = torch.zeros(cl)
    put("conv_in", "decoder.conv_in")

    def resnet(dst, src):
        for a, b in (("norm1", "norm1"), ("conv1", "conv1"), ("norm2", "norm2"), ("conv2", "conv2")):
            put(f"{dst}.{a}", f"{src}.{b}")
        if f"{src}.conv_shortcut.weight" in w:
            put(f"{dst}.nin_shortcut", f"{src}.conv_shortcut")

    resnet("mid.block_1", "decoder.mid_block.resnets.0")
    resnet("mid.block_2", "decoder.mid_block.resnets.1")
    an = "decoder.mid_block.attentions.0"
    put("mid.attn_1.norm", f"{an}.group_norm")
    for a, b in (("q", "to_q"), ("k", "to_k"), ("v", "to_v"), ("proj_out", "to_out.0")):
        put(f"mid.attn_1.{a}", f"{an}.{b}", conv1x1=True)
    for i in range(4):
        lvl = 3 - i  # diffusers up_blocks[i] == LDM up[3 - i]
        for j in range(3):
            resnet(f"up.{lvl}.block.{j}", f"decoder.up_blocks.{i}.resnets.{j}")
        if i < 3:
            put(f"up.{lvl}.upsample.conv", f"decoder.up_blocks.{i}.upsamplers.0.conv")
    put("norm_out", "decoder.conv_norm_out")
    put("conv_out", "decoder.conv_out")
    return out


def main():
    from vllm.model_executor.models.cheers import CheersVAEDecoder
    import vllm

    torch.set_num_threads(os.cpu_count() or 1)
    report = {"independent_impl": f"vllm {vllm.__version__} vllm/model_executor/models/cheers.py CheersVAEDecoder",
              "cases": []}
    for family, hw, seed, wseed, keep_float in CASES:
        cl, scaling, shift, _ = weights_ref.FAMILIES[family]
        W = weights_ref.make_weights(family, wseed)
        dec = CheersVAEDecoder({"z_channels": cl}).eval()
        missing, unexpected = dec.load_state_dict(cheers_state(W, family), strict=True)
        nparams = sum(p.numel() for p in dec.parameters())
        z = weights_ref.make_latents(family, 1, hw, hw, seed=seed)
        with torch.no_grad():
            zs = torch.from_numpy(z.astype(np.float32)) / scaling + shift
            theirs = dec(zs)
        ours = vae_ref.decode_float(z, W, family)
        fd = float((theirs - ours).abs().max())
        rgb_t = vae_ref.to_uint8(theirs)
        rgb_o = vae_ref.to_uint8(ours)
        d = np.abs(rgb_t.astype(np.int32) - rgb_o.astype(np.int32))
        name = f"pin_cheers_{family}_{hw}_seed{seed}.npz"
        extra = {"float_out": theirs.numpy().astype(np.float32)} if keep_float else {}
        np.savez_compressed(os.path.join(HERE, name), latents=z, rgb=rgb_t, weight_seed=np.int64(wseed),
                            family=np.array(family), **extra)
        case = {"family": family, "latent": [cl, hw, hw], "latent_seed": seed, "weight_seed": wseed,
                "cheers_params": nparams, "oracle_params": weights_ref.param_count(family) + (0 if _pq(family) else cl * cl + cl),
                "max_abs_float_diff": fd, "float_range": [float(theirs.min()), float(theirs.max())],
                "uint8_max_abs_diff": int(d.max()), "uint8_frac_identical": float((d == 0).mean()),
                "fixture": name, "rgb_sha256_16": hashlib.sha256(rgb_t.tobytes()).hexdigest()[:16]}
        print(json.dumps(case))
        report["cases"].append(case)
    with open(os.path.join(HERE, "pin_cheers.json"), "w") as f:
        json.dump(report, f, indent=1)


def _pq(family):
    return weights_ref.FAMILIES[family][3]


if __name__ == "__main__":
    main()
