#!/usr/bin/env python
"""A/B the full decode under different lbx_op_set_debug bit settings on the same GPU, interleaved
(A B A B ...) so power/clock drift hits both arms alike.  Not part of the product.

  python scripts/ab_decode.py --bits 1 17 --batch 32 --rounds 4 --steps 2
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_19385_b200 as lbx  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", type=int, nargs="+", default=[1, 17])
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--fam", default="sd15")
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--grep", default="", help="with --profile: print per-kernel rows whose name contains this")
    a = ap.parse_args()
    c = 4 if a.fam == "sd15" else 16
    dev = torch.device("cuda")
    rng = np.random.default_rng(7)
    lat = torch.from_numpy(rng.standard_normal((a.batch, c, 128, 128), dtype=np.float32).astype(np.float16)
                           .view(np.int16)).to(dev)
    rgb = torch.empty((a.batch, 1024, 1024, 3), dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    decs = {}
    for b in a.bits:  # the plan (and its graph) is fixed at first use under the current bits
        lbx.check(lbx.lib().lbx_op_set_debug(b, 0))
        d = lbx.Decoder(a.fam, (128, 128), seed=0, max_batch=a.batch)
        d.decode_ptr(lat.data_ptr(), a.batch, rgb.data_ptr(), stream.cuda_stream)
        torch.cuda.synchronize()
        decs[b] = d
        if a.profile:
            prof = d.profile(a.batch)
            tot = sum(p["ms"] for p in prof)
            print(f"bits {b}: eager profile total {tot:.2f} ms")
            if a.grep:
                agg = {}
                for p in prof:
                    if a.grep in p["name"]:
                        g = agg.setdefault(p["name"], [0.0, 0, 0.0])
                        g[0] += p["ms"]; g[1] += 1; g[2] += p["bytes"]
                for k, (ms, cnt, by) in sorted(agg.items()):
                    print(f"    {ms:8.2f} ms {cnt:3d}x {by / ms / 1e6:7.0f} GB/s  {k}")
    ref = None
    for b, d in decs.items():
        d.decode_ptr(lat.data_ptr(), a.batch, rgb.data_ptr(), stream.cuda_stream)
        torch.cuda.synchronize()
        if ref is None:
            ref = rgb.clone()
        else:
            diff = (rgb.int() - ref.int()).abs().max().item()
            print(f"bits {b}: max |rgb diff| vs bits {a.bits[0]} = {diff}")
    times = {b: [] for b in a.bits}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for r in range(a.rounds):
        for b, d in decs.items():
            e0.record(stream)
            for _ in range(a.steps):
                d.decode_ptr(lat.data_ptr(), a.batch, rgb.data_ptr(), stream.cuda_stream)
            e1.record(stream)
            torch.cuda.synchronize()
            times[b].append(e0.elapsed_time(e1) / a.steps)
    for b in a.bits:
        t = times[b]
        print(f"bits {b}: ms/step median {np.median(t):.2f} min {min(t):.2f}  -> {a.batch / np.median(t) * 1e3:.2f} img/s"
              f"   all {[round(x, 1) for x in t]}")
    lbx.check(lbx.lib().lbx_op_set_debug(1, 0))


if __name__ == "__main__":
    main()
