#!/usr/bin/env python
"""Two concurrent half-batches on two streams (two decoders, 16 images each) vs one batch of 32 on
one stream: does a second stream fill the persistent kernels' tails (and the GroupNorm applies'
power headroom)?  Not part of the product."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_19385_b200 as lbx  # noqa: E402

dev = torch.device("cuda")
rng = np.random.default_rng(7)
lat = torch.from_numpy(rng.standard_normal((32, 4, 128, 128), dtype=np.float32).astype(np.float16).view(np.int16)).to(dev)
rgb = torch.empty((32, 1024, 1024, 3), dtype=torch.uint8, device=dev)
one = lbx.Decoder("sd15", (128, 128), seed=0, max_batch=32)
halves = [lbx.Decoder("sd15", (128, 128), seed=0, max_batch=16) for _ in range(2)]
s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
half = 16 * 4 * 128 * 128 * 2
hrgb = 16 * 1024 * 1024 * 3


def run_one():
    one.decode_ptr(lat.data_ptr(), 32, rgb.data_ptr(), s0.cuda_stream)


def run_two():
    halves[0].decode_ptr(lat.data_ptr(), 16, rgb.data_ptr(), s0.cuda_stream)
    halves[1].decode_ptr(lat.data_ptr() + half, 16, rgb.data_ptr() + hrgb, s1.cuda_stream)


for f in (run_one, run_two):
    f()
torch.cuda.synchronize()
ref = None
res = {"one": [], "two": []}
for r in range(5):
    for name, f in (("one", run_one), ("two", run_two)):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s0)
        s1.wait_event(e0)
        for _ in range(3):
            f()
        ev = torch.cuda.Event()
        ev.record(s1)
        s0.wait_event(ev)
        e1.record(s0)
        torch.cuda.synchronize()
        res[name].append(e0.elapsed_time(e1) / 3)
        if name == "one":
            ref = rgb.clone()
        else:
            print("max diff two vs one:", (rgb.int() - ref.int()).abs().max().item())
for k, v in res.items():
    v = sorted(v)
    print(f"{k}: median {v[len(v) // 2]:.2f} ms per 32 images  all {[round(x, 1) for x in v]}")
