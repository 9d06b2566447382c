#!/usr/bin/env python
"""Time the full decode (CUDA graph, device-resident latents) of one library build: LBX_LIB=<so>
python scripts/ab_lib.py --batch 32 --steps 6.  scripts/gpu_ab_lib.sh alternates two builds."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_19385_b200 as lbx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--fam", default="sd15")
ap.add_argument("--bits", type=int, default=1)
ap.add_argument("--profile", default="", help="substring: print eager per-kernel times of matching names")
a = ap.parse_args()
lbx.check(lbx.lib().lbx_op_set_debug(a.bits, 0))
c = 4 if a.fam == "sd15" else 16
rng = np.random.default_rng(7)
dev = torch.device("cuda")
lat = torch.from_numpy(rng.standard_normal((a.batch, c, 128, 128), dtype=np.float32).astype(np.float16).view(np.int16)).to(dev)
rgb = torch.empty((a.batch, 1024, 1024, 3), dtype=torch.uint8, device=dev)
s = torch.cuda.Stream()
d = lbx.Decoder(a.fam, (128, 128), seed=0, max_batch=a.batch)
for _ in range(2):
    d.decode_ptr(lat.data_ptr(), a.batch, rgb.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(a.steps):
    d.decode_ptr(lat.data_ptr(), a.batch, rgb.data_ptr(), s.cuda_stream)
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.steps
h = int(rgb[:, ::64, ::64].to(torch.int64).sum().item())
print(f"{os.path.basename(lbx.LIB_PATH)} bits {a.bits}: {ms:.2f} ms/step {a.batch / ms * 1e3:.2f} img/s  rgbsum {h}")
if a.profile:
    agg = {}
    for p in d.profile(a.batch):
        if a.profile in p["name"]:
            g = agg.setdefault(p["name"], [0.0, 0])
            g[0] += p["ms"]; g[1] += 1
    for k, (m, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"   {m:8.2f} ms {n:2d}x  {k}")
