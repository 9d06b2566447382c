#!/usr/bin/env python
"""Per-kernel eager profile of config 1 (sd15 4x64x64 -> 512^2, batch 1): where batch-1 latency goes."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_19385_b200 as lbx  # noqa: E402

bits = int(sys.argv[1]) if len(sys.argv) > 1 else 1
lbx.check(lbx.lib().lbx_op_set_debug(bits, 0))
d = lbx.Decoder("sd15", (64, 64), seed=0, max_batch=1)
for _ in range(3):
    prof = d.profile(1)
agg = {}
for p in prof:
    g = agg.setdefault(p["name"], [0.0, 0, 0.0])
    g[0] += p["ms"]; g[1] += 1; g[2] += p["algo_flops"]
tot = sum(v[0] for v in agg.values())
print(f"bits {bits}: eager total {tot:.3f} ms, {len(prof)} launches")
for k, (ms, n, fl) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"  {ms:7.3f} ms {100 * ms / tot:5.1f}% {n:3d}x {fl / ms / 1e9 if ms else 0:7.0f} TFLOP/s  {k}")
lat = torch.randn(1, 4, 64, 64, device="cuda").half()
rgb = torch.empty(1, 512, 512, 3, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for _ in range(5):
    d.decode_ptr(lat.data_ptr(), 1, rgb.data_ptr(), s.cuda_stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(50):
    d.decode_ptr(lat.data_ptr(), 1, rgb.data_ptr(), s.cuda_stream)
e1.record(s)
torch.cuda.synchronize()
print(f"graph decode: {e0.elapsed_time(e1) / 50:.3f} ms per 512^2 image")
