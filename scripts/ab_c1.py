#!/usr/bin/env python
"""Config-1 (sd15 64x64 -> 512^2, batch 1) graph latency under lbx_op_set_debug bit settings,
interleaved in one process (one decoder per setting; the plan is fixed at first use)."""
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_19385_b200 as lbx  # noqa: E402

bits = [int(b) for b in sys.argv[1:]] or [1]
lat = torch.randn(1, 4, 64, 64, device="cuda").half()
rgb = torch.empty(1, 512, 512, 3, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
decs = {}
for b in bits:
    lbx.check(lbx.lib().lbx_op_set_debug(b, 0))
    d = lbx.Decoder("sd15", (64, 64), seed=0, max_batch=1)
    for _ in range(5):
        d.decode_ptr(lat.data_ptr(), 1, rgb.data_ptr(), s.cuda_stream)
    decs[b] = d
torch.cuda.synchronize()
res = {b: [] for b in bits}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for r in range(6):
    for b, d in decs.items():
        e0.record(s)
        for _ in range(50):
            d.decode_ptr(lat.data_ptr(), 1, rgb.data_ptr(), s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        res[b].append(e0.elapsed_time(e1) / 50)
for b, v in res.items():
    v = sorted(v)
    print(f"bits {b}: config-1 graph decode median {v[len(v) // 2]:.3f} ms  all {[round(x, 3) for x in v]}")
