#!/usr/bin/env python
"""Per-kernel eager profile at batch 1 (config 1: sd15 64x64 -> 512^2; the batcher's sd3 128x128 ->
1024^2 service unit): where batch-1 latency goes, with each GEMM's tile count vs the grid."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_19385_b200 as lbx  # noqa: E402

bits = int(sys.argv[1]) if len(sys.argv) > 1 else 1
lbx.check(lbx.lib().lbx_op_set_debug(bits, 0))
for fam, hw in (("sd15", 64), ("sd3", 128)):
    d = lbx.Decoder(fam, (hw, hw), seed=0, max_batch=1)
    profs = [d.profile(1) for _ in range(5)]
    prof = [dict(p, ms=sorted(q[i]["ms"] for q in profs)[2]) for i, p in enumerate(profs[0])]
    agg = {}
    for p in prof:
        g = agg.setdefault(p["name"], [0.0, 0, 0.0])
        g[0] += p["ms"]; g[1] += 1; g[2] += p["algo_flops"]
    tot = sum(v[0] for v in agg.values())
    print(f"{fam} {hw}x{hw} batch 1, bits {bits}: eager total {tot:.3f} ms, {len(prof)} launches")
    for k, (ms, n, fl) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"  {ms:7.3f} ms {100 * ms / tot:5.1f}% {n:3d}x {fl / ms / 1e9 if ms else 0:7.0f} TFLOP/s  {k}")
    c = 4 if fam == "sd15" else 16
    lat = torch.randn(1, c, hw, hw, device="cuda").half()
    rgb = torch.empty(1, 8 * hw, 8 * hw, 3, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    for _ in range(5):
        d.decode_ptr(lat.data_ptr(), 1, rgb.data_ptr(), s.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(30):
        d.decode_ptr(lat.data_ptr(), 1, rgb.data_ptr(), s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    print(f"graph decode: {e0.elapsed_time(e1) / 30:.3f} ms per image")
