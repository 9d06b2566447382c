#!/usr/bin/env python
"""One launch of every kernel class of the path, for an ncu capture (scripts/gpu_ncu_all.sh):
an eager decode (lbx_profile) of `--batch` sd15 4x128x128 latents -> 1024^2 (run twice; capture the
second), then the codec (device pack, unpack at 4096 latents) and the GPU PNG encode of 8 images."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_19385_b200 as lbx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--skip-decode", action="store_true")
a = ap.parse_args()
dev = torch.device("cuda")
s = torch.cuda.Stream()
if not a.skip_decode:
    dec = lbx.Decoder("sd15", (128, 128), seed=0, max_batch=a.batch)
    dec.profile(a.batch)
    torch.cuda.synchronize()
    print("launches per decode:", len(dec.profile(a.batch)))
    torch.cuda.synchronize()
    dec.close()
n, c, h, w = 4096, 16, 128, 128
z = torch.randn((n, c, h, w), device=dev).half()
stride = (lbx.pack_bound(c, h, w) + 15) // 16 * 16
blob = torch.empty(n * stride, dtype=torch.uint8, device=dev)
sizes = torch.empty(n, dtype=torch.int32, device=dev)
offs = torch.arange(n, dtype=torch.int64, device=dev) * stride
out = torch.empty_like(z)
err = torch.zeros(1, dtype=torch.int32, device=dev)
lbx.pack_device(z.data_ptr(), n, c, h, w, blob.data_ptr(), stride, sizes.data_ptr(), s.cuda_stream)
lbx.op_unpack(blob.data_ptr(), offs.data_ptr(), sizes.data_ptr(), n, c, h, w, out.data_ptr(), err.data_ptr(),
              s.cuda_stream)
rgb = torch.randint(0, 256, (8, 1024, 1024, 3), dtype=torch.uint8, device=dev)
pst = (lbx.png_bound(1024, 1024) + 15) // 16 * 16
pout = torch.empty(8 * pst, dtype=torch.uint8, device=dev)
psz = torch.empty(8, dtype=torch.int32, device=dev)
lbx.png_encode_device(rgb.data_ptr(), 8, 1024, 1024, pout.data_ptr(), pst, psz.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
print("ok")
