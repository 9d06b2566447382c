#!/usr/bin/env python
"""Time the flash-style attention core (lbx_op_attention) at the decoder's mid-block shape."""
import sys
import torch
sys.path.insert(0, '.')
import paper_2605_19385_b200 as lbx
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
L = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
qkv = (torch.randn(n, L, 1536, device='cuda') * 0.8).half()
out = torch.empty(n, L, 512, dtype=torch.half, device='cuda')
for _ in range(2):
    lbx.op_attention(qkv.data_ptr(), out.data_ptr(), n, L)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    lbx.op_attention(qkv.data_ptr(), out.data_ptr(), n, L)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
fl = n * 4.0 * L * L * 512
print(f"flash attention n{n} L{L}: {ms:.3f} ms  {fl / ms / 1e9:.0f} TFLOP/s")
