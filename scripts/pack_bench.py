import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2605_19385_b200 as lbx
n, c, h, w = 64, 16, 128, 128
rng = np.random.default_rng(1)
z = torch.from_numpy(rng.standard_normal((n, c, h, w), dtype=np.float32).astype(np.float16).view(np.int16)).cuda()
stride = (lbx.pack_bound(c, h, w) + 255) // 256 * 256
out = torch.zeros(n * stride, dtype=torch.uint8, device='cuda'); sizes = torch.zeros(n, dtype=torch.int32, device='cuda')
for _ in range(3): lbx.pack_device(z.data_ptr(), n, c, h, w, out.data_ptr(), stride, sizes.data_ptr())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): lbx.pack_device(z.data_ptr(), n, c, h, w, out.data_ptr(), stride, sizes.data_ptr())
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
tot = int(sizes.sum().item())
print(f"pack_device {n} latents 16x128x128: {ms:.3f} ms, {n/ms*1e3:.0f} latents/s, in {n*c*h*w*2/ms/1e6:.0f} GB/s, out {tot/ms/1e6:.0f} GB/s, ratio {n*c*h*w*2/tot:.3f}")
t = time.perf_counter(); zz = z.cpu().numpy().view(np.float16)
for i in range(8): lbx.pack(zz[i], 1)
print(f"host lbx_pack: {(time.perf_counter()-t)/8*1e3:.2f} ms per latent")
