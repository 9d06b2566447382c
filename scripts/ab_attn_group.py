import os, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2605_19385_b200 as lbx
dev = torch.device('cuda')
rng = np.random.default_rng(7)
lat = torch.from_numpy(rng.standard_normal((32, 4, 128, 128), dtype=np.float32).astype(np.float16).view(np.int16)).to(dev)
rgb = torch.empty((32, 1024, 1024, 3), dtype=torch.uint8, device=dev)
s = torch.cuda.Stream(dev); torch.cuda.set_stream(s)
decs = {}
for g in (8, 16, 4):
    os.environ['LBX_ATTN_GROUP'] = str(g)
    d = lbx.Decoder('sd15', (128, 128), seed=0, max_batch=32)
    d.decode_ptr(lat.data_ptr(), 32, rgb.data_ptr(), s.cuda_stream); torch.cuda.synchronize()
    prof = d.profile(32)
    att = sum(p['ms'] for p in prof if p['name'].startswith('attn'))
    print(f'group {g}: eager attention {att:.2f} ms', flush=True)
    decs[g] = d
ref = None
res = {g: [] for g in decs}
for r in range(5):
    for g, d in decs.items():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(3): d.decode_ptr(lat.data_ptr(), 32, rgb.data_ptr(), s.cuda_stream)
        e1.record(s); torch.cuda.synchronize()
        res[g].append(e0.elapsed_time(e1) / 3)
        if ref is None: ref = rgb.clone()
        else: assert torch.equal(ref, rgb), g
for g, v in res.items(): print(f'group {g}: median {np.median(v):.2f} ms/step  {32e3/np.median(v):.2f} img/s', flush=True)
