#!/usr/bin/env python
"""K1 (LBLP unpack) at scale: GB/s against the HBM roofline (measured at >= 4096
latents).  Not part of the product.

  python scripts/unpack_bench.py --n 4096
Latents (16x128x128 fp16) are packed on the GPU (lbx_pack_device, mode 1 lossless) into a device
buffer, unpacked with lbx_op_unpack (device-resident blobs), checked bit-exact against the originals,
then timed with CUDA events.  Mode 2 (q8) blobs come from the host packer, replicated.  Algorithmic
bytes = blob bytes read + 2 B per value written.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_19385_b200 as lbx  # noqa: E402


def peak_hbm():
    try:
        d = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
        for k in ("hbm_gbs", "hbm_copy_gbps", "hbm_gbps"):
            if k in d:
                return float(d[k])
        for k, v in d.items():
            if "hbm" in k.lower() and isinstance(v, (int, float)):
                return float(v)
    except Exception:
        pass
    return 6537.0


def latents(kind, n, dev, gen):
    if kind == "noise":
        return torch.randn((n, 16, 128, 128), generator=gen, device=dev).half()
    base = torch.randn((n, 16, 16, 16), generator=gen, device=dev)
    z = F.interpolate(base, size=(128, 128), mode="bilinear", align_corners=False)
    return (z + 0.05 * torch.randn(z.shape, generator=gen, device=dev)).half()


def time_unpack(blob, offs, sizes, n, out, err, reps, s):
    for _ in range(2):
        lbx.op_unpack(blob.data_ptr(), offs.data_ptr(), sizes.data_ptr(), n, 16, 128, 128, out.data_ptr(),
                      err.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        lbx.op_unpack(blob.data_ptr(), offs.data_ptr(), sizes.data_ptr(), n, 16, 128, 128, out.data_ptr(),
                      err.data_ptr(), s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--bits", type=int, default=1, help="lbx_op_set_debug bits (16777217: row kernel)")
    a = ap.parse_args()
    lbx.check(lbx.lib().lbx_op_set_debug(a.bits, 0))
    dev = torch.device("cuda")
    s = torch.cuda.current_stream()
    gen = torch.Generator(device=dev).manual_seed(3)
    n = a.n
    vals = 16 * 128 * 128
    stride = (lbx.pack_bound(16, 128, 128) + 15) // 16 * 16
    out = torch.empty((n, 16, 128, 128), dtype=torch.float16, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    res = {"n": n, "latent": [16, 128, 128], "peak_hbm_gbps": peak_hbm()}
    for kind in ("noise", "smooth"):
        z = latents(kind, n, dev, gen)
        blob = torch.empty(n * stride, dtype=torch.uint8, device=dev)
        sizes = torch.empty(n, dtype=torch.int32, device=dev)
        lbx.pack_device(z.data_ptr(), n, 16, 128, 128, blob.data_ptr(), stride, sizes.data_ptr(), s.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(3):
            lbx.pack_device(z.data_ptr(), n, 16, 128, 128, blob.data_ptr(), stride, sizes.data_ptr(), s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        pack_ms = e0.elapsed_time(e1) / 3
        offs = torch.arange(n, dtype=torch.int64, device=dev) * stride
        ms = time_unpack(blob, offs, sizes, n, out, err, a.reps, s)
        assert int(err.item()) == 0
        assert torch.equal(out.view(torch.int16), z.view(torch.int16)), f"{kind}: unpack is not bit-exact"
        blob_bytes = int(sizes.sum().item())
        algo = blob_bytes + 2 * vals * n
        res[f"mode1_{kind}"] = {"ms": round(ms, 3), "ratio": round(blob_bytes / (2 * vals * n), 3),
                                "algo_bytes": algo, "GBps": round(algo / ms / 1e6, 1),
                                "frac_of_hbm": round(algo / ms / 1e6 / res["peak_hbm_gbps"], 3),
                                "pack_ms": round(pack_ms, 3), "pack_GBps": round(algo / pack_ms / 1e6, 1)}
        del blob
    # mode 2 (q8 + per-channel affine): host packer, one blob per 64 latents replicated
    zq = latents("smooth", 64, dev, gen).cpu().numpy()
    q8 = [lbx.pack(zq[i], 2) for i in range(64)]
    qstride = (max(len(b) for b in q8) + 15) // 16 * 16
    host = np.zeros(n * qstride, np.uint8)
    qs = np.zeros(n, np.int32)
    for i in range(n):
        b = q8[i % 64]
        host[i * qstride:i * qstride + len(b)] = np.frombuffer(b, np.uint8)
        qs[i] = len(b)
    blob = torch.from_numpy(host).to(dev)
    sizes = torch.from_numpy(qs).to(dev)
    offs = torch.arange(n, dtype=torch.int64, device=dev) * qstride
    ms = time_unpack(blob, offs, sizes, n, out, err, a.reps, s)
    assert int(err.item()) == 0
    algo = int(qs.sum()) + 2 * vals * n
    res["mode2_q8"] = {"ms": round(ms, 3), "ratio": round(int(qs.sum()) / (2 * vals * n), 3), "algo_bytes": algo,
                       "GBps": round(algo / ms / 1e6, 1), "frac_of_hbm": round(algo / ms / 1e6 / res["peak_hbm_gbps"], 3)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
