#!/usr/bin/env python
"""GPU PNG encode of decoded images: throughput and size vs zlib (not part of the product).

  python scripts/png_bench.py --batch 32 --hw 1024
Decodes `batch` random sd15 latents to RGB on the GPU, then times lbx_png_encode_device on that RGB
(CUDA events, device-resident input), and the CPU encoder (oracle/png_ref.encode_png: same filters
+ zlib level 6) on a few images with all host threads.
"""
import argparse
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_19385_b200 as lbx  # noqa: E402
from oracle import png_ref as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--hw", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--cpu", type=int, default=4, help="images for the CPU encoder sample")
    a = ap.parse_args()
    dev = torch.device("cuda")
    lh = a.hw // 8
    dec = lbx.Decoder("sd15", (lh, lh), seed=0, max_batch=a.batch)
    rng = np.random.default_rng(3)
    lat = torch.from_numpy(rng.standard_normal((a.batch, 4, lh, lh), dtype=np.float32).astype(np.float16)
                           .view(np.int16)).to(dev)
    rgb = torch.empty((a.batch, a.hw, a.hw, 3), dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream()
    dec.decode_ptr(lat.data_ptr(), a.batch, rgb.data_ptr(), s.cuda_stream)
    stride = (lbx.png_bound(a.hw, a.hw) + 15) // 16 * 16
    out = torch.zeros(a.batch * stride, dtype=torch.uint8, device=dev)
    sizes = torch.zeros(a.batch, dtype=torch.int32, device=dev)

    def run():
        lbx.png_encode_device(rgb.data_ptr(), a.batch, a.hw, a.hw, out.data_ptr(), stride, sizes.data_ptr(),
                              s.cuda_stream)

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    sz = sizes.cpu().numpy().astype(np.int64)
    imgs = rgb[: a.cpu].cpu().numpy()
    o = out.cpu().numpy()
    for i in range(a.cpu):  # sanity: decodes exactly
        got, _, _ = P.decode_png(o[i * stride:i * stride + int(sz[i])].tobytes())
        assert np.array_equal(got, imgs[i])
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        cpu_pngs = list(ex.map(P.encode_png, imgs))
    cpu_s = time.perf_counter() - t0
    raw = a.hw * a.hw * 3
    res = {
        "batch": a.batch, "hw": a.hw,
        "gpu_ms_per_batch": round(ms, 3),
        "gpu_img_s": round(a.batch / ms * 1e3, 1),
        "gpu_GBps_rgb_in": round(a.batch * raw / ms / 1e6, 1),
        "gpu_bytes_mean": int(sz.mean()),
        "cpu_bytes_mean_zlib6": int(np.mean([len(p) for p in cpu_pngs])),
        "gpu_bytes_same_imgs": int(sz[: a.cpu].mean()),
        "cpu_img_s": round(a.cpu / cpu_s, 2), "cpu_threads": threads,
        "raw_bytes": raw,
    }
    print(json.dumps(res))


if __name__ == "__main__":
    main()
