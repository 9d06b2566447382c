"""GPU PNG encode (lbx_png_encode_device, csrc/png.cu) against the oracle (oracle/png_ref.py).

Parity bar (lossless format): every PNG decodes -- CRC-32s, zlib stream and Adler-32 checked by the
standard library -- to exactly the input RGB; the per-row filter types equal the oracle's
heuristic; sizes stay within lbx_png_bound.
"""
import numpy as np
import pytest
import torch

import paper_2605_19385_b200 as lbx
from oracle import png_ref as P

pytestmark = pytest.mark.gpu


def gpu_png(imgs):
    n, H, W, _ = imgs.shape
    dev = torch.device("cuda")
    x = torch.from_numpy(np.ascontiguousarray(imgs)).to(dev)
    stride = (lbx.png_bound(H, W) + 15) // 16 * 16
    out = torch.zeros(n * stride, dtype=torch.uint8, device=dev)
    sizes = torch.zeros(n, dtype=torch.int32, device=dev)
    lbx.png_encode_device(x.data_ptr(), n, H, W, out.data_ptr(), stride, sizes.data_ptr(),
                          torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    o, sz = out.cpu().numpy(), sizes.cpu().numpy()
    assert (sz > 0).all() and (sz <= lbx.png_bound(H, W)).all()
    return [o[i * stride:i * stride + int(sz[i])].tobytes() for i in range(n)]


def _images(H, W, seed):
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:H, 0:W]
    smooth = np.stack([(xx * 3 + yy) % 256, (yy * 2) % 256, ((xx + yy) // 3) % 256], -1).astype(np.uint8)
    noise = rng.integers(0, 256, (H, W, 3), dtype=np.uint8)
    const = np.full((H, W, 3), 77, np.uint8)
    mixed = smooth.copy()
    mixed[: H // 2, : W // 2] = noise[: H // 2, : W // 2]
    soft = np.clip(smooth.astype(np.int16) + rng.integers(-2, 3, (H, W, 3)), 0, 255).astype(np.uint8)
    return np.stack([smooth, noise, const, mixed, soft])


def _check(imgs, pngs):
    for i, (img, png) in enumerate(zip(imgs, pngs)):
        rgb, types, info = P.decode_png(png)
        assert rgb.shape == img.shape
        assert np.array_equal(rgb, img), f"image {i}: pixels differ"
        want, _ = P.choose_filters(img)
        assert np.array_equal(types, want), f"image {i}: filter types differ"


@pytest.mark.parametrize("H,W", [(1, 1), (2, 3), (37, 45), (9, 1000), (17, 1024), (64, 64), (130, 77), (3, 8192),
                                 (5, 5000), (700, 4)])
def test_png_shapes(H, W):
    imgs = _images(H, W, seed=H * 1000 + W)
    _check(imgs, gpu_png(imgs))


def test_png_1024_batch_and_ratio():
    imgs = _images(1024, 1024, seed=5)
    pngs = gpu_png(imgs)
    _check(imgs[[0, 2, 4]], [pngs[0], pngs[2], pngs[4]])  # noise/mixed are slow in the pure-Python unfilter
    for k in (1, 3):
        rgb, _, _ = P.decode_png(pngs[k])
        assert np.array_equal(rgb, imgs[k])
    for k, name in enumerate(["smooth", "noise", "const", "mixed", "soft"]):
        ref = len(P.encode_png(imgs[k]))
        print(f"[png {name}] gpu {len(pngs[k])} B, zlib-6 {ref} B, raw {imgs[k].nbytes} B")
    assert len(pngs[1]) < imgs[1].nbytes * 1.01  # incompressible: stored blocks, ~no overhead
    assert len(pngs[2]) < 40000                   # constant: long runs


def test_png_of_decoded_images():
    """The return path proper: decode latents on the GPU, PNG-encode the RGB where it lies."""
    dec = lbx.Decoder("sd15", (64, 64), seed=0, max_batch=2)
    rng = np.random.default_rng(11)
    lat = torch.from_numpy(rng.standard_normal((2, 4, 64, 64), dtype=np.float32).astype(np.float16).view(np.int16)).cuda()
    rgb = torch.empty((2, 512, 512, 3), dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    dec.decode_ptr(lat.data_ptr(), 2, rgb.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    imgs = rgb.cpu().numpy()
    pngs = gpu_png(imgs)
    _check(imgs, pngs)
    for k in range(2):
        print(f"[png decoded {k}] gpu {len(pngs[k])} B, zlib-6 {len(P.encode_png(imgs[k]))} B, raw {imgs[k].nbytes} B")


def test_png_rejects_bad_args():
    with pytest.raises(lbx.LbxError):
        lbx.png_encode_device(0, 1, 4, 4, 0, 1024, 0)
    assert lbx.png_bound(0, 5) == 0 and lbx.png_bound(4, 9000) == 0


def test_reconstruct_png_matches_reconstruct():
    """lbx_reconstruct_png (blobs -> PNG bytes on the host) decodes to exactly lbx_reconstruct's RGB."""
    dec = lbx.Decoder("sd15", (64, 64), seed=0, max_batch=3)
    rng = np.random.default_rng(5)
    lats = rng.standard_normal((3, 4, 64, 64), dtype=np.float32).astype(np.float16)
    blobs = [lbx.pack(lats[i], 1) for i in range(3)]
    rgb = dec.reconstruct(blobs)
    pngs = dec.reconstruct_png(blobs)
    assert len(pngs) == 3
    for i in range(3):
        got, types, _ = P.decode_png(pngs[i])
        assert np.array_equal(got, rgb[i])
    # a too-small cap reports the need and fails cleanly; the decoder stays usable
    with pytest.raises(lbx.LbxError):
        dec.reconstruct_png(blobs, out=np.empty(1000, np.uint8))
    again = dec.reconstruct_png(blobs[:1])
    assert again[0] == pngs[0]
