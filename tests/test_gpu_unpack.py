"""K1 parity: GPU LBLP unpack (csrc/unpack.cu) bit-exact against the C oracle (oracle/lblp_ref.c),
through the C ABI (lbx_unpack / lbx_reconstruct).  Edge cases: +-0, subnormals, +-inf, NaN payloads,
all-equal rows (width 0), maximum deltas (width 16), malformed blobs."""
import numpy as np
import pytest

import lblp
import weights_ref

pytestmark = pytest.mark.gpu

SPECIAL = np.array([0x0000, 0x8000, 0x0001, 0x8001, 0x03FF, 0x83FF, 0x0400, 0x7BFF, 0xFBFF, 0x7C00, 0xFC00,
                    0x7E00, 0x7C01, 0xFE01, 0x3C00, 0xBC00], dtype=np.uint16)


def _gpu_unpack(lbx, dec, blobs):
    import torch
    n = len(blobs)
    out = torch.zeros((n, dec.c, dec.h, dec.w), dtype=torch.int16, device="cuda")
    dec.unpack_ptr(blobs, out.data_ptr())
    torch.cuda.synchronize()
    return out.cpu().numpy().view(np.uint16)


def _latents_with_specials(seed):
    z = weights_ref.make_latents("sd3", 3, 64, 64, seed=seed).view(np.uint16).copy()
    z[0, 0, 0, :] = np.resize(SPECIAL, 64)                     # special values
    z[0, 1, :, :] = 0x3C00                                     # constant plane -> width-0 mini-blocks
    z[0, 2, 0, :] = np.where(np.arange(64) % 2, 0xFC00, 0x7C00)  # alternating +-inf -> width-16
    z[1, 3, 5, :] = np.random.default_rng(seed).integers(0, 65536, 64, dtype=np.uint16)  # random bit patterns
    return z.view(np.float16)


@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_unpack_bit_exact_vs_oracle(lbx, mode):
    z = _latents_with_specials(21)
    if mode == 2:  # q8 is lossy: specials would blow the per-channel range; use finite data
        z = weights_ref.make_latents("sd3", 3, 64, 64, seed=22)
    dec = lbx.Decoder("sd3", (64, 64), seed=0, max_batch=3)
    blobs = [lblp.encode(z[i], mode) for i in range(3)]
    got = _gpu_unpack(lbx, dec, blobs)
    ref = np.stack([lblp.decode(b, 16, 64, 64).view(np.uint16) for b in blobs])
    assert np.array_equal(got, ref)
    if mode in (0, 1, 3):
        assert np.array_equal(got, z.view(np.uint16))  # lossless round trip


@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_unpack_product_packer_blobs(lbx, mode):
    """Product packer (lbx_pack) -> GPU unpack == oracle decode of the same bytes, at config-3 shape."""
    z = weights_ref.make_latents("sd3", 4, 128, 128, seed=3, smooth=True)
    dec = lbx.Decoder("sd3", (128, 128), seed=0, max_batch=4)
    blobs = [lbx.pack(z[i], mode) for i in range(4)]
    got = _gpu_unpack(lbx, dec, blobs)
    ref = np.stack([lblp.decode(b, 16, 128, 128).view(np.uint16) for b in blobs])
    assert np.array_equal(got, ref)


def test_malformed_blob_rejected(lbx):
    z = weights_ref.make_latents("sd3", 1, 64, 64, seed=1)
    dec = lbx.Decoder("sd3", (64, 64), seed=0, max_batch=1)
    good = lblp.encode(z[0], 1)
    bad = bytearray(good)
    bad[0] = ord("X")
    with pytest.raises(lbx.LbxError) as e:
        dec.reconstruct([bytes(bad)])
    assert e.value.status == lbx.E_FORMAT
    trunc = good[:-8]
    with pytest.raises(lbx.LbxError) as e:
        dec.reconstruct([trunc])
    assert e.value.status == lbx.E_FORMAT
    # the decoder stays usable after a rejected call
    rgb = dec.reconstruct([good])
    assert rgb.shape == (1, 512, 512, 3)


def test_reconstruct_from_blobs_equals_from_latents(lbx):
    z = weights_ref.make_latents("sd3", 2, 64, 64, seed=4)
    dec = lbx.Decoder("sd3", (64, 64), seed=0, max_batch=2)
    a = dec.reconstruct([lbx.pack(z[i], 1) for i in range(2)])
    b = dec.reconstruct_latents(z)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("shape,smooth", [((16, 64, 64), False), ((16, 128, 128), True), ((4, 64, 64), False),
                                          ((4, 32, 96), False)])
def test_device_pack_equals_host_packer(lbx, shape, smooth):
    """lbx_pack_device (GPU write path) produces the same bytes as the host packer (lbx_pack mode 1)
    and as the C oracle's encoder, including special values and width-0 / width-16 mini-blocks;
    the blobs round-trip through the GPU unpack bit-exactly."""
    import torch
    c, h, w = shape
    n = 3
    if (h, w) == (64, 64) and c == 16 and not smooth:
        z = _latents_with_specials(31)
    else:
        fam = "sd3" if c == 16 else "sd15"
        z = weights_ref.make_latents(fam, n, h, w, seed=32, smooth=smooth) if (h == w) else \
            np.random.default_rng(33).standard_normal((n, c, h, w), dtype=np.float32).astype(np.float16)
    zd = torch.from_numpy(np.ascontiguousarray(z).view(np.int16)).cuda()
    stride = (lbx.pack_bound(c, h, w) + 255) // 256 * 256
    out = torch.zeros(n * stride, dtype=torch.uint8, device="cuda")
    sizes = torch.zeros(n, dtype=torch.int32, device="cuda")
    lbx.pack_device(zd.data_ptr(), n, c, h, w, out.data_ptr(), stride, sizes.data_ptr())
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    for i in range(n):
        blob = o[i * stride:i * stride + int(sizes[i].item())].tobytes()
        assert blob == lbx.pack(z[i], 1), i
        assert blob == lblp.encode(z[i], 1), i
    if (c, h, w) == (16, 64, 64):
        dec = lbx.Decoder("sd3", (64, 64), seed=0, max_batch=n)
        blobs = [o[i * stride:i * stride + int(sizes[i].item())].tobytes() for i in range(n)]
        assert np.array_equal(_gpu_unpack(lbx, dec, blobs), np.ascontiguousarray(z).view(np.uint16))


@pytest.mark.parametrize("n,c,h,w", [(3, 4, 256, 256), (2, 3, 40, 96), (2, 2, 7, 32), (2, 1, 3, 1024), (5, 16, 64, 64)])
def test_device_pack_unpack_round_trip_shapes(lbx, n, c, h, w):
    """lbx_pack_device -> lbx_op_unpack on device-resident blobs is the identity for shapes that take
    every kernel path: planes over 16 K values (row kernel), W/32 = 3 (lane-per-row decode), W/32 = 1
    and 32 (segment widths at both ends), plus the decoder's 64x64; the bytes equal the host packer's."""
    import torch
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(n * 1000 + c * 100 + w)
    z = (torch.randn((n, c, h, w), generator=g, device=dev) * 3).half()
    z[0, 0, 0, :8] = torch.tensor([0.0, -0.0, 65504.0, -65504.0, 1e-7, -1e-7, float("inf"), float("-inf")],
                                  dtype=torch.float16)
    stride = (lbx.pack_bound(c, h, w) + 15) // 16 * 16
    blob = torch.zeros(n * stride, dtype=torch.uint8, device=dev)
    sizes = torch.zeros(n, dtype=torch.int32, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    lbx.pack_device(z.data_ptr(), n, c, h, w, blob.data_ptr(), stride, sizes.data_ptr(), s)
    offs = torch.arange(n, dtype=torch.int64, device=dev) * stride
    out = torch.empty_like(z)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    lbx.op_unpack(blob.data_ptr(), offs.data_ptr(), sizes.data_ptr(), n, c, h, w, out.data_ptr(), err.data_ptr(), s)
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    assert torch.equal(out.view(torch.int16), z.view(torch.int16))
    zh = z.cpu().numpy()
    bh, sz = blob.cpu().numpy(), sizes.cpu().numpy()
    for i in range(n):
        assert bh[i * stride:i * stride + sz[i]].tobytes() == lbx.pack(zh[i], 1)


def test_noncanonical_row_order_decodes(lbx):
    """A valid blob whose rows are stored in reverse order (row table rewritten) decodes to the same
    latent: the plane kernel stages only the canonical contiguous layout and must fall back to
    reading such rows from global memory."""
    import struct
    import torch
    rng = np.random.default_rng(9)
    c, h, w = 4, 64, 64
    z = rng.standard_normal((c, h, w)).astype(np.float16)
    blob = bytearray(lbx.pack(z, 1))
    rows = c * h
    table_off, payload = struct.unpack_from("<II", blob, 20)
    offs = list(struct.unpack_from(f"<{rows}I", blob, table_off))
    ends = offs[1:] + [len(blob) - payload]
    pieces = [bytes(blob[payload + offs[r]:payload + ends[r]]) for r in range(rows)]
    new_payload, new_offs, pos = b"", [0] * rows, 0
    for r in reversed(range(rows)):
        new_offs[r] = pos
        new_payload += pieces[r]
        pos += len(pieces[r])
    rev = bytes(blob[:table_off]) + struct.pack(f"<{rows}I", *new_offs) + new_payload
    assert len(rev) == len(blob)
    dec = lbx.Decoder("sd15", (64, 64), seed=0, max_batch=2)
    dev = torch.device("cuda")
    lat = torch.empty((2, c, h, w), dtype=torch.float16, device=dev)
    dec.unpack_ptr([bytes(blob), rev], lat.data_ptr())
    torch.cuda.synchronize()
    got = lat.cpu().numpy()
    assert np.array_equal(got[0].view(np.int16), z.view(np.int16))
    assert np.array_equal(got[1].view(np.int16), z.view(np.int16))


@pytest.mark.parametrize("fam,c,h,w,n", [("sd3", 16, 128, 128, 8), ("sd15", 4, 64, 64, 3)])
def test_entropy_mode_decode_and_reconstruct(lbx, fam, c, h, w, n):
    """LBLP mode 3 (binned rANS, one GPU thread per column) at the decoder shapes: GPU unpack is
    bit-exact with the oracle and with the latents, and lbx_reconstruct from mode-3 blobs equals the
    same decode from mode-1 blobs."""
    z = weights_ref.make_latents(fam, n, h, w, seed=41, smooth=True)
    z[0, 0, 0, :16] = SPECIAL.view(np.float16)
    dec = lbx.Decoder(fam, (h, w), seed=0, max_batch=n)
    blobs = [lbx.pack(z[i], 3) for i in range(n)]
    got = _gpu_unpack(lbx, dec, blobs)
    assert np.array_equal(got, np.stack([lblp.decode(b, c, h, w).view(np.uint16) for b in blobs]))
    assert np.array_equal(got, z.view(np.uint16))
    zf = weights_ref.make_latents(fam, n, h, w, seed=43, smooth=True)  # finite values for the decode
    assert np.array_equal(dec.reconstruct([lbx.pack(zf[i], 3) for i in range(n)]),
                          dec.reconstruct([lbx.pack(zf[i], 1) for i in range(n)]))


def test_entropy_mode_malformed(lbx):
    """Structural damage to a mode-3 blob is LBX_E_FORMAT (host validation), and the device decoder
    flags the same damage on HBM-resident blobs (lbx_op_unpack err word) without faulting."""
    import struct
    import torch
    z = weights_ref.make_latents("sd3", 1, 64, 64, seed=42)
    good = lbx.pack(z[0], 3)
    payload = struct.unpack_from("<I", good, 24)[0]
    plane0 = payload + struct.unpack_from("<I", good, 32)[0]
    bad = bytearray(good)
    struct.pack_into("<H", bad, plane0 + 18, struct.unpack_from("<H", good, plane0 + 18)[0] + 1)  # freq sum != 4096
    dec = lbx.Decoder("sd3", (64, 64), seed=0, max_batch=2)
    with pytest.raises(lbx.LbxError) as e:
        dec.reconstruct([bytes(bad)])
    assert e.value.status == lbx.E_FORMAT
    dev = torch.device("cuda")
    stride = (len(good) + 255) // 256 * 256
    buf = torch.zeros(2 * stride, dtype=torch.uint8)
    buf[:len(good)] = torch.frombuffer(bytearray(good), dtype=torch.uint8)
    buf[stride:stride + len(bad)] = torch.frombuffer(bad, dtype=torch.uint8)
    bd = buf.to(dev)
    offs = torch.tensor([0, stride], dtype=torch.int64, device=dev)
    sizes = torch.tensor([len(good), len(bad)], dtype=torch.int32, device=dev)
    out = torch.empty((2, 16, 64, 64), dtype=torch.float16, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    lbx.op_unpack(bd.data_ptr(), offs.data_ptr(), sizes.data_ptr(), 2, 16, 64, 64, out.data_ptr(), err.data_ptr())
    torch.cuda.synchronize()
    assert int(err.item()) == 4
    assert np.array_equal(out[0].cpu().numpy().view(np.uint16), z[0].view(np.uint16))  # the good blob still decodes
    assert dec.reconstruct([good]).shape == (1, 512, 512, 3)  # and the decoder stays usable
