"""CPU checks of the PNG oracle (oracle/png_ref.py): its encoder round-trips through its decoder,
and the decoder rejects corrupted CRCs / streams (so the GPU tests' acceptance means something)."""
import zlib

import numpy as np
import pytest

from oracle import png_ref as P


@pytest.mark.parametrize("H,W", [(1, 1), (5, 7), (33, 20)])
def test_oracle_round_trip(H, W):
    rng = np.random.default_rng(H * W)
    yy, xx = np.mgrid[0:H, 0:W]
    smooth = np.stack([(xx * 5 + yy) % 256, yy % 256, (xx ^ yy) % 256], -1).astype(np.uint8)
    for img in (smooth, rng.integers(0, 256, (H, W, 3), dtype=np.uint8)):
        png = P.encode_png(img)
        rgb, types, info = P.decode_png(png)
        assert np.array_equal(rgb, img)
        assert np.array_equal(types, P.choose_filters(img)[0])
        assert info["chunks"] == [b"IHDR", b"IDAT", b"IEND"]


def test_oracle_filter_definitions():
    # one row pair by hand: bpp 3, a = left, b = up, c = up-left
    img = np.array([[[10, 20, 30], [12, 25, 29]], [[11, 19, 33], [200, 0, 255]]], np.uint8)
    types, filt = P.choose_filters(img)
    rs = 7
    row1 = np.frombuffer(filt[rs:2 * rs], np.uint8)
    cur = img[1].reshape(-1).astype(int)
    up = img[0].reshape(-1).astype(int)
    a = np.r_[0, 0, 0, cur[:3]]
    c = np.r_[0, 0, 0, up[:3]]
    cands = [cur, cur - a, cur - up, cur - (a + up) // 2]
    p = a + up - c
    pae = np.where((abs(p - a) <= abs(p - up)) & (abs(p - a) <= abs(p - c)), a, np.where(abs(p - up) <= abs(p - c), up, c))
    cands.append(cur - pae)
    cost = [np.abs(np.asarray(x, np.int64).astype(np.uint8).view(np.int8).astype(int)).sum() for x in cands]
    assert types[1] == int(np.argmin(cost))
    assert np.array_equal(row1[1:], np.asarray(cands[types[1]]).astype(np.uint8))


def test_oracle_detects_corruption():
    img = np.arange(4 * 6 * 3, dtype=np.uint8).reshape(4, 6, 3)
    png = bytearray(P.encode_png(img))
    bad = bytearray(png)
    bad[40] ^= 1  # inside IDAT data -> CRC mismatch
    with pytest.raises(ValueError):
        P.decode_png(bytes(bad))
    # a valid CRC over a broken zlib stream (Adler-32 wrong) must fail in zlib
    i = png.index(b"IDAT")
    n = int.from_bytes(png[i - 4:i], "big")
    body = bytearray(png[i + 4:i + 4 + n])
    body[-1] ^= 0xFF
    crc = zlib.crc32(b"IDAT" + bytes(body)).to_bytes(4, "big")
    forged = png[:i + 4] + body + crc + png[i + 4 + n + 4:]
    with pytest.raises((ValueError, zlib.error)):
        P.decode_png(bytes(forged))
