"""CPU restatement of the return-path PNG encode -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench/baseline scripts may import this module, and only as
the checker or the CPU baseline; the product path is csrc/png.cu behind lbx_png_encode_device.

The reference has no image encoder: the paper PNG-encodes decoded images in a CPU compute pool
 and ships PNGs.  What is pinned here is the format, through the
Python standard library's zlib (the DEFLATE/zlib decoder every PNG reader uses):
  * decode_png    parses chunks, checks every CRC-32 (zlib.crc32), inflates the concatenated IDAT
                  data (zlib.decompress also checks the Adler-32), undoes the row filters;
  * choose_filters the per-row filter heuristic the GPU encoder uses (libpng's: the filter whose
                  residual bytes, read as int8, have the smallest sum of absolute values; ties go
                  to the lower filter type);
  * encode_png    a CPU encoder (same filters + zlib.compress) -- the CPU baseline's work.
PNG 1.2 filter definitions (section 6): bpp = 3, a = left, b = up, c = up-left, 0 outside.
"""
import struct
import zlib

import numpy as np

_SIG = b"\x89PNG\r\n\x1a\n"


def _paeth(a, b, c):
    p = a + b - c
    pa, pb, pc = np.abs(p - a), np.abs(p - b), np.abs(p - c)
    return np.where((pa <= pb) & (pa <= pc), a, np.where(pb <= pc, b, c))


def _candidates(cur, up):
    """The five filtered versions (uint8) of one row `cur` given the row above `up` (int arrays)."""
    a = np.concatenate([np.zeros(3, np.int32), cur[:-3]])
    c = np.concatenate([np.zeros(3, np.int32), up[:-3]])
    b = up
    return np.stack([cur, cur - a, cur - b, cur - ((a + b) >> 1), cur - _paeth(a, b, c)]).astype(np.uint8)


def choose_filters(rgb):
    """rgb uint8 [H][W][3] -> (filter types [H] uint8, filtered stream bytes H*(3W+1))."""
    H, W, _ = rgb.shape
    rows = rgb.reshape(H, 3 * W).astype(np.int32)
    types = np.zeros(H, np.uint8)
    out = bytearray()
    up = np.zeros(3 * W, np.int32)
    for y in range(H):
        cand = _candidates(rows[y], up)
        cost = np.abs(cand.view(np.int8).astype(np.int32)).sum(axis=1)
        k = int(np.argmin(cost))  # first minimum = lowest type on ties
        types[y] = k
        out.append(k)
        out += cand[k].tobytes()
        up = rows[y]
    return types, bytes(out)


def _chunk(kind, data):
    return struct.pack(">I", len(data)) + kind + data + struct.pack(">I", zlib.crc32(kind + data) & 0xFFFFFFFF)


def encode_png(rgb, level=6):
    """CPU PNG encoder: the same per-row filters, zlib at `level`, one IDAT."""
    H, W, _ = rgb.shape
    _, filt = choose_filters(rgb)
    ihdr = struct.pack(">IIBBBBB", W, H, 8, 2, 0, 0, 0)
    return _SIG + _chunk(b"IHDR", ihdr) + _chunk(b"IDAT", zlib.compress(filt, level)) + _chunk(b"IEND", b"")


def _unfilter(raw, H, W):
    rs = 3 * W + 1
    if len(raw) != H * rs:
        raise ValueError(f"inflated {len(raw)} bytes, expected {H * rs}")
    out = np.zeros((H, 3 * W), np.uint8)
    types = np.zeros(H, np.uint8)
    up = np.zeros(3 * W, np.int32)
    for y in range(H):
        t = raw[y * rs]
        f = np.frombuffer(raw, np.uint8, 3 * W, y * rs + 1).astype(np.int32)
        types[y] = t
        if t == 0:
            cur = f
        elif t == 1:  # Sub: a running sum per channel
            cur = (np.cumsum(f.reshape(W, 3), axis=0) & 255).reshape(-1)
        elif t == 2:
            cur = (f + up) & 255
        elif t in (3, 4):  # Average / Paeth: sequential over the row
            fl, ul, cl = f.tolist(), up.tolist(), [0] * (3 * W)
            for i in range(3 * W):
                a = cl[i - 3] if i >= 3 else 0
                b = ul[i]
                if t == 3:
                    pred = (a + b) >> 1
                else:
                    c = ul[i - 3] if i >= 3 else 0
                    p = a + b - c
                    pa, pb, pc = abs(p - a), abs(p - b), abs(p - c)
                    pred = a if (pa <= pb and pa <= pc) else (b if pb <= pc else c)
                cl[i] = (fl[i] + pred) & 255
            cur = np.array(cl, np.int32)
        else:
            raise ValueError(f"row {y}: filter type {t}")
        out[y] = cur
        up = cur
    return out.reshape(H, W, 3), types


def decode_png(data):
    """PNG bytes -> (rgb [H][W][3] uint8, filter types [H], info dict).  Raises on any CRC, zlib,
    Adler-32 or structure error."""
    if data[:8] != _SIG:
        raise ValueError("bad signature")
    pos, idat, ihdr, chunks = 8, [], None, []
    while pos < len(data):
        (n,) = struct.unpack(">I", data[pos:pos + 4])
        kind = data[pos + 4:pos + 8]
        body = data[pos + 8:pos + 8 + n]
        (crc,) = struct.unpack(">I", data[pos + 8 + n:pos + 12 + n])
        if zlib.crc32(kind + body) & 0xFFFFFFFF != crc:
            raise ValueError(f"CRC mismatch in {kind!r} at {pos}")
        chunks.append(kind)
        if kind == b"IHDR":
            ihdr = struct.unpack(">IIBBBBB", body)
        elif kind == b"IDAT":
            idat.append(body)
        elif kind == b"IEND":
            pos += 12 + n
            break
        pos += 12 + n
    if pos != len(data):
        raise ValueError("trailing bytes after IEND")
    W, H, depth, ctype, comp, filt, inter = ihdr
    if (depth, ctype, comp, filt, inter) != (8, 2, 0, 0, 0):
        raise ValueError(f"unsupported IHDR {ihdr}")
    d = zlib.decompressobj()
    raw = d.decompress(b"".join(idat)) + d.flush()
    if not d.eof or d.unused_data:
        raise ValueError("zlib stream not terminated cleanly")
    rgb, types = _unfilter(raw, H, W)
    return rgb, types, {"chunks": chunks, "idat": len(idat), "bytes": len(data)}
