"""ORACLE (test infrastructure only) -- ctypes wrapper over oracle/_build/liblblp_ref.so.

Only tests/ and __graft_entry__.smoke() use this; see lblp_ref.c for the restated algorithm and
include/lbx/lblp.h for the normative format.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liblblp_ref.so")
_lib = None


def build() -> str:
    src = os.path.join(_HERE, "lblp_ref.c")
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        L.lblp_ref_encoded_size.restype = ctypes.c_long
        L.lblp_ref_encoded_size.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.lblp_ref_encode.restype = ctypes.c_long
        L.lblp_ref_encode.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_void_p, ctypes.c_long]
        L.lblp_ref_decode.restype = ctypes.c_long
        L.lblp_ref_decode.argtypes = [ctypes.c_void_p, ctypes.c_long, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_void_p]
        _lib = L
    return _lib


def encode(latent_f16: np.ndarray, mode: int) -> bytes:
    """One latent (C,H,W) fp16 -> LBLP blob."""
    a = np.ascontiguousarray(latent_f16.astype(np.float16)).view(np.uint16)
    c, h, w = a.shape
    L = lib()
    need = L.lblp_ref_encoded_size(a.ctypes.data, mode, c, h, w)
    if need < 0:
        raise ValueError(f"lblp_ref_encoded_size error {need}")
    out = np.zeros(need, dtype=np.uint8)
    r = L.lblp_ref_encode(a.ctypes.data, mode, c, h, w, out.ctypes.data, need)
    if r != need:
        raise ValueError(f"lblp_ref_encode error {r}")
    return out.tobytes()


def decode(blob: bytes, c: int, h: int, w: int) -> np.ndarray:
    """LBLP blob -> (C,H,W) fp16."""
    buf = np.frombuffer(blob, dtype=np.uint8).copy()
    out = np.zeros((c, h, w), dtype=np.uint16)
    r = lib().lblp_ref_decode(buf.ctypes.data, len(blob), c, h, w, out.ctypes.data)
    if r < 0:
        raise ValueError(f"lblp_ref_decode error {r}")
    return out.view(np.float16)
