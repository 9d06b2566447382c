"""paper_2605_19385_b200 -- B200-native decode-on-miss reconstruction for LatentBox.

Thin ctypes binding over the C ABI in include/lbx/reconstruct.h (liblbx.so, built in-tree by
build.py).  The product path is the C++/CUDA library; this module only marshals pointers.  There is
no CPU fallback: if liblbx.so is missing or no sm_100 device is present, calls fail loudly.

Reference interface mirrored: the GPU job of the simulator (proj/src/sim.cpp:409-442), see
include/lbx/reconstruct.h for the mapping.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LBX_LIB") or os.path.join(_HERE, "liblbx.so")  # LBX_LIB: A/B of two builds

FAMILY = {"sd15": 0, "sd3": 1, "flux": 2}
LATENT_CHANNELS = {"sd15": 4, "sd3": 16, "flux": 16}

OK, E_RUNTIME, E_CONFIG, E_CUDA, E_FORMAT = 0, 1, 2, 3, 4
_STATUS = {1: "LBX_E_RUNTIME", 2: "LBX_E_CONFIG", 3: "LBX_E_CUDA", 4: "LBX_E_FORMAT"}

# exported symbols (checked against include/lbx/reconstruct.h by tests/test_abi_cpu.py)
SYMBOLS = [
    "lbx_param_count", "lbx_generate_params", "lbx_decoder_create", "lbx_decoder_destroy", "lbx_unpack", "lbx_decode",
    "lbx_reconstruct", "lbx_reconstruct_latents", "lbx_pack", "lbx_last_error", "lbx_op_gemm",
    "lbx_subpixel_weights", "lbx_op_groupnorm", "lbx_op_gn_stats", "lbx_profile", "lbx_launch_count", "lbx_op_set_debug", "lbx_op_gemm_desc", "lbx_decoder_prepare",
    "lbx_op_conv_out", "lbx_pack_bound", "lbx_pack_device", "lbx_op_attention",
    "lbx_png_bound", "lbx_png_encode_device", "lbx_reconstruct_png", "lbx_op_unpack", "lbx_op_set_grid_limits",
    "lbx_host_alloc", "lbx_host_free", "lbx_reconstruct_v", "lbx_reconstruct_submit", "lbx_reconstruct_wait",
    "lbx_graph_captures", "lbx_decoder_get_counters",
]


class LbxError(RuntimeError):
    """Raised on a non-zero lbx_status; .status holds the code (LBX_E_CONFIG ~ ConfigError)."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class ProfEntry(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 96), ("ms", ctypes.c_double), ("flops", ctypes.c_double),
                ("algo_flops", ctypes.c_double), ("bytes", ctypes.c_double)]


class DecoderCounters(ctypes.Structure):
    _fields_ = [("graph_captures", ctypes.c_uint64), ("peer_copies", ctypes.c_uint64), ("peer_bytes", ctypes.c_uint64),
                ("peer_ms", ctypes.c_double), ("attn_fallbacks", ctypes.c_uint64)]


class GemmDesc(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int), ("M", ctypes.c_int), ("N", ctypes.c_int), ("K", ctypes.c_int),
                ("A", ctypes.c_void_p), ("lda", ctypes.c_int), ("b", ctypes.c_int), ("h", ctypes.c_int),
                ("w", ctypes.c_int), ("c", ctypes.c_int), ("A2", ctypes.c_void_p), ("lda2", ctypes.c_int),
                ("K2", ctypes.c_int), ("B", ctypes.c_void_p), ("ldb", ctypes.c_int), ("out", ctypes.c_void_p),
                ("ldo", ctypes.c_int), ("bias", ctypes.c_void_p), ("resid", ctypes.c_void_p), ("ldr", ctypes.c_int),
                ("row_scale", ctypes.c_void_p), ("alpha", ctypes.c_float), ("gn_stats", ctypes.c_void_p),
                ("cta_group", ctypes.c_int), ("bn", ctypes.c_int), ("gn_ss", ctypes.c_void_p),
                ("b_mn_major", ctypes.c_int)]


class _Desc(ctypes.Structure):
    _fields_ = [
        ("family", ctypes.c_int),
        ("latent_h", ctypes.c_uint32),
        ("latent_w", ctypes.c_uint32),
        ("weight_seed", ctypes.c_uint64),
        ("weights", ctypes.c_void_p),
        ("weights_count", ctypes.c_size_t),
        ("device", ctypes.c_int),
        ("max_batch", ctypes.c_uint32),
        ("precise_activations", ctypes.c_int),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    """Load liblbx.so (building it first when nvcc is available and the .so is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from . import build as _b
        _b.build()
    L = ctypes.CDLL(LIB_PATH)
    vp, u32, i32, sz = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_int, ctypes.c_size_t
    L.lbx_param_count.restype = sz
    L.lbx_param_count.argtypes = [i32]
    L.lbx_last_error.restype = ctypes.c_char_p
    L.lbx_generate_params.argtypes = [i32, ctypes.c_uint64, vp, sz]
    L.lbx_decoder_create.argtypes = [ctypes.POINTER(_Desc), ctypes.POINTER(vp)]
    L.lbx_decoder_destroy.argtypes = [vp]
    L.lbx_decoder_prepare.argtypes = [vp, u32]
    L.lbx_unpack.argtypes = [vp, vp, vp, u32, vp, vp]
    L.lbx_decode.argtypes = [vp, vp, u32, vp, vp]
    L.lbx_reconstruct.argtypes = [vp, vp, vp, u32, vp, vp]
    L.lbx_reconstruct_latents.argtypes = [vp, vp, u32, vp, vp]
    L.lbx_pack.argtypes = [vp, i32, u32, u32, u32, vp, sz, ctypes.POINTER(sz)]
    L.lbx_op_gemm.argtypes = [i32, i32, i32, i32, vp, i32, i32, i32, i32, i32, vp, i32, vp, i32, vp, vp, i32, vp,
                              ctypes.c_float, vp, i32, i32, vp]
    L.lbx_subpixel_weights.argtypes = [vp, i32, i32, vp]
    L.lbx_op_groupnorm.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, i32, ctypes.c_float, vp]
    L.lbx_op_gn_stats.argtypes = [vp, vp, i32, i32, i32, vp]
    L.lbx_profile.argtypes = [vp, u32, ctypes.POINTER(ProfEntry), i32, ctypes.POINTER(i32)]
    L.lbx_launch_count.argtypes = [vp, u32]
    L.lbx_op_set_debug.argtypes = [i32, i32]
    L.lbx_op_gemm_desc.argtypes = [ctypes.POINTER(GemmDesc), vp]
    L.lbx_op_conv_out.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, i32, vp]
    L.lbx_op_attention.argtypes = [vp, vp, i32, i32, vp]
    L.lbx_pack_bound.argtypes = [u32, u32, u32]
    L.lbx_pack_bound.restype = ctypes.c_size_t
    L.lbx_pack_device.argtypes = [vp, u32, u32, u32, u32, vp, ctypes.c_size_t, vp, vp]
    L.lbx_png_bound.argtypes = [u32, u32]
    L.lbx_png_bound.restype = ctypes.c_size_t
    L.lbx_png_encode_device.argtypes = [vp, u32, u32, u32, vp, ctypes.c_size_t, vp, vp]
    L.lbx_reconstruct_png.argtypes = [vp, vp, vp, u32, vp, ctypes.c_size_t, vp, vp]
    L.lbx_op_unpack.argtypes = [vp, vp, vp, u32, u32, u32, u32, vp, vp, vp]
    L.lbx_op_set_grid_limits.argtypes = [i32, i32]
    L.lbx_host_alloc.argtypes = [ctypes.c_size_t]
    L.lbx_host_alloc.restype = vp
    L.lbx_host_free.argtypes = [vp]
    L.lbx_host_free.restype = None
    L.lbx_reconstruct_v.argtypes = [vp, vp, vp, u32, vp, vp]
    L.lbx_reconstruct_submit.argtypes = [vp, vp, vp, u32, vp, ctypes.POINTER(ctypes.c_uint64)]
    L.lbx_reconstruct_wait.argtypes = [vp, ctypes.c_uint64]
    L.lbx_decoder_get_counters.argtypes = [vp, ctypes.POINTER(DecoderCounters)]
    L.lbx_graph_captures.argtypes = [vp]
    L.lbx_graph_captures.restype = ctypes.c_uint64
    for name in SYMBOLS:
        if name not in ("lbx_param_count", "lbx_last_error", "lbx_pack_bound", "lbx_png_bound", "lbx_host_alloc",
                        "lbx_host_free", "lbx_graph_captures"):
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def check(status: int) -> None:
    if status != OK:
        raise LbxError(status, lib().lbx_last_error().decode(errors="replace"))


def param_count(family: str) -> int:
    return int(lib().lbx_param_count(FAMILY[family]))


def generate_params(family: str, seed: int) -> np.ndarray:
    """The fp32 parameters (canonical order) the C++ generator produces for `seed`."""
    n = param_count(family)
    out = np.empty(n, dtype=np.float32)
    check(lib().lbx_generate_params(FAMILY[family], seed, out.ctypes.data, n))
    return out


def pack(latent: np.ndarray, mode: int) -> bytes:
    """Host LBLP packer (write path): one fp16 (C,H,W) latent -> blob."""
    a = np.ascontiguousarray(latent.astype(np.float16)).view(np.uint16)
    c, h, w = a.shape
    n = ctypes.c_size_t(0)
    check(lib().lbx_pack(a.ctypes.data, mode, c, h, w, None, 0, ctypes.byref(n)))
    out = np.empty(n.value, dtype=np.uint8)
    check(lib().lbx_pack(a.ctypes.data, mode, c, h, w, out.ctypes.data, n.value, ctypes.byref(n)))
    return out.tobytes()


class Decoder:
    """One decoder per GPU (single owner; calls serialised by the owning thread)."""

    def __init__(self, family: str = "sd15", latent_hw=(64, 64), seed: int = 0, device: int = 0,
                 max_batch: int = 1, weights: np.ndarray | None = None, precise: bool = False):
        self.family = family
        self.h, self.w = latent_hw
        self.c = LATENT_CHANNELS[family]
        self.max_batch = max_batch
        d = _Desc()
        d.family = FAMILY[family]
        d.latent_h, d.latent_w = self.h, self.w
        d.weight_seed = seed
        d.precise_activations = int(precise)
        self._weights = None
        if weights is not None:
            self._weights = np.ascontiguousarray(weights, dtype=np.float32)
            d.weights = self._weights.ctypes.data
            d.weights_count = self._weights.size
        d.device = device
        d.max_batch = max_batch
        h = ctypes.c_void_p()
        check(lib().lbx_decoder_create(ctypes.byref(d), ctypes.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().lbx_decoder_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def out_hw(self):
        return 8 * self.h, 8 * self.w

    @property
    def rgb_bytes(self):
        """Bytes of one decoded image (8h x 8w x 3 uint8)."""
        return 64 * self.h * self.w * 3

    # -- device-pointer entry points (pointers are ints, e.g. torch.Tensor.data_ptr()) --------
    def decode_ptr(self, latents_dev: int, n: int, rgb_dev: int, stream: int = 0) -> None:
        check(lib().lbx_decode(self._h, latents_dev, n, rgb_dev, stream or None))

    def unpack_ptr(self, blobs, latents_dev: int, stream: int = 0) -> None:
        arr, sizes, keep = _blob_arrays(blobs)
        check(lib().lbx_unpack(self._h, arr, sizes, len(blobs), latents_dev, stream or None))

    def profile(self, n: int):
        """Per-launch device times of one eager decode of n latents: list of dicts."""
        cap = 4096
        arr = (ProfEntry * cap)()
        cnt = ctypes.c_int(0)
        check(lib().lbx_profile(self._h, n, arr, cap, ctypes.byref(cnt)))
        return [{"name": arr[i].name.decode(), "ms": arr[i].ms, "flops": arr[i].flops,
                 "algo_flops": arr[i].algo_flops, "bytes": arr[i].bytes} for i in range(cnt.value)]

    def launch_count(self, n: int) -> int:
        return int(lib().lbx_launch_count(self._h, n))

    def graph_captures(self) -> int:
        """CUDA graphs captured so far (one per batch size)."""
        return int(lib().lbx_graph_captures(self._h))

    def counters(self) -> dict:
        """lbx_decoder_get_counters: graph captures, NVLink peer copies, attention fallbacks."""
        c = DecoderCounters()
        check(lib().lbx_decoder_get_counters(self._h, ctypes.byref(c)))
        return {name: getattr(c, name) for name, _ in DecoderCounters._fields_}

    def prepare(self, n_max: int) -> None:
        check(lib().lbx_decoder_prepare(self._h, n_max))

    # -- asynchronous pipeline (lbx_reconstruct_submit / lbx_reconstruct_wait) ------------------
    def submit(self, blobs, outs) -> int:
        """Enqueue a batch (blobs -> outs[i], each a uint8 array of one image); returns a ticket.
        At most two batches in flight; the buffers are kept alive until wait(ticket)."""
        if len(outs) != len(blobs):
            raise LbxError(E_CONFIG, "outs: one output buffer per blob")
        for o in outs:
            _check_out(o, self.rgb_bytes, "outs[i]")
        arr, sizes, keep = _blob_arrays(blobs)
        optr = (ctypes.c_void_p * len(outs))(*[o.ctypes.data for o in outs])
        t = ctypes.c_uint64(0)
        check(lib().lbx_reconstruct_submit(self._h, arr, sizes, len(blobs), optr, ctypes.byref(t)))
        if not hasattr(self, "_inflight"):
            self._inflight = {}
        self._inflight[t.value] = (keep, outs, optr)
        return t.value

    def wait(self, ticket: int) -> None:
        try:
            check(lib().lbx_reconstruct_wait(self._h, ticket))
        finally:
            getattr(self, "_inflight", {}).pop(ticket, None)

    # -- host entry points ---------------------------------------------------------------------
    def reconstruct(self, blobs, out: np.ndarray | None = None, stream: int = 0) -> np.ndarray:
        """Packed LBLP blobs (host) -> uint8 RGB (n, 8h, 8w, 3).  Synchronous."""
        n = len(blobs)
        if out is None:
            out = np.empty((n, 8 * self.h, 8 * self.w, 3), dtype=np.uint8)
        _check_out(out, n * self.rgb_bytes, "out")
        arr, sizes, keep = _blob_arrays(blobs)
        check(lib().lbx_reconstruct(self._h, arr, sizes, n, out.ctypes.data, stream or None))
        return out

    def reconstruct_png(self, blobs, out: np.ndarray | None = None, stream: int = 0, copy: bool = True) -> list:
        """lbx_reconstruct_png: LBLP blobs -> PNG files, encoded on the GPU.  Returns bytes objects, or
        (copy=False) uint8 views into `out`."""
        n = len(blobs)
        h, w = self.out_hw
        if out is None:
            out = np.empty(n * png_bound(h, w), np.uint8)
        _check_out(out, 1, "out")
        arr, sizes, keep = _blob_arrays(blobs)
        psz = (ctypes.c_size_t * max(n, 1))()
        check(lib().lbx_reconstruct_png(self._h, arr, sizes, n, out.ctypes.data, out.nbytes, psz, stream or None))
        res, off = [], 0
        for i in range(n):
            v = out[off:off + psz[i]]
            res.append(v.tobytes() if copy else v)
            off += psz[i]
        return res

    def reconstruct_latents(self, latents: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        """fp16 NCHW latents (host) -> uint8 RGB (n, 8h, 8w, 3)."""
        lat = np.ascontiguousarray(latents.astype(np.float16))
        if lat.ndim != 4 or lat.shape[1:] != (self.c, self.h, self.w):
            raise LbxError(E_CONFIG, f"latents: shape {lat.shape} != (n, {self.c}, {self.h}, {self.w})")
        n = lat.shape[0]
        if out is None:
            out = np.empty((n, 8 * self.h, 8 * self.w, 3), dtype=np.uint8)
        _check_out(out, n * self.rgb_bytes, "out")
        check(lib().lbx_reconstruct_latents(self._h, lat.ctypes.data, n, out.ctypes.data, None))
        return out


def _check_out(out, min_bytes, name):
    """A host output buffer handed to the C ABI must be uint8, C-contiguous and large enough: the
    library writes min_bytes through its raw pointer (a short or strided buffer would be overrun)."""
    if not isinstance(out, np.ndarray) or out.dtype != np.uint8 or not out.flags.c_contiguous or not out.flags.writeable:
        raise LbxError(E_CONFIG, f"{name}: must be a writeable C-contiguous uint8 numpy array")
    if out.nbytes < min_bytes:
        raise LbxError(E_CONFIG, f"{name}: {out.nbytes} bytes < the {min_bytes} the call writes")


def _blob_arrays(blobs):
    bufs = [np.frombuffer(b, dtype=np.uint8) for b in blobs]
    ptrs = (ctypes.c_void_p * len(bufs))(*[b.ctypes.data for b in bufs])
    sizes = (ctypes.c_size_t * len(bufs))(*[b.size for b in bufs])
    return ptrs, sizes, bufs


def op_gemm(mode, M, N, K, A, lda, B, ldb, out, ldo, *, b=0, h=0, w=0, c=0, bias=0, resid=0, ldr=0, row_scale=0,
            alpha=1.0, gn_stats=0, cta_group=0, bn=0, stream=0, a2=0, lda2=0, k2=0, gn_ss=0, b_mn_major=False):
    """Diagnostic entry to the tcgen05 GEMM/conv kernel (device pointers as ints).  a2/lda2/k2 add
    the extra K segment (lbx_op_gemm_desc)."""
    if k2 or gn_ss or b_mn_major:
        d = GemmDesc(mode, M, N, K, A, lda, b, h, w, c, a2 or None, lda2, k2, B, ldb, out, ldo, bias or None,
                     resid or None, ldr, row_scale or None, alpha, gn_stats or None, cta_group, bn, gn_ss or None,
                     int(b_mn_major))
        check(lib().lbx_op_gemm_desc(ctypes.byref(d), stream or None))
        return
    check(lib().lbx_op_gemm(mode, M, N, K, A, lda, b, h, w, c, B, ldb, out, ldo, bias or None, resid or None, ldr,
                            row_scale or None, ctypes.c_float(alpha), gn_stats or None, cta_group, bn,
                            stream or None))


def subpixel_weights(w3x3: np.ndarray) -> np.ndarray:
    """[N][3][3][C] fp32 conv weight -> [4][N][2][2][C] fp16 sub-pixel kernels."""
    w = np.ascontiguousarray(w3x3, dtype=np.float32)
    n, _, _, c = w.shape
    out = np.empty((4, n, 2, 2, c), dtype=np.uint16)
    check(lib().lbx_subpixel_weights(w.ctypes.data, n, c, out.ctypes.data))
    return out.view(np.float16)


def op_groupnorm(x, y, stats, gamma, beta, b, hw, c, silu=True, eps=1e-6, stream=0):
    check(lib().lbx_op_groupnorm(x, y, stats, gamma, beta, b, hw, c, int(silu), ctypes.c_float(eps), stream or None))


def op_conv_out(x, ss, w, b, rgb, n, h, w_, impl=0, stream=0):
    """Decoder tail (lbx_op_conv_out): impl 0 tensor cores, 2 tensor cores + packed-half SiLU, 1 CUDA cores."""
    check(lib().lbx_op_conv_out(x, ss, w, b, rgb, n, h, w_, impl, stream or None))


def op_attention(qkv, out, n, L, stream=0):
    """Flash-style attention core (lbx_op_attention): out = softmax(Q K^T / sqrt(512)) V."""
    check(lib().lbx_op_attention(qkv, out, n, L, stream or None))


def pack_bound(c: int, h: int, w: int) -> int:
    """Largest LBLP mode-1 blob for one c x h x w latent (stride for pack_device)."""
    return int(lib().lbx_pack_bound(c, h, w))


def pack_device(latents_ptr, n, c, h, w, out_ptr, stride, sizes_ptr, stream=0):
    """Device-side LBLP mode-1 pack (lbx_pack_device): blob i at out + i*stride, size in sizes[i]."""
    check(lib().lbx_pack_device(latents_ptr, n, c, h, w, out_ptr, stride, sizes_ptr, stream or None))


def op_unpack(blobs_ptr, offs_ptr, sizes_ptr, n, c, h, w, out_ptr, err_ptr, stream=0):
    """Device-resident LBLP blobs -> fp16 latents (lbx_op_unpack)."""
    check(lib().lbx_op_unpack(blobs_ptr, offs_ptr, sizes_ptr, n, c, h, w, out_ptr, err_ptr, stream or None))


def png_bound(h: int, w: int) -> int:
    """Largest PNG lbx_png_encode_device writes for one h x w RGB image (its stride)."""
    return int(lib().lbx_png_bound(h, w))


def png_encode_device(rgb_ptr, n, h, w, out_ptr, stride, sizes_ptr, stream=0):
    """GPU PNG encode (lbx_png_encode_device): PNG i at out + i*stride, size in sizes[i]."""
    check(lib().lbx_png_encode_device(rgb_ptr, n, h, w, out_ptr, stride, sizes_ptr, stream or None))


def op_gn_stats(x, stats, b, hw, c, stream=0):
    check(lib().lbx_op_gn_stats(x, stats, b, hw, c, stream or None))


def gn_stats_buffer(b, device="cuda"):
    """A zeroed GroupNorm statistics buffer for b images: int64 [b][32][2 (sum, sumsq)][2 (hi, lo)],
    the exact fixed-point layout the kernels accumulate into (csrc/gnfix.cuh)."""
    import torch
    return torch.zeros(b, 32, 2, 2, dtype=torch.int64, device=device)


def gn_stats_values(stats):
    """float64 [b][32][2] (sum, sumsq) from a gn_stats_buffer: hi * 4 + lo * 2^-30."""
    hi = stats[..., 0].double()
    lo = stats[..., 1].view(-1).cpu().numpy().view("uint64").astype("float64")
    import torch
    return hi * 4.0 + torch.from_numpy(lo).reshape(hi.shape).to(hi.device) * 2.0 ** -30


# ---------------------------------------------------------------------------- batcher (batcher.h)
class Shape(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int), ("latent_h", ctypes.c_uint32), ("latent_w", ctypes.c_uint32)]


class BatcherDesc(ctypes.Structure):
    _fields_ = [("devices", ctypes.POINTER(ctypes.c_int)), ("n_devices", ctypes.c_int),
                ("shapes", ctypes.POINTER(Shape)), ("n_shapes", ctypes.c_int), ("max_batch", ctypes.c_uint32),
                ("max_wait_us", ctypes.c_uint32), ("weight_seed", ctypes.c_uint64), ("policy", ctypes.c_uint32)]


class Completion(ctypes.Structure):
    _fields_ = [("request_id", ctypes.c_uint64), ("status", ctypes.c_int), ("device", ctypes.c_int),
                ("batch_size", ctypes.c_uint32), ("t_submit_us", ctypes.c_uint64), ("t_start_us", ctypes.c_uint64),
                ("t_end_us", ctypes.c_uint64), ("worker", ctypes.c_int)]


class BatcherStats(ctypes.Structure):
    _fields_ = [("spills", ctypes.c_uint64), ("spill_bytes", ctypes.c_uint64), ("peer_copies", ctypes.c_uint64),
                ("peer_ms", ctypes.c_double), ("graph_captures", ctypes.c_uint64)]


def _batcher_lib():
    L = lib()
    if not getattr(L, "_batcher_ready", False):
        vp = ctypes.c_void_p
        L.lbx_batcher_create.argtypes = [ctypes.POINTER(BatcherDesc), ctypes.POINTER(vp)]
        L.lbx_batcher_create.restype = ctypes.c_int
        L.lbx_batcher_destroy.argtypes = [vp]
        L.lbx_batcher_destroy.restype = ctypes.c_int
        L.lbx_batcher_submit.argtypes = [vp, ctypes.c_uint64, ctypes.c_int, vp, ctypes.c_size_t, vp]
        L.lbx_batcher_submit.restype = ctypes.c_int
        L.lbx_batcher_poll.argtypes = [vp, ctypes.POINTER(Completion), ctypes.c_int, ctypes.c_uint32]
        L.lbx_batcher_poll.restype = ctypes.c_int
        L.lbx_batcher_submit_device.argtypes = [vp, ctypes.c_uint64, ctypes.c_int, vp, ctypes.c_size_t, ctypes.c_int,
                                                vp]
        L.lbx_batcher_submit_device.restype = ctypes.c_int
        L.lbx_batcher_get_stats.argtypes = [vp, ctypes.POINTER(BatcherStats)]
        L.lbx_batcher_get_stats.restype = ctypes.c_int
        L.lbx_batcher_pending.argtypes = [vp]
        L.lbx_batcher_pending.restype = ctypes.c_uint64
        L.lbx_now_us.restype = ctypes.c_uint64
        L.lbx_batch_pick.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_uint32, ctypes.c_uint32,
                                     ctypes.c_uint32]
        L.lbx_batch_pick.restype = ctypes.c_uint32
        L._batcher_ready = True
    return L


class Batcher:
    """Multi-GPU request batcher: one worker + decoder per (device, shape class)."""

    def __init__(self, devices, shapes, max_batch=32, max_wait_us=5000, seed=0, policy="greedy"):
        """policy "greedy": batches of up to max_batch; "cost": the size lbx_batch_pick chooses from
        each device's measured service curve."""
        L = _batcher_lib()
        self._devs = (ctypes.c_int * len(devices))(*devices)
        self._shapes = (Shape * len(shapes))(*[Shape(FAMILY[f], h, w) for f, h, w in shapes])
        d = BatcherDesc(self._devs, len(devices), self._shapes, len(shapes), max_batch, max_wait_us, seed,
                        {"greedy": 0, "cost": 1}[policy])
        h = ctypes.c_void_p()
        check(L.lbx_batcher_create(ctypes.byref(d), ctypes.byref(h)))
        self._h = h
        self._rgb_bytes = [64 * sh * sw * 3 for _, sh, sw in shapes]
        self._keep = {}

    def submit(self, request_id: int, shape: int, blob: bytes, out: np.ndarray):
        """Enqueue one request; `out` (uint8, one image) is written by a worker and kept alive here
        until its completion is polled.  A request_id already in flight is rejected (LBX_E_CONFIG)."""
        if not 0 <= shape < len(self._rgb_bytes):
            raise LbxError(E_CONFIG, f"shape: no shape class {shape}")
        _check_out(out, self._rgb_bytes[shape], "out")
        buf = np.frombuffer(blob, dtype=np.uint8)
        check(_batcher_lib().lbx_batcher_submit(self._h, request_id, shape, buf.ctypes.data, buf.size,
                                                out.ctypes.data))
        self._keep[request_id] = out  # after the C side accepted it: a rejected duplicate keeps the original

    def submit_device(self, request_id: int, shape: int, blob_ptr: int, nbytes: int, blob_device: int,
                      out: np.ndarray, keep=None):
        """Enqueue a request whose LBLP blob is resident in GPU memory (blob_ptr on CUDA device
        blob_device, e.g. a torch tensor's data_ptr()); `keep` (e.g. that tensor) is held until the
        completion is polled.  A worker on another GPU fetches it with a peer copy (NVLink spill)."""
        if not 0 <= shape < len(self._rgb_bytes):
            raise LbxError(E_CONFIG, f"shape: no shape class {shape}")
        _check_out(out, self._rgb_bytes[shape], "out")
        check(_batcher_lib().lbx_batcher_submit_device(self._h, request_id, shape, blob_ptr, nbytes, blob_device,
                                                       out.ctypes.data))
        self._keep[request_id] = (out, keep)

    def stats(self) -> dict:
        st = BatcherStats()
        check(_batcher_lib().lbx_batcher_get_stats(self._h, ctypes.byref(st)))
        return {"spills": st.spills, "spill_bytes": st.spill_bytes, "peer_copies": st.peer_copies,
                "peer_ms": st.peer_ms, "graph_captures": st.graph_captures}

    def poll(self, cap=256, wait_us=1000):
        arr = (Completion * cap)()
        n = _batcher_lib().lbx_batcher_poll(self._h, arr, cap, wait_us)
        res = []
        for i in range(n):
            c = arr[i]
            self._keep.pop(c.request_id, None)
            res.append({"id": c.request_id, "status": c.status, "device": c.device, "batch": c.batch_size,
                        "t_submit": c.t_submit_us, "t_start": c.t_start_us, "t_end": c.t_end_us,
                        "worker": c.worker})
        return res

    def pending(self) -> int:
        return int(_batcher_lib().lbx_batcher_pending(self._h))

    def close(self):
        if getattr(self, "_h", None):
            _batcher_lib().lbx_batcher_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def batch_pick(cost_ms, queued: int, max_batch: int) -> int:
    """lbx_batch_pick: batch size to close from `queued` requests given cost_ms[b-1] (None: greedy)."""
    L = _batcher_lib()
    if cost_ms is None:
        return int(L.lbx_batch_pick(None, 0, queued, max_batch))
    arr = (ctypes.c_double * len(cost_ms))(*cost_ms)
    return int(L.lbx_batch_pick(arr, len(cost_ms), queued, max_batch))


def now_us() -> int:
    return int(_batcher_lib().lbx_now_us())
