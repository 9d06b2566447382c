// K1: LBLP v1 latent unpack on the GPU (format: include/lbx/lblp.h).  Two kernels:
//   lblp_unpack_plane_kernel (default; planes of <= 16 K values, W % 32 == 0): one CTA per
//     (latent, channel) plane.  A producer warp validates each plane's header once and stages its
//     rows into a 2-slot shared-memory ring with a 1-D TMA copy (full / empty mbarriers); the
//     decode warps give each row W/32 lanes, one 32-value mini-block per lane (funnel-shift bit
//     reader, register prefix sum, one segmented shuffle scan for the carries), and write 16-byte
//     vectors.  q8 / raw planes stream through with 16-byte vectors.
//   lblp_unpack_kernel (fallback for larger planes; debug bit 24): one warp per latent row, lane k
//     owns value k of every mini-block, warp-wide scans rebuild the values.
// Bit-exact by construction; checked against the C oracle (oracle/lblp_ref.c) in
// tests/test_gpu_unpack.py.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "gemm_tc.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace lbx {

static bool g_unpack_rows = false;  // row kernel instead of the plane kernel (diagnostics)
void kernels_set_unpack_rows(bool on) { g_unpack_rows = on; }

__device__ __forceinline__ uint32_t ld_u32(const uint8_t* p) { return *reinterpret_cast<const uint32_t*>(p); }
__device__ __forceinline__ uint16_t ld_u16(const uint8_t* p) { return *reinterpret_cast<const uint16_t*>(p); }
__device__ __forceinline__ uint16_t omap_inv(uint16_t v) {
  return (v & 0x8000u) ? (uint16_t)(v & 0x7FFFu) : (uint16_t)(~v);
}
__device__ __forceinline__ uint16_t omap(uint16_t u) {
  return (u & 0x8000u) ? (uint16_t)(~u) : (uint16_t)(u | 0x8000u);
}

__global__ void __launch_bounds__(256) lblp_unpack_kernel(const uint8_t* __restrict__ blobs,
                                                          const unsigned long long* __restrict__ offs,
                                                          const unsigned int* __restrict__ sizes, int n, int C, int H,
                                                          int W, __half* __restrict__ out, int* err) {
  const int lane = threadIdx.x & 31;
  const long long rows_per = (long long)C * H;
  const long long total_rows = rows_per * n;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  uint16_t* o16 = reinterpret_cast<uint16_t*>(out);
  for (long long gr = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); gr < total_rows; gr += warps) {
    const int bi = (int)(gr / rows_per);
    const uint32_t r = (uint32_t)(gr - (long long)bi * rows_per);
    const uint8_t* base = blobs + offs[bi];
    const uint32_t nbytes = sizes[bi];
    uint16_t* dst = o16 + (size_t)gr * W;
    int code = 0;
    if (nbytes < 32 || base[0] != 'L' || base[1] != 'B' || base[2] != 'L' || base[3] != 'P' || base[4] != 1 ||
        base[5] != 1)
      code = 2;
    else if (ld_u16(base + 8) != C || ld_u16(base + 10) != H || ld_u16(base + 12) != W)
      code = 3;
    else if (ld_u32(base + 16) != nbytes)
      code = 4;
    const int mode = code ? -1 : base[6];
    const uint32_t table = code ? 0 : ld_u32(base + 20), payload = code ? 0 : ld_u32(base + 24);
    if (!code) {
      if (mode == 0) {
        if (payload != 32 || 32ull + 2ull * rows_per * W > nbytes) code = 4;
        else
          for (int k = lane; k < W; k += 32) dst[k] = ld_u16(base + payload + 2ull * ((size_t)r * W + k));
      } else if (mode == 2) {
        if (table != 32 || payload != 32u + 8u * (uint32_t)C || (unsigned long long)payload + rows_per * W > nbytes)
          code = 4;
        else {
          const uint32_t c = r / H;
          const float scale = __uint_as_float(ld_u32(base + 32 + 4 * c));
          const int zp = (int)ld_u32(base + 32 + 4 * C + 4 * c);
          const int8_t* q = reinterpret_cast<const int8_t*>(base + payload) + (size_t)r * W;
          for (int k = lane; k < W; k += 32) {
            const float f = __fmul_rn((float)((int)q[k] - zp), scale);
            dst[k] = __half_as_ushort(__float2half_rn(f));
          }
        }
      } else if (mode == 1) {
        const uint32_t head = (2u + (uint32_t)(W / 32) + 3u) & ~3u;
        if ((W & 31) || table != 32 || payload != 32u + 4u * (uint32_t)rows_per || payload > nbytes) code = 4;
        else {
          const uint32_t roff = ld_u32(base + 32 + 4 * r);
          if ((unsigned long long)payload + roff + head > nbytes || (roff & 3)) code = 4;
          else {
            const uint8_t* row = base + payload + roff;
            uint16_t carry = omap(ld_u16(row));
            uint32_t wpos = head;
            for (int j = 0; j < W / 32; ++j) {
              const uint32_t bw = row[2 + j];
              if (bw > 16 || (unsigned long long)payload + roff + wpos + 4ull * bw > nbytes) { code = 4; break; }
              uint32_t z = 0;
              if (bw) {
                const uint32_t bit = (uint32_t)lane * bw;
                const uint8_t* wp = row + wpos + 4 * (bit >> 5);
                uint32_t lo = ld_u32(wp) >> (bit & 31);
                if ((bit & 31) + bw > 32) lo |= ld_u32(wp + 4) << (32 - (bit & 31));
                z = lo & ((1u << bw) - 1u);
              }
              uint32_t d = (j == 0 && lane == 0) ? 0u : (uint32_t)(uint16_t)((z >> 1) ^ (uint32_t)(-(int)(z & 1)));
              // inclusive scan mod 2^16 (carry kept in 32 bits, truncated at the end)
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, d, o);
                if (lane >= o) d += t;
              }
              const uint16_t v = (uint16_t)(carry + d);
              dst[32 * j + lane] = omap_inv(v);
              carry = (uint16_t)__shfl_sync(0xffffffffu, v, 31);
              wpos += 4u * bw;
            }
          }
        }
      } else {
        code = 5;
      }
    }
    if (code) {
      for (int k = lane; k < W; k += 32) dst[k] = 0;
      if (lane == 0) atomicExch(err, code);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Plane kernel (the default for planes of <= kPlaneMaxVals values): see the file comment.  A row
// whose table offset lies outside the staged canonical range (a valid but non-canonical layout)
// is decoded from global memory.  Bit-exact with the row kernel above; same error codes.
constexpr int kPlaneMaxVals = 16384;           // 128 x 128
constexpr int kPlaneInBytes = 34 * 1024 + 64;  // mode-1 plane at 128 x 128: <= 128 x 264 B
constexpr int kPlaneThreads = 256;  // decode threads (W/32 per mode-1 row) + one producer warp

// decode one mode-1 row (W values) on ONE lane (used when W/32 is not a power of two): the prefix
// sum runs sequentially in registers over a 64-bit bit reader (no warp shuffles); 8 values per
// 16-byte store to `dst` (global, 16-byte aligned).  Bounds as in the row kernel; on an error the
// caller zeroes the row.
__device__ __forceinline__ int decode_row_lane(const uint8_t* row, uint32_t avail, int W, uint16_t* dst) {
  const uint32_t head = (2u + (uint32_t)(W / 32) + 3u) & ~3u;
  if (avail < head) return 4;
  uint32_t prev = omap(*reinterpret_cast<const uint16_t*>(row));
  uint32_t wpos = head;
  uint4* d16 = reinterpret_cast<uint4*>(dst);
  for (int j = 0; j < W / 32; ++j) {
    const uint32_t bw = row[2 + j];
    if (bw > 16 || wpos + 4ull * bw > avail) return 4;
    const uint32_t* wp = reinterpret_cast<const uint32_t*>(row + wpos);
    const uint32_t mask = (1u << bw) - 1u;
    uint64_t buf = 0;
    uint32_t nb = 0, wi = 0;
    uint32_t pk[16];
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (nb < bw) {
        buf |= (uint64_t)wp[wi++] << nb;
        nb += 32;
      }
      const uint32_t z = (uint32_t)buf & mask;
      buf >>= bw;
      nb -= bw;
      const uint32_t d = (j == 0 && k == 0) ? 0u : (uint32_t)(uint16_t)((z >> 1) ^ (uint32_t)(-(int)(z & 1)));
      prev = (prev + d) & 0xFFFFu;
      const uint32_t h = omap_inv((uint16_t)prev);
      if (k & 1) pk[k >> 1] |= h << 16; else pk[k >> 1] = h;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) d16[4 * j + q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
    wpos += 4u * bw;
  }
  return 0;
}

// decode one mode-1 row on L = W/32 lanes (a power of two <= 32): lane j of the row's segment
// takes mini-block j -- widths prefix, bit extraction and a register prefix sum of its 32 deltas --
// then a segmented shuffle scan across the L lanes supplies each block's carry-in.  Every lane of
// the warp must call it (inactive rows pass active = false).  Returns the row's error code
// (uniform over the segment); on an error nothing is stored.
__device__ __forceinline__ int decode_row_split(const uint8_t* row, uint32_t avail, int L, int lane, bool active,
                                                uint16_t* dst) {
  const int j = lane & (L - 1);
  const uint32_t head = (2u + (uint32_t)L + 3u) & ~3u;
  const bool hok = active && avail >= head;
  const uint32_t bits0 = hok ? *reinterpret_cast<const uint16_t*>(row) : 0u;
  const uint32_t bw = hok ? row[2 + j] : 0u;
  uint32_t incl = bw;
  for (int o = 1; o < L; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o, L);
    if (j >= o) incl += u;
  }
  const uint32_t wpos = head + 4u * (incl - bw);
  const bool bad = active && (!hok || bw > 16 || wpos + 4ull * bw > avail);
  const uint32_t seg = (uint32_t)(lane & ~(L - 1));
  const uint32_t gmask = (L == 32 ? 0xffffffffu : ((1u << L) - 1u)) << seg;
  const bool seg_bad = (__ballot_sync(0xffffffffu, bad) & gmask) != 0;
  uint32_t sv[16];  // running sums mod 2^16, two per register
  uint32_t acc = 0;
  if (active && !seg_bad) {
    const uint32_t* wp = reinterpret_cast<const uint32_t*>(row + wpos);
    const uint32_t mask = (1u << bw) - 1u;
    // two-word window (nxt:cur) and a bit position < 32: one funnel shift per value
    uint32_t cur = bw ? wp[0] : 0u, nxt = bw > 1 ? wp[1] : 0u, pos = 0, wi = 2;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const uint32_t z = __funnelshift_r(cur, nxt, pos) & mask;
      pos += bw;
      if (pos >= 32) {
        pos -= 32;
        cur = nxt;
        nxt = wi < bw ? wp[wi] : 0u;
        ++wi;
      }
      const uint32_t d = (j == 0 && k == 0) ? 0u : ((z >> 1) ^ (uint32_t)(-(int)(z & 1)));
      acc += d;
      if (k & 1) sv[k >> 1] |= (acc & 0xFFFFu) << 16; else sv[k >> 1] = acc & 0xFFFFu;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 16; ++k) sv[k] = 0;
  }
  // carry-in of block j: omap(bits0) + the totals of blocks 0..j-1 (mod 2^16)
  uint32_t tin = acc;
  for (int o = 1; o < L; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, tin, o, L);
    if (j >= o) tin += u;
  }
  if (!active || seg_bad) return seg_bad ? 4 : 0;
  const uint32_t off = ((uint32_t)omap((uint16_t)bits0) + tin - acc) & 0xFFFFu;
  const uint32_t off2 = off | off << 16, off2lo = off2 & 0x7FFF7FFFu;
  uint32_t pk[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {  // both halves at once: add mod 2^16 per half, then the inverse order map
    const uint32_t v = ((sv[k] & 0x7FFF7FFFu) + off2lo) ^ ((sv[k] ^ off2) & 0x80008000u);
    const uint32_t neg = ((v & 0x80008000u) >> 15) * 0x7FFFu;  // 0x7FFF in each half whose bit 15 is set
    pk[k] = ~(v ^ neg);  // bit 15 set: v ^ 0x8000 (= v & 0x7FFF); clear: ~v
  }
  uint4* d16 = reinterpret_cast<uint4*>(dst + 32 * j);
#pragma unroll
  for (int q = 0; q < 4; ++q) d16[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
  return 0;
}

__device__ __forceinline__ void ubulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   ptx::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(ptx::smem_u32(bar))
               : "memory");
}

// ---------------------------------------------------------------- mode 3 (binned rANS, lblp.h)
// One plane per CTA: the decode warps build the slot -> bin table in shared memory (in the plane's
// unused staging buffer), then thread t decodes columns t, t + 256, ...: per row one rANS step
// (the warp's renormalisation words are consumed in lane order: ballot + popc), the raw low bits
// from the column's own bit stream, the inverse delta down the column; row y's values of a warp are
// 32 consecutive halves (coalesced stores).
constexpr uint32_t kEntL = 12, kEntM = 1u << kEntL;
__device__ __forceinline__ void ent_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kPlaneThreads) : "memory"); }

// Returns 0 or an error code (4) -- uniform over the decode threads; on an error the caller zeroes
// the plane.  pl / plen: the plane's bytes (global); smem: >= 4096 + 256 * 8 bytes.  s_bad: the
// slot's error flag (per ring slot, so a fast thread resetting it for its next plane cannot race a
// slow thread still reading it for this one: the slot is refilled only after every warp is done).
__device__ int decode_entropy_plane(const uint8_t* pl, uint32_t plen, int H, int W, int t, int lane, uint8_t* smem,
                                    uint16_t* dst, int& s_bad) {
  uint8_t* slot2k = smem;                                          // [4096]
  uint32_t* bins = reinterpret_cast<uint32_t*>(smem + kEntM);     // [256]: hi | f << 16
  uint32_t* cums = bins + 256;                                     // [256]
  const int delta = pl[0], Lb = pl[1], b = pl[2], K = ld_u16(pl + 4);
  const uint32_t raw = ld_u32(pl + 8);
  const uint32_t hdr = (16u + 4u * (uint32_t)K + 3u) & ~3u;
  const uint32_t nwo = (uint32_t)(((uint64_t)H * b + 31) / 32);
  bool bad = delta > 1 || Lb != (int)kEntL || b > 16 || K < 1 || K > 256 || (raw & 3u) ||
             (uint64_t)hdr + 4ull * W + 4ull * (W / 32) > raw || (uint64_t)raw + 4ull * nwo * W > plen;
  if (t == 0) s_bad = 0;
  ent_bar();
  if (!bad && t < K) {
    const uint32_t v = ld_u32(pl + 16 + 4 * t);
    const uint32_t hv = v & 0xFFFFu, fv = v >> 16;
    bins[t] = v;
    if (fv == 0 || (hv >> (16 - b))) bad = true;
    if (t && hv <= (ld_u32(pl + 12 + 4 * t) & 0xFFFFu)) bad = true;
  }
  if (bad) s_bad = 1;
  ent_bar();
  if (s_bad) return 4;
  if (t < K) {  // exclusive prefix of the frequencies (K <= 256: a short sequential sum per bin)
    uint32_t c = 0;
    for (int k = 0; k < t; ++k) c += bins[k] >> 16;
    cums[t] = c;
    if (t == K - 1 && c + (bins[t] >> 16) != kEntM) s_bad = 1;
  }
  ent_bar();
  if (s_bad) return 4;
  for (uint32_t sl = (uint32_t)t; sl < kEntM; sl += kPlaneThreads) {  // slot -> bin: binary search
    int lo = 0, hi = K - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (cums[mid] <= sl) lo = mid; else hi = mid - 1;
    }
    slot2k[sl] = (uint8_t)lo;
  }
  ent_bar();
  const uint32_t* states = reinterpret_cast<const uint32_t*>(pl + hdr);
  const uint32_t* woff = states + W;
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t bmask = b ? ((1u << b) - 1u) : 0u;
  int err = 0;
  for (int x = t; x < W; x += kPlaneThreads) {  // warp-uniform: W % 32 == 0
    const int g = x >> 5;
    const uint32_t ws = woff[g], we = g + 1 < W / 32 ? woff[g + 1] : raw;
    const bool wbad = (ws & 3u) || ws < hdr + 4u * W + 4u * (W / 32) || we > raw || ws > we;
    const uint32_t nw = wbad ? 0u : (we - ws) / 2;
    const uint16_t* words = reinterpret_cast<const uint16_t*>(pl + ws);
    const uint32_t* rw = reinterpret_cast<const uint32_t*>(pl + raw) + (size_t)nwo * x;
    uint32_t st = states[x], wi = 0, prev = 0, rwi = 0;
    uint64_t rbuf = 0;
    uint32_t rfill = 0;
    bool cbad = wbad;
    for (int y = 0; y < H; ++y) {
      const uint32_t sl = st & (kEntM - 1);
      const int k = slot2k[sl];
      const uint32_t bv = bins[k];
      st = (bv >> 16) * (st >> kEntL) + sl - cums[k];
      const bool need = st < (1u << 16);
      const uint32_t m = __ballot_sync(0xffffffffu, need);
      if (need) {
        const uint32_t pos = wi + __popc(m & lt);
        if (pos < nw) st = (st << 16) | words[pos];
        else cbad = true;
      }
      wi += __popc(m);
      uint32_t o = 0;
      if (b) {
        if (rfill < (uint32_t)b) {
          rbuf |= (uint64_t)(rwi < nwo ? rw[rwi] : 0u) << rfill;
          ++rwi;
          rfill += 32;
        }
        o = (uint32_t)rbuf & bmask;
        rbuf >>= b;
        rfill -= b;
      }
      const uint32_t s = (b == 16 ? 0u : ((bv & 0xFFFFu) << b)) | o;
      const uint32_t u = delta ? ((prev + ((s >> 1) ^ (uint32_t)(-(int)(s & 1)))) & 0xFFFFu) : s;
      prev = u;
      dst[(size_t)y * W + x] = omap_inv((uint16_t)u);
    }
    if (cbad) err = 4;
  }
  if (err) s_bad = 1;
  ent_bar();
  return s_bad ? 4 : 0;
}

struct PlaneInfo {
  int code, mode;
  uint32_t plen;          // mode 3: the plane's length (its bytes start at `start`)
  uint32_t start, bytes;  // mode 1: the plane's canonical byte range (bytes = 0: rows from global)
  uint32_t payload, nbytes;
  uint32_t lo;            // staged copy of [lo, start + bytes) at the buffer's base (lo = start & ~15)
  int use_bar;            // the bulk part of the copy completes on the buffer's mbarrier
};

// thread 0: validate the plane's header, and for mode 1 start staging its rows into `buf`
__device__ void plane_prep(const uint8_t* base, uint32_t nbytes, bool aligned16, int c, int C, int H, int W,
                           PlaneInfo& pi, uint8_t* buf, uint64_t* bar) {
  int code = 0, mode = -1;
  uint32_t start = 0, bytes = 0, table = 0, payload = 0, plen = 0;
  if (nbytes < 32 || base[0] != 'L' || base[1] != 'B' || base[2] != 'L' || base[3] != 'P' || base[4] != 1 ||
      base[5] != 1)
    code = 2;
  else if (ld_u16(base + 8) != C || ld_u16(base + 10) != H || ld_u16(base + 12) != W)
    code = 3;
  else if (ld_u32(base + 16) != nbytes)
    code = 4;
  if (!code) {
    mode = base[6];
    table = ld_u32(base + 20);
    payload = ld_u32(base + 24);
    const long long rows_per = (long long)C * H;
    if (mode == 0) {
      if (payload != 32 || 32ull + 2ull * rows_per * W > nbytes) code = 4;
    } else if (mode == 2) {
      if (table != 32 || payload != 32u + 8u * (uint32_t)C || (unsigned long long)payload + rows_per * W > nbytes)
        code = 4;
    } else if (mode == 1) {
      if ((W & 31) || table != 32 || payload != 32u + 4u * (uint32_t)rows_per || payload > nbytes) {
        code = 4;
      } else {  // canonical layout: this plane's rows are contiguous from row c*H's offset
        const uint32_t r0 = ld_u32(base + 32 + 4 * (c * H));
        const uint32_t r1 = c + 1 < C ? ld_u32(base + 32 + 4 * ((c + 1) * H)) : nbytes - payload;
        start = payload + r0;
        bytes = (aligned16 && r1 > r0 && (r0 & 3) == 0 && (r1 & 3) == 0 && r1 - r0 <= (uint32_t)kPlaneInBytes &&
                 (unsigned long long)payload + r1 <= nbytes) ? r1 - r0 : 0u;
      }
    } else if (mode == 3) {
      if ((W & 31) || W > 1024 || table != 32 || payload != 32u + 4u * (uint32_t)C || payload > nbytes) {
        code = 4;
      } else {  // the plane's byte range; the decode warps validate its contents
        const uint32_t p0 = ld_u32(base + 32 + 4 * c);
        const uint32_t p1 = c + 1 < C ? ld_u32(base + 32 + 4 * (c + 1)) : nbytes - payload;
        if ((p0 & 3) || p1 > nbytes - payload || (unsigned long long)p0 + 16 > p1) code = 4;
        else {
          start = payload + p0;
          plen = p1 - p0;  // staged into shared memory like a mode-1 plane when it fits
          bytes = (aligned16 && plen <= (uint32_t)kPlaneInBytes) ? plen : 0u;
        }
      }
    } else {
      code = 5;
    }
  }
  pi.code = code; pi.mode = mode; pi.start = start; pi.bytes = bytes; pi.payload = payload; pi.nbytes = nbytes;
  pi.plen = plen;
  pi.use_bar = 0;
  pi.lo = start & ~15u;
  if (!code && (mode == 1 || mode == 3) && bytes) {
    const uint32_t end = start + bytes, hi = end & ~15u;  // [lo, hi) by TMA (the caller), [hi, end) here
    for (uint32_t o = hi > pi.lo ? hi : pi.lo; o < end; o += 4)
      *reinterpret_cast<uint32_t*>(buf + (o - pi.lo)) = ld_u32(base + o);
  }
}

__global__ void __launch_bounds__(kPlaneThreads + 32, 3) lblp_unpack_plane_kernel(
    const uint8_t* __restrict__ blobs, const unsigned long long* __restrict__ offs,
    const unsigned int* __restrict__ sizes, int n, int C, int H, int W, __half* __restrict__ out, int* err) {
  // warps 0..kPlaneThreads/32-1 decode; the last warp is the producer: it validates each plane's
  // header and stages its rows (TMA) into a 2-slot ring, full / empty mbarriers, no block barrier
  extern __shared__ __align__(16) uint8_t s_dyn[];
  constexpr int kBuf = kPlaneInBytes + 32, kDecWarps = kPlaneThreads / 32;
  uint8_t* s_in[2] = {s_dyn, s_dyn + kBuf};
  __shared__ PlaneInfo s_pi[2];
  __shared__ __align__(8) uint64_t s_full[2], s_empty[2];
  __shared__ int s_ent_bad[2];  // mode-3 error flag per ring slot
  __shared__ __align__(16) uint8_t s_ent_tab[kEntM + 256 * 8];  // mode-3 slot -> bin table, bins, cums
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const long long planes = (long long)n * C;
  const int vals = H * W;
  if (t == 0) {
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&s_empty[i], kDecWarps);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (warp == kDecWarps) {  // producer
    if (lane == 0) {
      int k = 0;
      for (long long pl = blockIdx.x; pl < planes; pl += gridDim.x, ++k) {
        const int b = k & 1;
        ptx::mbar_wait(&s_empty[b], (uint32_t)(((k >> 1) & 1) ^ 1));  // slot free (first use: passes)
        const int bi = (int)(pl / C), c = (int)(pl - (long long)bi * C);
        const uint8_t* base = blobs + offs[bi];
        PlaneInfo& pi = s_pi[b];
        plane_prep(base, sizes[bi], (offs[bi] & 15) == 0, c, C, H, W, pi, s_in[b], nullptr);
        // plane_prep issued nothing (null barrier): issue the staging copy here with its bytes
        uint32_t tx = 0;
        if (!pi.code && (pi.mode == 1 || pi.mode == 3) && pi.bytes) {
          const uint32_t end = pi.start + pi.bytes, hi = end & ~15u;
          if (hi > pi.lo) tx = hi - pi.lo;
        }
        pi.use_bar = tx ? 1 : 0;
        if (tx) {
          ptx::mbar_arrive_expect_tx(&s_full[b], tx);
          ubulk_load(s_in[b], base + pi.lo, tx, &s_full[b]);
        } else {
          ptx::mbar_arrive(&s_full[b]);
        }
      }
    }
    return;
  }
  int k = 0;
  for (long long pl = blockIdx.x; pl < planes; pl += gridDim.x, ++k) {
    const int b = k & 1;
    ptx::mbar_wait(&s_full[b], (uint32_t)((k >> 1) & 1));
    const PlaneInfo pi = s_pi[b];
    const int bi = (int)(pl / C), c = (int)(pl - (long long)bi * C);
    const uint8_t* base = blobs + offs[bi];
    uint16_t* dst = reinterpret_cast<uint16_t*>(out) + (size_t)pl * vals;
    if (pi.code) {
      for (int i = t; i < vals; i += kPlaneThreads) dst[i] = 0;
      if (t == 0) atomicExch(err, pi.code);
    } else if (pi.mode == 0) {  // raw fp16: 16-byte vectors when aligned
      const uint8_t* src = base + pi.payload + 2ull * c * H * W;
      if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        const uint4* s16 = reinterpret_cast<const uint4*>(src);
        uint4* d16 = reinterpret_cast<uint4*>(dst);
        for (int i = t; i < vals / 8; i += kPlaneThreads) d16[i] = __ldg(s16 + i);
      } else {
        const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src);
        uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
        for (int i = t; i < vals / 2; i += kPlaneThreads) d32[i] = __ldg(s32 + i);
      }
    } else if (pi.mode == 2) {  // q8: 16 values per 16-byte load (4 per 32-bit load if unaligned)
      const float scale = __uint_as_float(ld_u32(base + 32 + 4 * c));
      const int zp = (int)ld_u32(base + 32 + 4 * C + 4 * c);
      const uint8_t* qb = base + pi.payload + (size_t)c * H * W;
      auto deq4 = [&](uint32_t w4, uint32_t& lo, uint32_t& hi) {
        uint16_t h[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float f = __fmul_rn((float)((int)(int8_t)(w4 >> (8 * e)) - zp), scale);
          h[e] = __half_as_ushort(__float2half_rn(f));
        }
        lo = h[0] | (uint32_t)h[1] << 16;
        hi = h[2] | (uint32_t)h[3] << 16;
      };
      if ((reinterpret_cast<uintptr_t>(qb) & 15) == 0) {
        const uint4* q = reinterpret_cast<const uint4*>(qb);
        uint4* d16 = reinterpret_cast<uint4*>(dst);
        for (int i = t; i < vals / 16; i += kPlaneThreads) {
          const uint4 w = __ldg(q + i);
          uint4 o0, o1;
          deq4(w.x, o0.x, o0.y);
          deq4(w.y, o0.z, o0.w);
          deq4(w.z, o1.x, o1.y);
          deq4(w.w, o1.z, o1.w);
          d16[2 * i] = o0;
          d16[2 * i + 1] = o1;
        }
      } else {
        const uint32_t* q = reinterpret_cast<const uint32_t*>(qb);
        uint2* d64 = reinterpret_cast<uint2*>(dst);
        for (int i = t; i < vals / 4; i += kPlaneThreads) {
          uint2 o;
          deq4(__ldg(q + i), o.x, o.y);
          d64[i] = o;
        }
      }
    } else if (pi.mode == 3) {
      const uint8_t* pl = pi.bytes ? s_in[b] + (pi.start - pi.lo) : base + pi.start;  // staged or global
      const int code = decode_entropy_plane(pl, pi.plen, H, W, t, lane, s_ent_tab, dst, s_ent_bad[b]);
      if (code) {
        for (int i = t; i < vals; i += kPlaneThreads) dst[i] = 0;
        if (t == 0) atomicExch(err, code);
      }
    } else {  // mode 1 from the staged copy
      const uint8_t* sb = s_in[b] + (pi.start - pi.lo);  // the plane's first byte
      int code = 0;
      const int L = W / 32;
      if ((L & (L - 1)) == 0 && L <= 32) {  // L lanes per row
        const int rows_per_pass = kPlaneThreads / L;
        for (int y0 = 0; y0 < H; y0 += rows_per_pass) {
          const int y = y0 + t / L;
          const bool active = y < H;
          const uint32_t roff = active ? ld_u32(base + 32 + 4 * (c * H + y)) : 0u, at = pi.payload + roff;
          uint16_t* drow = dst + (size_t)(active ? y : 0) * W;
          const bool fmt = active && ((roff & 3) || (unsigned long long)at > pi.nbytes);
          const bool staged = pi.bytes && at >= pi.start && at < pi.start + pi.bytes;
          const uint8_t* src = staged ? sb + (at - pi.start) : base + at;
          const uint32_t avail = fmt ? 0u : (staged ? pi.start + pi.bytes - at : pi.nbytes - at);
          int rc = decode_row_split(src, avail, L, lane, active && !fmt, drow);
          const bool retry = rc != 0 && staged;  // the row runs past the staged range: from global
          if (__any_sync(0xffffffffu, retry)) {
            const int rc2 = decode_row_split(base + at, pi.nbytes - at, L, lane, active && !fmt && retry, drow);
            if (retry) rc = rc2;
          }
          if (fmt) rc = 4;
          if (rc && active) {
            for (int e = 32 * (t & (L - 1)); e < 32 * (t & (L - 1)) + 32; e += 8)
              *reinterpret_cast<uint4*>(drow + e) = make_uint4(0, 0, 0, 0);
            code = rc;
          }
        }
      } else {
        for (int y = t; y < H; y += kPlaneThreads) {
          const uint32_t roff = ld_u32(base + 32 + 4 * (c * H + y)), at = pi.payload + roff;
          uint16_t* drow = dst + (size_t)y * W;
          int rc;
          if ((roff & 3) || (unsigned long long)at > pi.nbytes) {
            rc = 4;
          } else if (pi.bytes && at >= pi.start && at < pi.start + pi.bytes) {
            rc = decode_row_lane(sb + (at - pi.start), pi.start + pi.bytes - at, W, drow);
            if (rc) rc = decode_row_lane(base + at, pi.nbytes - at, W, drow);  // runs past the staged range
          } else {
            rc = decode_row_lane(base + at, pi.nbytes - at, W, drow);
          }
          if (rc) {
            for (int e = 0; e < W; e += 8) *reinterpret_cast<uint4*>(drow + e) = make_uint4(0, 0, 0, 0);
            code = rc;
          }
        }
      }
      if (code) atomicExch(err, code);
    }
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&s_empty[b]);  // this warp is done with slot b
  }
}

void launch_lblp_unpack(const uint8_t* blobs, const unsigned long long* offs, const unsigned int* sizes, int n,
                        int C, int H, int W, __half* out, int* err, cudaStream_t s) {
  if ((long long)H * W <= kPlaneMaxVals && W % 32 == 0 && !g_unpack_rows) {
    const long long planes = (long long)n * C;
    const long long cap = (long long)num_sms() * 3;  // three 70 KB CTAs per SM
    constexpr int smem = 2 * (kPlaneInBytes + 32);
    if (ensure_smem_attr(reinterpret_cast<const void*>(lblp_unpack_plane_kernel), smem)) {
      lblp_unpack_plane_kernel<<<(int)(planes < cap ? planes : cap), kPlaneThreads + 32, smem, s>>>(blobs, offs, sizes,
                                                                                                     n, C, H, W, out, err);
      return;
    }
  }
  const long long rows = (long long)n * C * H;
  long long blocks = (rows + 7) / 8;
  const long long cap = (long long)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  lblp_unpack_kernel<<<(int)blocks, 256, 0, s>>>(blobs, offs, sizes, n, C, H, W, out, err);
}

}  // namespace lbx
