// LBLP v1 mode-1 (lossless) packer on the GPU -- the write path of SURVEY.md 8(f) item 2 for latents
// that are already on the device (e.g. straight out of a VAE encoder).  Byte-identical to the host
// packer (csrc/codec.cpp lblp_pack) and to the C oracle; format in include/lbx/lblp.h.
//
//   K-a  lblp_rows_lane_kernel  W/32 lanes per latent row (c, y), one 32-value mini-block per
//                               lane: order-map, delta against the value before, zigzag, width =
//                               bit length of the OR; the row's byte size (head + 4 * sum widths).
//   K-b  lblp_scan_kernel       one block per latent: exclusive scan of the row sizes -> row
//                               table, header, total size.
//   K-c  lblp_write_lane_kernel lanes as in K-a pack their words from a 64-bit accumulator into
//                               the warp's rows in shared memory (bits0, widths, padding, words);
//                               each row is then copied out with 4-byte stores across the warp.
// The warp-per-row forms (lblp_rows_kernel / lblp_write_kernel: warp OR-reductions per word) are
// kept for widths whose W/32 is not a power of two.
// Blob i is written at out + i * stride (stride >= lbx_pack_bound); its size goes to sizes[i].
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "gemm_tc.cuh"
#include "kernels.cuh"

namespace lbx {

namespace {

__device__ __forceinline__ uint16_t omap16(uint16_t u) { return (u & 0x8000u) ? (uint16_t)~u : (uint16_t)(u | 0x8000u); }

// zigzag delta of lane's value against its predecessor in the row (0 for the row's first value)
__device__ __forceinline__ uint32_t zz_of(const uint16_t* row, int j, int lane, uint16_t& carry) {
  const uint16_t v = omap16(row[32 * j + lane]);
  uint16_t prev = (uint16_t)__shfl_up_sync(0xffffffffu, v, 1);
  if (lane == 0) prev = (j == 0) ? v : carry;
  carry = (uint16_t)__shfl_sync(0xffffffffu, v, 31);
  const uint16_t d = (uint16_t)(v - prev);
  return (uint16_t)((uint16_t)(d << 1) ^ (uint16_t)((int16_t)d >> 15));
}

__global__ void __launch_bounds__(256) lblp_rows_kernel(const uint16_t* __restrict__ x, int n, int C, int H, int W,
                                                        uint8_t* __restrict__ widths, uint32_t* __restrict__ row_bytes) {
  const int lane = threadIdx.x & 31, nmb = W / 32;
  const uint32_t head = (2u + (uint32_t)nmb + 3u) & ~3u;
  const long long rows = (long long)n * C * H;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long r = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    const uint16_t* row = x + r * W;
    uint16_t carry = 0;
    uint32_t words = 0;
    for (int j = 0; j < nmb; ++j) {
      const uint32_t z = zz_of(row, j, lane, carry);
      const uint32_t m = __reduce_or_sync(0xffffffffu, z);  // same bit length as the max
      const uint32_t bw = m ? 32u - __clz(m) : 0u;
      if (lane == 0) widths[r * nmb + j] = (uint8_t)bw;
      words += bw;
    }
    if (lane == 0) row_bytes[r] = head + 4u * words;
  }
}

__global__ void __launch_bounds__(1024) lblp_scan_kernel(const uint32_t* __restrict__ row_bytes, int rows_per, int C,
                                                         int H, int W, uint8_t* __restrict__ out, long long stride,
                                                         uint32_t* __restrict__ sizes) {
  __shared__ uint32_t part[1024];
  const int img = blockIdx.x, t = threadIdx.x;
  const uint32_t* rb = row_bytes + (size_t)img * rows_per;
  uint8_t* blob = out + (size_t)img * stride;
  const uint32_t payload = 32u + 4u * (uint32_t)rows_per;
  const int per = (rows_per + 1023) / 1024, r0 = t * per;
  uint32_t s = 0;
  for (int r = r0; r < r0 + per && r < rows_per; ++r) s += rb[r];
  part[t] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele inclusive scan of the per-thread sums
    const uint32_t v = t >= o ? part[t - o] : 0u;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  uint32_t off = part[t] - s;  // exclusive prefix of this thread's rows
  uint32_t* table = reinterpret_cast<uint32_t*>(blob + 32);
  for (int r = r0; r < r0 + per && r < rows_per; ++r) {
    table[r] = off;
    off += rb[r];
  }
  if (t == 0) {
    const uint32_t total = payload + part[1023];
    uint32_t* h32 = reinterpret_cast<uint32_t*>(blob);
    h32[0] = 0x504C424Cu;                                    // "LBLP"
    h32[1] = 1u | (1u << 8) | (1u << 16);                    // version 1, dtype fp16, mode 1, flags 0
    h32[2] = (uint32_t)C | ((uint32_t)H << 16);
    h32[3] = (uint32_t)W;                                    // W, reserved 0
    h32[4] = total;
    h32[5] = 32u;
    h32[6] = payload;
    h32[7] = 0u;
    sizes[img] = total;
  }
}

__global__ void __launch_bounds__(256) lblp_write_kernel(const uint16_t* __restrict__ x, int n, int C, int H, int W,
                                                         const uint8_t* __restrict__ widths, uint8_t* __restrict__ out,
                                                         long long stride) {
  const int lane = threadIdx.x & 31, nmb = W / 32;
  const uint32_t head = (2u + (uint32_t)nmb + 3u) & ~3u;
  const long long rows_per = (long long)C * H, rows = rows_per * n;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long r = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    const long long img = r / rows_per, rr = r - img * rows_per;
    uint8_t* blob = out + img * stride;
    const uint32_t payload = 32u + 4u * (uint32_t)rows_per;
    const uint32_t roff = reinterpret_cast<const uint32_t*>(blob + 32)[rr];
    uint8_t* orow = blob + payload + roff;  // 4-byte aligned (payload and every row size are)
    const uint16_t* row = x + r * W;
    const uint8_t* wr = widths + r * nmb;
    // head: bits0, widths, zero padding to a multiple of 4 bytes
    for (uint32_t b = (uint32_t)lane; b < head; b += 32)
      orow[b] = b < 2 ? (uint8_t)(row[0] >> (8 * b)) : (b < 2u + (uint32_t)nmb ? wr[b - 2] : (uint8_t)0);
    uint32_t* words = reinterpret_cast<uint32_t*>(orow + head);
    uint16_t carry = 0;
    uint32_t wpos = 0;
    for (int j = 0; j < nmb; ++j) {
      const uint32_t z = zz_of(row, j, lane, carry);
      const uint32_t bw = wr[j];
      if (bw) {
        const uint32_t bit = (uint32_t)lane * bw, wi = bit >> 5, sh = bit & 31;
        const uint32_t lo = z << sh, hi = sh + bw > 32 ? z >> (32 - sh) : 0u;
        for (uint32_t i = 0; i < bw; ++i) {  // word i: OR of the lanes' shares that land in it
          const uint32_t mine = (wi == i ? lo : 0u) | (wi + 1 == i ? hi : 0u);
          const uint32_t word = __reduce_or_sync(0xffffffffu, mine);
          if (lane == (int)i) words[wpos + i] = word;
        }
      }
      wpos += bw;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Lane-per-mini-block forms (W/32 a power of two <= 32): lane j of a row's segment owns mini-block
// j.  Its 32 zigzag deltas need only the value before the block (no prefix), its width is the bit
// length of their OR, and it packs its own words from a 64-bit accumulator -- no warp reductions.
// Bytes identical to the warp-per-row kernels above.
__device__ __forceinline__ void block_deltas(const uint16_t* row, int j, uint32_t (&z)[32]) {
  const uint4* p = reinterpret_cast<const uint4*>(row + 32 * j);
  uint32_t w[16];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 u = __ldg(p + q);
    w[4 * q] = u.x; w[4 * q + 1] = u.y; w[4 * q + 2] = u.z; w[4 * q + 3] = u.w;
  }
  uint16_t prev = j ? omap16(row[32 * j - 1]) : omap16((uint16_t)(w[0] & 0xFFFFu));
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const uint16_t v = omap16((uint16_t)(w[k >> 1] >> (16 * (k & 1))));
    const uint16_t d = (uint16_t)(v - prev);
    z[k] = (uint16_t)((uint16_t)(d << 1) ^ (uint16_t)((int16_t)d >> 15));
    prev = v;
  }
}

__global__ void __launch_bounds__(256) lblp_rows_lane_kernel(const uint16_t* __restrict__ x, int n, int C, int H,
                                                             int W, uint8_t* __restrict__ widths,
                                                             uint32_t* __restrict__ row_bytes) {
  const int L = W / 32, lane = threadIdx.x & 31, j = lane & (L - 1);
  const uint32_t head = (2u + (uint32_t)L + 3u) & ~3u;
  const long long rows = (long long)n * C * H;
  const long long seg = (long long)blockIdx.x * (blockDim.x / L) + threadIdx.x / L;
  const long long segs = (long long)gridDim.x * (blockDim.x / L);
  const long long iters = (rows + segs - 1) / segs;  // warp-uniform trip count (shuffles below)
  for (long long it = 0; it < iters; ++it) {
    const long long r = seg + it * segs;
    const bool active = r < rows;
    uint32_t bw = 0;
    if (active) {
      uint32_t z[32];
      block_deltas(x + r * W, j, z);
      uint32_t m = 0;
#pragma unroll
      for (int k = 0; k < 32; ++k) m |= z[k];
      bw = m ? 32u - __clz(m) : 0u;
      widths[r * L + j] = (uint8_t)bw;
    }
    uint32_t sum = bw;
    for (int o = 1; o < L; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o, L);
    if (active && j == 0) row_bytes[r] = head + 4u * sum;
  }
}

__global__ void __launch_bounds__(256) lblp_write_lane_kernel(const uint16_t* __restrict__ x, int n, int C, int H,
                                                              int W, const uint8_t* __restrict__ widths,
                                                              uint8_t* __restrict__ out, long long stride) {
  // each warp assembles its 32/L rows in shared memory (head + words), then copies every row out
  // with 4-byte stores across the warp (rows are 4-byte aligned): full sectors instead of one
  // scattered word per lane per store
  extern __shared__ __align__(16) uint8_t s_rows[];
  const int L = W / 32, lane = threadIdx.x & 31, j = lane & (L - 1), warp = threadIdx.x >> 5;
  const uint32_t head = (2u + (uint32_t)L + 3u) & ~3u, rmax = head + 2u * (uint32_t)W;  // bytes per row slot
  const int rpw = 32 / L;  // rows per warp
  uint8_t* wbuf = s_rows + (size_t)warp * rpw * rmax;
  const long long rows_per = (long long)C * H, rows = rows_per * n;
  const long long seg = (long long)blockIdx.x * (blockDim.x / L) + threadIdx.x / L;
  const long long segs = (long long)gridDim.x * (blockDim.x / L);
  const long long iters = (rows + segs - 1) / segs;
  const uint32_t payload = 32u + 4u * (uint32_t)rows_per;
  for (long long it = 0; it < iters; ++it) {
    const long long r = seg + it * segs;
    const bool active = r < rows;
    const uint32_t bw = active ? widths[r * L + j] : 0u;
    uint32_t incl = bw;
    for (int o = 1; o < L; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o, L);
      if (j >= o) incl += u;
    }
    const uint32_t rbytes = head + 4u * __shfl_sync(0xffffffffu, incl, (lane & ~(L - 1)) + L - 1);
    uint8_t* srow = wbuf + (size_t)(lane / L) * rmax;
    if (active) {
      const uint16_t* row = x + r * W;
      srow[2 + j] = (uint8_t)bw;
      if (j == 0) {
        *reinterpret_cast<uint16_t*>(srow) = row[0];
        for (uint32_t b = 2u + (uint32_t)L; b < head; ++b) srow[b] = 0;
      }
      if (bw) {
        uint32_t z[32];
        block_deltas(row, j, z);
        uint32_t* wout = reinterpret_cast<uint32_t*>(srow + head) + (incl - bw);
        uint64_t acc = 0;
        uint32_t nacc = 0, wi = 0;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          acc |= (uint64_t)z[k] << nacc;
          nacc += bw;
          if (nacc >= 32) {
            wout[wi++] = (uint32_t)acc;
            acc >>= 32;
            nacc -= 32;
          }
        }
      }
    }
    __syncwarp();
    // copy the warp's rows out, one row at a time across all 32 lanes
    for (int q = 0; q < rpw; ++q) {
      const long long rq = __shfl_sync(0xffffffffu, r, q * L);
      const uint32_t nb = __shfl_sync(0xffffffffu, rbytes, q * L);
      if (rq >= rows) continue;  // warp-uniform
      const long long img = rq / rows_per, rr = rq - img * rows_per;
      uint8_t* blob = out + img * stride;
      uint32_t* dst = reinterpret_cast<uint32_t*>(blob + payload + reinterpret_cast<const uint32_t*>(blob + 32)[rr]);
      const uint32_t* src = reinterpret_cast<const uint32_t*>(wbuf + (size_t)q * rmax);
      for (uint32_t i = lane; i < nb / 4; i += 32) dst[i] = src[i];
    }
    __syncwarp();
  }
}

}  // namespace

size_t lblp_pack_bound(int C, int H, int W) {
  const size_t head = (2u + (size_t)(W / 32) + 3u) & ~size_t(3);
  return 32 + 4 * (size_t)C * H + (size_t)C * H * (head + 2 * (size_t)W);  // every mini-block 16 bits wide
}

cudaError_t launch_lblp_pack(const uint16_t* x, int n, int C, int H, int W, uint8_t* out, long long stride,
                             uint32_t* sizes, uint8_t* widths_tmp, uint32_t* row_bytes_tmp, cudaStream_t s) {
  if (n <= 0 || W % 32 || C <= 0 || H <= 0 || C > 65535 || H > 65535 || W > 65535 ||
      (size_t)stride < lblp_pack_bound(C, H, W) || (stride & 3))
    return cudaErrorInvalidValue;
  const long long rows = (long long)n * C * H;
  long long blocks = (rows + 7) / 8;
  const long long cap = (long long)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  const int L = W / 32;
  const bool lanes = (L & (L - 1)) == 0 && L <= 32;  // lane-per-mini-block kernels
  const long long lane_blocks = std::min<long long>((rows * L + 255) / 256, (long long)num_sms() * 8);
  if (lanes) lblp_rows_lane_kernel<<<(int)lane_blocks, 256, 0, s>>>(x, n, C, H, W, widths_tmp, row_bytes_tmp);
  else lblp_rows_kernel<<<(int)blocks, 256, 0, s>>>(x, n, C, H, W, widths_tmp, row_bytes_tmp);
  lblp_scan_kernel<<<n, 1024, 0, s>>>(row_bytes_tmp, C * H, C, H, W, out, stride, sizes);
  const int wsmem = 8 * (32 / (L ? L : 1)) * (int)(((2u + (uint32_t)L + 3u) & ~3u) + 2u * (uint32_t)W);
  if (lanes && wsmem <= 48 * 1024)
    lblp_write_lane_kernel<<<(int)lane_blocks, 256, wsmem, s>>>(x, n, C, H, W, widths_tmp, out, stride);
  else
    lblp_write_kernel<<<(int)blocks, 256, 0, s>>>(x, n, C, H, W, widths_tmp, out, stride);
  return cudaGetLastError();
}

}  // namespace lbx
