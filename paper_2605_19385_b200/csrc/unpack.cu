// K1: LBLP v1 latent unpack on the GPU (format: include/lbx/lblp.h).  One warp per latent row
// (c, y): lane k owns value k of every 32-value mini-block, extracts its zigzag delta from the
// bit-packed words, and a warp-wide inclusive scan (mod 2^16) rebuilds the order-mapped values.
// Stores are 64 contiguous bytes per warp per mini-block.  Bit-exact by construction; checked
// against the C oracle (oracle/lblp_ref.c) in tests/test_gpu_unpack.py.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "gemm_tc.cuh"
#include "kernels.cuh"

namespace lbx {

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

void launch_lblp_unpack(const uint8_t* blobs, const unsigned long long* offs, const unsigned int* sizes, int n,
                        int C, int H, int W, __half* out, int* err, cudaStream_t s) {
  const long long rows = (long long)n * C * H;
  long long blocks = (rows + 7) / 8;
  const long long cap = (long long)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  lblp_unpack_kernel<<<(int)blocks, 256, 0, s>>>(blobs, offs, sizes, n, C, H, W, out, err);
}

}  // namespace lbx
