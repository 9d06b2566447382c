// Decoder tail on the tensor cores: GroupNorm(128) + SiLU -> conv3x3 128 -> 3
// (+bias) -> (x/2 + 0.5).clamp(0, 1) * 255 -> round-half-even -> uint8 HWC.
//
// The layer is HBM-bound (it reads 256 B and writes 3 B per output pixel), so the design goal is
// to touch every input element once: a persistent CTA walks a 128-pixel-wide column strip of R
// output rows and keeps a ring of input rows in shared memory.  Each input row (130 px with the
// 1-pixel halo x 128 channels) is loaded once by TMA, normalised + activated in place by eight
// transform warps (GroupNorm affine in fp32, SiLU, one fp16 rounding; out-of-image pixels keep
// TMA's zero fill because the conv pads *after* the activation), and then feeds the three output
// rows that need it.  The three kernel rows are folded into N: per INPUT row y',
//   E_y'[px, 4 ky + c] = sum over (kx, 64-channel block, K16) of A_y'[px + kx] . W[ky][kx][c]
// with A = rows of input row y' shifted by kx pixels (a row-shifted UMMA descriptor into the same
// 128B-swizzled buffer, as in gemm_tc.cu's halo staging) and B = [16 x 384] fp16 weights resident
// in smem (rows 4 ky + c, c < 3; the rest zero): 24 tcgen05.mma (M = 128 pixels, N = 16, K = 16)
// into a 4-deep ring of 16-column TMEM accumulators.  Output row y = E_{y-1}[., 0..2] +
// E_y[., 4..6] + E_{y+1}[., 8..10] is summed by four epilogue warps (one pixel per thread), which
// write the uint8 RGB.  An input row's smem slot is released right after its own 24 MMAs, so the
// whole ring prefetches (the first version kept three rows resident for 72 MMAs per output row
// and ran latency-bound at ~2.5 TB/s).
//
// Warps: 0 TMA producer, 1 TMEM allocator + MMA issuer, 2..5 epilogue, 6.. transform in
// KCO_GROUPS groups of eight that take input rows round-robin.  One group was the kernel's serial
// stage (~1.1 us per row against ~0.8 us for the row's HBM share): batch 32 at 1024^2 went
// 4.31 TB/s (one group) -> 4.72 (two) -> 5.43 (three, 3 chunks in flight per thread) = 0.83 of
// the measured HBM copy rate (scripts/gpu_tail2.sh).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "act.cuh"
#include "gemm_tc.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace lbx {

namespace {

#ifndef KCO_GROUPS
#define KCO_GROUPS 3
#endif
#ifndef KCO_NK
#define KCO_NK 3
#endif
constexpr int kCoXfGroups = KCO_GROUPS;                   // transform groups (alternate input rows)
constexpr int kCoThreads = 192 + kCoXfGroups * 256;
constexpr int kCoNK = KCO_NK;                     // transform chunks in flight per thread
constexpr int kCoSlots = 6;                       // input-row ring depth
constexpr int kCoBoxBytes = 64 * 130 * 2;         // one TMA box: 64 channels x 130 pixels
constexpr int kCoCbPitch = 17408;                 // 1024-aligned pitch of one 64-channel block
constexpr int kCoSlotBytes = 2 * kCoCbPitch;      // one input row, 128 channels
constexpr int kCoBBytes = 6 * 2048;               // 6 k-blocks (kx, channel block) x (16 rows x 128 B)
constexpr int kCoE = 4;                           // TMEM ring of per-input-row partial sums
constexpr int kCoSmem = 1024 + kCoSlots * kCoSlotBytes + kCoBBytes + 256;
constexpr uint32_t kCoIdesc = ptx::idesc_f16(128, 16);

struct CoParams {
  const float2* ss;   // [n][128] GroupNorm affine (scale, shift)
  const float* w;     // [3][9][128] fp32 (K index = tap * 128 + channel)
  const float* bias;  // [3]
  uint8_t* rgb;       // [n][H][W][3]
  int n, H, W, R;     // R output rows per work item
  int strips, bands, items;
};

__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}

__device__ __forceinline__ void item_coords(const CoParams& p, int it, int& img, int& x0, int& y0) {
  const int per_img = p.strips * p.bands;
  img = it / per_img;
  const int r = it - img * per_img;
  const int band = r / p.strips;
  x0 = (r - band * p.strips) * 128;
  y0 = band * p.R;
}

template <bool H2>
__global__ void __launch_bounds__(kCoThreads, 1)
    conv_out_tc_kernel(const __grid_constant__ CUtensorMap tmX, const CoParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sRow = smem;
  uint8_t* sB = smem + kCoSlots * kCoSlotBytes;
  uint64_t* slot_full = reinterpret_cast<uint64_t*>(sB + kCoBBytes);
  uint64_t* slot_xf = slot_full + kCoSlots;
  uint64_t* slot_empty = slot_xf + kCoSlots;
  uint64_t* acc_full = slot_empty + kCoSlots;
  uint64_t* acc_empty = acc_full + kCoE;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + kCoE);

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();

  // weights -> smem once: fp32 [c][ky][kx][ci] -> fp16 B[n = 4 ky + c][k = kx * 128 + ci], K-major
  // SW128 in 6 k-blocks of 64; rows with c = 3 or ky = 3 are zero
  for (int q = threadIdx.x; q < 6 * 16 * 8; q += blockDim.x) {
    const int kb = q / 128, rem = q - kb * 128, row = rem >> 3, ch = rem & 7;
    const int ky = row >> 2, c = row & 3;
    uint32_t wd[4] = {0, 0, 0, 0};
    if (ky < 3 && c < 3) {
      const int kx = kb >> 1, cb = kb & 1;
      const float* src = p.w + ((c * 3 + ky) * 3 + kx) * 128 + cb * 64 + ch * 8;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const __half2 h = __floats2half2_rn(src[2 * j], src[2 * j + 1]);
        wd[j] = *reinterpret_cast<const uint32_t*>(&h);
      }
    }
    *reinterpret_cast<uint4*>(sB + kb * 2048 + row * 128 + ((ch ^ (row & 7)) << 4)) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
  }
  ptx::fence_proxy_async_smem();
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&tmX);
    for (int s = 0; s < kCoSlots; ++s) {
      ptx::mbar_init(&slot_full[s], 1);
      ptx::mbar_init(&slot_xf[s], 8);
      ptx::mbar_init(&slot_empty[s], 1);
    }
    for (int i = 0; i < kCoE; ++i) {
      ptx::mbar_init(&acc_full[i], 1);
      ptx::mbar_init(&acc_empty[i], 4);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<1>(tmem_slot, 16 * kCoE);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int rows_in = p.R + 2;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (ptx::elect_one()) {
      uint32_t gi = 0;
      for (int it = blockIdx.x; it < p.items; it += gridDim.x) {
        int img, x0, y0;
        item_coords(p, it, img, x0, y0);
        for (int r = 0; r < rows_in; ++r, ++gi) {
          const int s = gi % kCoSlots;
          ptx::mbar_wait(&slot_empty[s], ((gi / kCoSlots) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&slot_full[s], 2 * kCoBoxBytes);
          uint8_t* dst = sRow + s * kCoSlotBytes;
          ptx::tma_load_4d(&tmX, &slot_full[s], dst, 0, x0 - 1, y0 - 1 + r, img);
          ptx::tma_load_4d(&tmX, &slot_full[s], dst + kCoCbPitch, 64, x0 - 1, y0 - 1 + r, img);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (one thread)
    // input row i of the CTA's global sequence -> E slot i % kCoE; it waits for the slot's previous
    // occupant E_{i-4}, whose last reader is the epilogue of output row i - 4 of the same band (or
    // the band's end)
    if (ptx::elect_one()) {
      uint32_t gi = 0;
      const uint64_t b_desc0 = ptx::sdesc_k_sw128(ptx::smem_u32(sB));
      for (int it = blockIdx.x; it < p.items; it += gridDim.x) {
        for (int r = 0; r < rows_in; ++r, ++gi) {
          const uint32_t s_row = gi % kCoSlots, e = gi % kCoE;
          ptx::mbar_wait(&slot_xf[s_row], (gi / kCoSlots) & 1);
          ptx::mbar_wait(&acc_empty[e], ((gi / kCoE) & 1) ^ 1);
          ptx::tc_fence_after();
          const uint64_t a_desc0 = ptx::sdesc_k_sw128(ptx::smem_u32(sRow + s_row * kCoSlotBytes));
          const uint32_t d_tmem = tmem_base + e * 16;
#pragma unroll
          for (int kx = 0; kx < 3; ++kx) {
#pragma unroll
            for (int cb = 0; cb < 2; ++cb) {
              const uint64_t a_desc = a_desc0 + (uint64_t)((cb * kCoCbPitch + kx * 128) >> 4);
              const uint64_t b_desc = b_desc0 + (uint64_t)(((kx * 2 + cb) * 2048) >> 4);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                ptx::mma_f16_ss<1>(d_tmem, a_desc + 2 * k, b_desc + 2 * k, kCoIdesc, (kx | cb | k) != 0);
            }
          }
          ptx::mma_commit<1>(&acc_full[e]);
          ptx::mma_commit<1>(&slot_empty[s_row]);  // the input row is consumed
        }
      }
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------------ epilogue (one pixel per thread)
    // output row j of a band whose first input row has global index base: E_{base+j} (ky = 0),
    // E_{base+j+1} (ky = 1), E_{base+j+2} (ky = 2); afterwards E_{base+j} has no later reader
    const uint32_t q = warp & 3;
    const float b0 = p.bias[0], b1 = p.bias[1], b2 = p.bias[2];
    uint32_t gi = 0;
    for (int it = blockIdx.x; it < p.items; it += gridDim.x) {
      int img, x0, y0;
      item_coords(p, it, img, x0, y0);
      const int x = x0 + (int)(q * 32 + lane);
      const uint32_t base = gi;
      for (int j = 0; j < p.R; ++j) {
        float acc[3] = {b0, b1, b2};
#pragma unroll
        for (int ky = 0; ky < 3; ++ky) {
          const uint32_t i = base + j + ky, e = i % kCoE;
          ptx::mbar_wait(&acc_full[e], (i / kCoE) & 1);
          ptx::tc_fence_after();
          uint32_t r[4];
          tmem_ld4(tmem_base + ((q * 32u) << 16) + e * 16 + ky * 4, r);
          ptx::tmem_ld_wait();
          acc[0] += __uint_as_float(r[0]);
          acc[1] += __uint_as_float(r[1]);
          acc[2] += __uint_as_float(r[2]);
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          ptx::mbar_arrive_relaxed(&acc_empty[(base + j) % kCoE]);
          if (j == p.R - 1) {  // the band's last two input rows have no later reader either
            ptx::mbar_arrive_relaxed(&acc_empty[(base + j + 1) % kCoE]);
            ptx::mbar_arrive_relaxed(&acc_empty[(base + j + 2) % kCoE]);
          }
        }
        uint8_t* o = p.rgb + (((size_t)img * p.H + (y0 + j)) * p.W + x) * 3;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          float t = __fadd_rn(__fmul_rn(acc[k], 0.5f), 0.5f);
          t = fminf(fmaxf(t, 0.f), 1.f);
          o[k] = (uint8_t)__float2int_rn(__fmul_rn(t, 255.f));  // round-half-even
        }
      }
      gi = base + rows_in;
    }
  } else {
    // ------------------------------------------------------------------ transform (warps 6..21)
    // group g = (warp - 6) / 8 takes the input rows with gi % kCoXfGroups == g (kCoSlots is a
    // multiple of the group count, so a group keeps to its own slots); within a group thread t owns
    // logical chunk lc = t & 7 (8 channels) of channel block cb = (t >> 3) & 1 for pixels
    // (t >> 4) + 16 k; the physical 16-byte chunk is lc ^ (px & 7) (128B swizzle).
    static_assert(kCoSlots % kCoXfGroups == 0, "slots per transform group");
    const uint32_t grp = (warp - 6) >> 3;
    const int t = ((int)threadIdx.x - 6 * 32) & 255;
    const int lc = t & 7, cb = (t >> 3) & 1, p0 = t >> 4;
    const int c0 = cb * 64 + lc * 8;
    uint32_t gi = 0;
    int cur_img = -1;
    float a[8], b[8];
    for (int it = blockIdx.x; it < p.items; it += gridDim.x) {
      int img, x0, y0;
      item_coords(p, it, img, x0, y0);
      if (img != cur_img) {
        cur_img = img;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float2 v = p.ss[(size_t)img * 128 + c0 + k];
          a[k] = H2 ? 0.5f * v.x : v.x;  // H2: halved for gn_silu8_h2_half
          b[k] = H2 ? 0.5f * v.y : v.y;
        }
      }
      for (int r = 0; r < rows_in; ++r, ++gi) {
        if (gi % kCoXfGroups != grp) continue;
        const int s = gi % kCoSlots;
        ptx::mbar_wait(&slot_full[s], (gi / kCoSlots) & 1);
        const int y = y0 - 1 + r;
        if (y >= 0 && y < p.H) {
          const uint32_t blk = ptx::smem_u32(sRow + s * kCoSlotBytes + cb * kCoCbPitch);  // shared-space
                                                                                       // address: LDS/STS, not generic LD/ST
          // this thread's chunks of the row (pixels p0 + 16k, k < 9) in passes of kCoNK: each pass
          // loads all its chunks before transforming any (independent LDS -> math -> STS chains)
#pragma unroll
          for (int k0 = 0; k0 < 9; k0 += kCoNK) {
            uint4 v[kCoNK];
            bool ok[kCoNK];
#pragma unroll
            for (int k = 0; k < kCoNK; ++k) {
              const int px = p0 + 16 * (k0 + k);
              const int gx = x0 - 1 + px;
              ok[k] = k0 + k < 9 && px < 130 && gx >= 0 && gx < p.W;  // padding stays zero
              if (ok[k]) v[k] = ptx::lds128(blk + px * 128 + ((lc ^ (px & 7)) << 4));
            }
#pragma unroll
            for (int k = 0; k < kCoNK; ++k) {
              const int px = p0 + 16 * (k0 + k);
              if (ok[k])
                ptx::sts128(blk + px * 128 + ((lc ^ (px & 7)) << 4), H2 ? gn_silu8_h2_half(v[k], a, b) : gn_act8<true>(v[k], a, b));
            }
          }
          ptx::fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&slot_xf[s]);
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<1>(tmem_base, 16 * kCoE);
  }
}

}  // namespace

cudaError_t launch_conv_out_tc(const __half* x, const float2* ss, const float* w, const float* b, uint8_t* rgb,
                               int n, int H, int W, bool h2, cudaStream_t s) {
  if (!ensure_smem_attr(reinterpret_cast<const void*>(conv_out_tc_kernel<true>), kCoSmem) ||
      !ensure_smem_attr(reinterpret_cast<const void*>(conv_out_tc_kernel<false>), kCoSmem))
    return cudaErrorNotSupported;
  if (n <= 0 || W % 128 || H < 1) return cudaErrorInvalidValue;
  CUtensorMap tm;
  const uint64_t dims[4] = {128, (uint64_t)W, (uint64_t)H, (uint64_t)n};
  const uint64_t strides[3] = {128 * 2, (uint64_t)W * 128 * 2, (uint64_t)H * W * 128 * 2};
  const uint32_t box[4] = {64, 130, 1, 1};
  if (!make_tensor_map_f16(&tm, x, 4, dims, strides, box)) return cudaErrorInvalidValue;
  CoParams p;
  p.ss = ss; p.w = w; p.bias = b; p.rgb = rgb;
  p.n = n; p.H = H; p.W = W;
  p.strips = W / 128;
  // band height: the largest R (<= 32, dividing H) that still gives >= 4 work items per SM
  const int sms = num_sms();
  int R = 32;
  while (R > 4 && (H % R || (long long)n * p.strips * (H / R) < 4LL * sms)) R >>= 1;
  if (H % R) R = 1;
  p.R = R;
  p.bands = H / R;
  p.items = n * p.strips * p.bands;
  const int grid = p.items < sms ? p.items : sms;
  if (h2) conv_out_tc_kernel<true><<<grid, kCoThreads, kCoSmem, s>>>(tm, p);
  else conv_out_tc_kernel<false><<<grid, kCoThreads, kCoSmem, s>>>(tm, p);
  return cudaGetLastError();
}

}  // namespace lbx
