// Mid-block attention without the L x L score tensor: O = softmax(Q K^T / sqrt(d)) V,
// d = 512, one head, per image; Q, K, V are column blocks of the QKV GEMM output [n][L][1536].
//
// d = 512 is what makes a one-CTA flash kernel impossible on B200: the fp32 O accumulator of 128
// query rows is 128 x 512 x 4 B = all 512 TMEM columns, leaving nothing for S.  So a CTA PAIR (a
// 2-CTA cluster) owns 128 queries and splits d: CTA r holds Q[:, 256r : 256r+256] and accumulates
// O[:, 256r : 256r+256] (256 TMEM columns) next to a double-buffered S block (2 x 128 columns).
// For every 128-key block:
//   S_r = Q_r K_r^T        partial scores over CTA r's half of d (16 tcgen05.mma, M=N=128, K=16)
//   exchange (DSMEM)       CTA r keeps the columns of "its" 64 keys and sends the other 64 to the
//                          peer; both add the peer's partial -> full scores for 64 keys each
//   row max (DSMEM)        the two halves' maxima are swapped, so both CTAs use the same running
//                          max (lazy rescale: only when the max grows by > 2^8; O rescaled in TMEM)
//   P = exp2(c (S - m))    fp16, written into the A-operand layout of BOTH CTAs' P buffers
//   O_r += P V_r           32 tcgen05.mma (M=128, N=64, K=16), V read in place as MN-major B
// and at the end O_r / (l_0 + l_1) -> fp16.  FLOPs are exactly those of the two GEMMs; the L x L
// scores never leave the SMs.
//
// Warps (per CTA): 0 Q/K producer (TMA), 1 MMA issuer (one thread), 2..5 softmax + epilogue (one
// query row per thread), 6 V producer (TMA).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "gemm_tc.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace lbx {

namespace {

constexpr int kFaThreads = 224;
constexpr int kQBytes = 4 * 16384;   // 4 d-chunks of 128 rows x 64 d (K-major SW128)
constexpr int kKSt = 3;              // K ring: chunks of 128 keys x 64 d
constexpr int kVSt = 2;              // V ring: chunks of 128 keys x 64 d (MN-major SW128)
constexpr int kChunk = 16384;
constexpr int kPBytes = 2 * 16384;   // P: 128 rows x 128 keys fp16, two 64-key k-blocks
constexpr int kXBytes = 128 * 64 * 4;  // partial scores from the peer: 128 rows x 64 fp32
constexpr uint32_t kIdescS = ptx::idesc_f16(128, 128);
constexpr uint32_t kIdescPV = ptx::idesc_f16(128, 64) | (1u << 16);  // B (V) MN-major
constexpr float kRescale = 8.0f;     // lazy rescale threshold, log2 units

struct FaParams {
  int n, L;
  int nkb;         // L / 128 key blocks
  int items;       // n * L / 128 query blocks
  __half* out;     // [n][L][512]
  float c;         // log2(e) / sqrt(d)
};

struct FaSmem {
  uint8_t* q;
  uint8_t* k;
  uint8_t* v;
  uint8_t* p;
  float* x;
  float* mx;   // [2][128]
  float* lp;   // [128]
};

__device__ __forceinline__ void mma_commit_both(uint64_t* bar) {  // arrive on `bar` in both CTAs
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          ptx::smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared::cluster.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_cluster() {
  asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void __launch_bounds__(kFaThreads, 1)
    attn_fa_kernel(const __grid_constant__ CUtensorMap tmQK, const __grid_constant__ CUtensorMap tmV, const FaParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  FaSmem sm;
  sm.q = base;
  sm.k = sm.q + kQBytes;
  sm.v = sm.k + kKSt * kChunk;
  sm.p = sm.v + kVSt * kChunk;
  sm.x = reinterpret_cast<float*>(sm.p + kPBytes);
  sm.mx = sm.x + 128 * 64;
  sm.lp = sm.mx + 256;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm.lp + 128);
  uint64_t* q_full = bars;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;             // [kKSt]
  uint64_t* k_empty = k_full + kKSt;       // [kKSt]
  uint64_t* v_full = k_empty + kKSt;       // [kVSt]
  uint64_t* v_empty = v_full + kVSt;       // [kVSt]
  uint64_t* s_full = v_empty + kVSt;       // [2]
  uint64_t* s_empty = s_full + 2;          // [2]
  uint64_t* x_full = s_empty + 2;          // peer's partial scores landed in my x
  uint64_t* x_free = x_full + 1;           // the peer has read its x: I may write it again
  uint64_t* mx_full = x_free + 1;          // [2] peer's row maxima landed
  uint64_t* p_full = mx_full + 2;          // both halves of P written (4 local + 4 remote warps)
  uint64_t* p_empty = p_full + 1;          // both CTAs' P.V of the previous block done
  uint64_t* l_full = p_empty + 1;          // peer's row sums landed
  uint64_t* o_full = l_full + 1;           // last P.V of the item done
  uint64_t* o_empty = o_full + 1;          // O drained by the epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 1);

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  const uint32_t rank = ptx::cluster_ctarank(), peer = rank ^ 1u;
  const int cluster_id = blockIdx.x >> 1, nclusters = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&tmQK);
    ptx::tma_prefetch(&tmV);
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(q_empty, 1);
    for (int i = 0; i < kKSt; ++i) { ptx::mbar_init(&k_full[i], 1); ptx::mbar_init(&k_empty[i], 1); }
    for (int i = 0; i < kVSt; ++i) { ptx::mbar_init(&v_full[i], 1); ptx::mbar_init(&v_empty[i], 1); }
    // barriers that peer threads arrive on count every thread (each arrive releases its own DSMEM stores)
    for (int i = 0; i < 2; ++i) { ptx::mbar_init(&s_full[i], 1); ptx::mbar_init(&s_empty[i], 4); ptx::mbar_init(&mx_full[i], 128); }
    ptx::mbar_init(x_full, 128);
    ptx::mbar_init(x_free, 128);
    ptx::mbar_init(p_full, 256);
    ptx::mbar_init(p_empty, 2);
    ptx::mbar_init(l_full, 128);
    ptx::mbar_init(o_full, 1);
    ptx::mbar_init(o_empty, 4);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<1>(tmem_slot, 512);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nkb = p.nkb;

  if (warp == 0) {
    // ------------------------------------------------------------------ Q / K producer
    if (ptx::elect_one()) {
      uint32_t ks = 0, kph = 0, qph = 0;
      for (int it = cluster_id; it < p.items; it += nclusters) {
        const int img = it / (p.L / 128), q0 = (it % (p.L / 128)) * 128;
        const int row0 = img * p.L;
        ptx::mbar_wait(q_empty, qph ^ 1);
        ptx::mbar_arrive_expect_tx(q_full, kQBytes);
        for (int dc = 0; dc < 4; ++dc)
          ptx::tma_load_2d(&tmQK, q_full, sm.q + dc * kChunk, 256 * rank + 64 * dc, row0 + q0);
        qph ^= 1;
        for (int kb = 0; kb < nkb; ++kb)
          for (int dc = 0; dc < 4; ++dc) {
            ptx::mbar_wait(&k_empty[ks], kph ^ 1);
            ptx::mbar_arrive_expect_tx(&k_full[ks], kChunk);
            ptx::tma_load_2d(&tmQK, &k_full[ks], sm.k + ks * kChunk, 512 + 256 * rank + 64 * dc, row0 + kb * 128);
            if (++ks == kKSt) { ks = 0; kph ^= 1; }
          }
      }
    }
  } else if (warp == 6) {
    // ------------------------------------------------------------------ V producer
    if (ptx::elect_one()) {
      uint32_t vs = 0, vph = 0;
      for (int it = cluster_id; it < p.items; it += nclusters) {
        const int row0 = (it / (p.L / 128)) * p.L;
        for (int kb = 0; kb < nkb; ++kb)
          for (int dc = 0; dc < 4; ++dc) {
            ptx::mbar_wait(&v_empty[vs], vph ^ 1);
            ptx::mbar_arrive_expect_tx(&v_full[vs], kChunk);
            for (int h = 0; h < 2; ++h)  // two 64-key boxes -> 16 consecutive 8-row K groups
              ptx::tma_load_2d(&tmV, &v_full[vs], sm.v + vs * kChunk + h * 8192, 1024 + 256 * rank + 64 * dc,
                               row0 + kb * 128 + 64 * h);
            if (++vs == kVSt) { vs = 0; vph ^= 1; }
          }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (one thread)
    if (ptx::elect_one()) {
      uint32_t ks = 0, kph = 0, vs = 0, vph = 0, qph = 0, oph = 0;
      uint32_t sfill = 0;   // S blocks issued (buffer = sfill & 1)
      uint32_t pcount = 0;  // P blocks consumed
      const uint64_t q_desc0 = ptx::sdesc_k_sw128(ptx::smem_u32(sm.q));
      const uint64_t k_desc0 = ptx::sdesc_k_sw128(ptx::smem_u32(sm.k));
      const uint64_t p_desc0 = ptx::sdesc_k_sw128(ptx::smem_u32(sm.p));
      const uint64_t v_desc0 = ptx::sdesc_mn_sw128(ptx::smem_u32(sm.v), 8192, 1024);
      auto issue_s = [&]() {
        const uint32_t buf = sfill & 1;
        ptx::mbar_wait(&s_empty[buf], ((sfill >> 1) & 1) ^ 1);
        ptx::tc_fence_after();
        for (int dc = 0; dc < 4; ++dc) {
          ptx::mbar_wait(&k_full[ks], kph);
          ptx::tc_fence_after();
          const uint64_t qd = q_desc0 + (uint64_t)((dc * kChunk) >> 4);
          const uint64_t kd = k_desc0 + (uint64_t)((ks * kChunk) >> 4);
#pragma unroll
          for (int k = 0; k < 4; ++k) ptx::mma_f16_ss<1>(tmem + buf * 128, qd + 2 * k, kd + 2 * k, kIdescS, (dc | k) != 0);
          ptx::mma_commit<1>(&k_empty[ks]);
          if (++ks == kKSt) { ks = 0; kph ^= 1; }
        }
        ptx::mma_commit<1>(&s_full[buf]);
        ++sfill;
      };
      for (int it = cluster_id; it < p.items; it += nclusters) {
        ptx::mbar_wait(q_full, qph);
        qph ^= 1;
        issue_s();
        if (nkb > 1) issue_s();
        ptx::mbar_wait(o_empty, oph ^ 1);  // the previous item's O has been drained
        oph ^= 1;
        for (int kb = 0; kb < nkb; ++kb) {
          ptx::mbar_wait_cluster(p_full, pcount & 1);
          ptx::tc_fence_after();
          for (int dc = 0; dc < 4; ++dc) {
            ptx::mbar_wait(&v_full[vs], vph);
            ptx::tc_fence_after();
            const uint64_t vd = v_desc0 + (uint64_t)((vs * kChunk) >> 4);
#pragma unroll
            for (int j = 0; j < 8; ++j)  // K = 128 keys: k-block j/4 of P, +32 B per K16 inside it
              ptx::mma_f16_ss<1>(tmem + 256 + dc * 64, p_desc0 + (uint64_t)((j >> 2) * (16384 >> 4)) + 2 * (j & 3),
                                 vd + (uint64_t)(j * (2048 >> 4)), kIdescPV, (kb | j) != 0);
            ptx::mma_commit<1>(&v_empty[vs]);
            if (++vs == kVSt) { vs = 0; vph ^= 1; }
          }
          mma_commit_both(p_empty);  // this CTA's read of both P buffers' halves is done
          ++pcount;
          if (kb + 2 < nkb) issue_s();
        }
        ptx::mma_commit<1>(o_full);
        ptx::mma_commit<1>(q_empty);
      }
    }
  } else {
    // ------------------------------------------------------------------ softmax + epilogue (warps 2..5)
    const uint32_t qw = warp & 3;
    const int row = (int)(qw * 32 + lane);
    const uint32_t t_row = tmem + ((qw * 32u) << 16);
    const uint32_t x_peer = ptx::mapa(ptx::smem_u32(sm.x), peer) + row * 256;
    const uint32_t mx_peer = ptx::mapa(ptx::smem_u32(sm.mx), peer);
    const uint32_t lp_peer = ptx::mapa(ptx::smem_u32(sm.lp), peer);
    const uint32_t p_loc = ptx::smem_u32(sm.p) + rank * 16384 + row * 128;  // k-block `rank` = my 64 keys
    const uint32_t p_rem = ptx::mapa(p_loc, peer);
    uint32_t scount = 0, xcount = 0, pcount = 0, ocount = 0, mcount = 0;
    for (int it = cluster_id; it < p.items; it += nclusters) {
      const int img = it / (p.L / 128), q0 = (it % (p.L / 128)) * 128;
      float m_used = -INFINITY, l_mine = 0.f;
      for (int kb = 0; kb < nkb; ++kb) {
        const uint32_t buf = scount & 1;
        ptx::mbar_wait(&s_full[buf], (scount >> 1) & 1);
        ptx::tc_fence_after();
        // partial scores of this row: keys 0..63 (half 0) and 64..127 (half 1)
        uint32_t mine[64], send[32];
        ptx::tmem_ld32(t_row + buf * 128 + rank * 64, *reinterpret_cast<uint32_t(*)[32]>(mine));
        ptx::tmem_ld32(t_row + buf * 128 + rank * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(mine + 32));
        ptx::tmem_ld_wait();
        // the peer's 64 keys, sent in two 32-column pieces
        ptx::mbar_wait(x_free, (xcount & 1) ^ 1);
        for (int piece = 0; piece < 2; ++piece) {
          ptx::tmem_ld32(t_row + buf * 128 + peer * 64 + piece * 32, send);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 8; ++i)
            st_cluster_v4(x_peer + piece * 128 + i * 16, make_uint4(send[4 * i], send[4 * i + 1], send[4 * i + 2], send[4 * i + 3]));
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&s_empty[buf]);
        ptx::mbar_arrive_cluster(x_full, peer);  // release.cluster: this thread's DSMEM writes first
        ++scount;
        // the peer's partials for my keys
        ptx::mbar_wait_cluster(x_full, xcount & 1);
        float s[64];
        const float4* xr = reinterpret_cast<const float4*>(sm.x + row * 64);
        float mx = -INFINITY;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float4 v = xr[i];
          s[4 * i] = __uint_as_float(mine[4 * i]) + v.x;
          s[4 * i + 1] = __uint_as_float(mine[4 * i + 1]) + v.y;
          s[4 * i + 2] = __uint_as_float(mine[4 * i + 2]) + v.z;
          s[4 * i + 3] = __uint_as_float(mine[4 * i + 3]) + v.w;
          mx = fmaxf(mx, fmaxf(fmaxf(s[4 * i], s[4 * i + 1]), fmaxf(s[4 * i + 2], s[4 * i + 3])));
        }
        ptx::mbar_arrive_cluster(x_free, peer);  // my x may be overwritten
        ++xcount;
        // agree on the row max with the peer
        const uint32_t mb = mcount & 1;
        st_cluster_f32(mx_peer + (mb * 128 + row) * 4, mx);
        ptx::mbar_arrive_cluster(&mx_full[mb], peer);
        ptx::mbar_wait_cluster(&mx_full[mb], (mcount >> 1) & 1);
        ++mcount;
        const float m_blk = fmaxf(mx, sm.mx[mb * 128 + row]) * p.c;
        // both CTAs wait for both P.V of the previous block before touching O or either P buffer
        ptx::mbar_wait_cluster(p_empty, (pcount & 1) ^ 1);
        ptx::tc_fence_after();
        // lazy rescale, decided per row; the TMEM accesses are warp-collective (.sync.aligned), so a
        // warp rescales when any of its rows must (factor 1 for the others)
        float f = 1.f;
        if (m_blk > m_used + kRescale || m_used == -INFINITY) {
          if (m_used != -INFINITY) f = ex2(m_used - m_blk);
          m_used = m_blk;
        }
        if (__any_sync(0xffffffffu, f != 1.f)) {
          l_mine *= f;
          for (int cc = 0; cc < 8; ++cc) {
            uint32_t o[32];
            ptx::tmem_ld32(t_row + 256 + cc * 32, o);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
            ptx::tmem_st32(t_row + 256 + cc * 32, o);
          }
          ptx::tmem_st_wait();
        }
        // P = exp2(c s - m_used) in fp16, the sum of the rounded values
        uint4 pk[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          uint32_t w[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const __half2 h = __floats2half2_rn(ex2(fmaf(s[8 * i + 2 * k], p.c, -m_used)),
                                                ex2(fmaf(s[8 * i + 2 * k + 1], p.c, -m_used)));
            const float2 f = __half22float2(h);
            l_mine += f.x + f.y;
            w[k] = *reinterpret_cast<const uint32_t*>(&h);
          }
          pk[i] = make_uint4(w[0], w[1], w[2], w[3]);
        }
        // row `row`, keys of k-block `rank`: 8 chunks of 16 B, 128B-swizzled
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t off = (uint32_t)((i ^ (row & 7)) << 4);
          ptx::sts128(p_loc + off, pk[i]);
          st_cluster_v4(p_rem + off, pk[i]);
        }
        fence_proxy_async_cluster();  // generic-proxy P writes (local and remote) -> the tensor cores
        ptx::mbar_arrive_cluster(p_full, rank);
        ptx::mbar_arrive_cluster(p_full, peer);
        ++pcount;
      }
      // ---- epilogue: O_r / (l_0 + l_1) -> fp16
      st_cluster_f32(lp_peer + row * 4, l_mine);
      ptx::mbar_arrive_cluster(l_full, peer);
      ptx::mbar_wait_cluster(l_full, ocount & 1);
      const float inv = 1.0f / (l_mine + sm.lp[row]);
      ptx::mbar_wait(o_full, ocount & 1);
      ptx::tc_fence_after();
      __half* orow = p.out + ((size_t)img * p.L + q0 + row) * 512 + 256 * rank;
      for (int cc = 0; cc < 8; ++cc) {
        uint32_t o[32];
        ptx::tmem_ld32(t_row + 256 + cc * 32, o);
        ptx::tmem_ld_wait();
        uint32_t w[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const __half2 h = __floats2half2_rn(__uint_as_float(o[2 * i]) * inv, __uint_as_float(o[2 * i + 1]) * inv);
          w[i] = *reinterpret_cast<const uint32_t*>(&h);
        }
        uint4* dst = reinterpret_cast<uint4*>(orow + cc * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i) dst[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(o_empty);
      ++ocount;
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<1>(tmem, 512);
  }
}

}  // namespace

cudaError_t launch_attn_fa(const __half* qkv, __half* out, int n, int L, cudaStream_t s) {
  constexpr int smem = 1024 + kQBytes + (kKSt + kVSt) * kChunk + kPBytes + kXBytes + 256 * 4 + 128 * 4 + 256;
  if (!ensure_smem_attr(reinterpret_cast<const void*>(attn_fa_kernel), smem)) return cudaErrorNotSupported;
  if (n <= 0 || L % 128) return cudaErrorInvalidValue;
  CUtensorMap tmQK, tmV;
  const uint64_t dims[2] = {1536, (uint64_t)n * L};
  const uint64_t strides[1] = {1536 * 2};
  const uint32_t boxQK[2] = {64, 128}, boxV[2] = {64, 64};
  if (!make_tensor_map_f16(&tmQK, qkv, 2, dims, strides, boxQK) || !make_tensor_map_f16(&tmV, qkv, 2, dims, strides, boxV))
    return cudaErrorInvalidValue;
  FaParams p;
  p.n = n;
  p.L = L;
  p.nkb = L / 128;
  p.items = n * L / 128;
  p.out = out;
  p.c = 1.4426950408889634f / sqrtf(512.f);
  const int clusters = num_sms() / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * (p.items < clusters ? p.items : clusters));
  cfg.blockDim = dim3(kFaThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr1[1];
  attr1[0].id = cudaLaunchAttributeClusterDimension;
  attr1[0].val.clusterDim.x = 2;
  attr1[0].val.clusterDim.y = 1;
  attr1[0].val.clusterDim.z = 1;
  cfg.attrs = attr1;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, attn_fa_kernel, tmQK, tmV, p);
}

}  // namespace lbx
