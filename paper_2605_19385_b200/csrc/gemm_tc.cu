// tcgen05 implicit-GEMM for the VAE decoder's dense contractions:
//   conv3x3 (pad 1, NHWC), conv1x1 / linear (plain GEMM), and nearest-2x upsample fused with the
//   following conv3x3 as four 2x2 sub-pixel convolutions (GEMM_SUBPIX; 4/9 of the FLOPs).
//
// Structure (persistent, warp-specialised, one CTA or one CTA pair per tile):
//   warp 0      TMA producer: A tile (128 pixels x 64 channels, tap-shifted box; TMA OOB zero-fill
//               provides the conv halo) + B tile (weights) into a STAGES-deep smem ring.
//   warp 1      TMEM allocator; in the leader CTA one elected lane issues tcgen05.mma
//               (M = 128*CG, N = BN, K = 16 per instruction) into a double-buffered TMEM accumulator.
//   warps 2..5  epilogue: tcgen05.ld -> alpha/row-scale/bias/residual in fp32 -> fp16 store, plus
//               GroupNorm-32 partial sums of the stored values (fp64 atomics) for the next norm.
// CG = 2 runs the tile on a CTA pair (cta_group::2): each CTA stages half of A (its 128 rows) and
// half of B (BN/2 rows); the leader's MMA reads both halves, halving smem operand traffic per SM.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <mutex>

#include "gemm_tc.cuh"
#include "ptx.cuh"

namespace lbx {

struct KParams {
  int mode;
  int M, N, K;
  int num_kb;          // K / 64
  int cblocks;         // conv: C / 64
  int H, W, Wt, Ht;    // conv geometry (A box = 64 x Wt x Ht x 1)
  int m_tiles, n_tiles, tiles;
  __half* out;
  int ldo;
  const float* bias;
  const __half* resid;
  int ldr;
  const float* row_scale;
  float alpha;
  double* gn_stats;
  int gn_cpg;
  int rows_per_img;
};

template <int BN, int CG>
struct Cfg {
  static constexpr int BM_CTA = 128;                 // A rows per CTA
  static constexpr int BK = 64;                      // 128 bytes of fp16 (one SW128 row)
  static constexpr int A_BYTES = BM_CTA * BK * 2;    // 16 KiB
  static constexpr int B_ROWS = BN / CG;             // B rows staged per CTA
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 8 ? 8 : (200 * 1024) / STAGE_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;           // double-buffered fp32 accumulator
  static constexpr int SMEM_BYTES = 1024 /*align slack*/ + STAGES * STAGE_BYTES + 256;
  static constexpr int THREADS = 320;  // 2 non-epilogue + 8 epilogue warps
  static constexpr uint32_t IDESC = ptx::idesc_f16(128 * CG, BN);
  static constexpr uint32_t TX_BYTES = CG * STAGE_BYTES;  // bytes landing per stage per tile (pair)
};

__device__ __forceinline__ void tile_coords(const KParams& p, int t, int& m_tile, int& n_tile, int& phase) {
  n_tile = t % p.n_tiles;
  int r = t / p.n_tiles;
  if (p.mode == GEMM_SUBPIX) {
    phase = r & 3;
    m_tile = r >> 2;
  } else {
    phase = 0;
    m_tile = r;
  }
}

// Per-chunk GroupNorm partials.  pk holds this lane's 32 stored fp16 values (one pixel, 32
// consecutive channels) as half2 pairs.  NV = 2 * groups-per-chunk values per lane (group sums,
// then group sums of squares) are reduce-scattered across the warp with NV + log2(32/NV)
// shuffles (instead of 5 * NV for a butterfly per value): lane L ends up owning the warp total
// of value index (L >> (5 - log2 NV)) & (NV - 1).
template <int NV>
__device__ __forceinline__ float chunk_group_stats(const uint32_t (&pk)[16], uint32_t lane) {
  constexpr int G = NV / 2, H2 = 16 / G;  // half2 words per group
  constexpr int LG = NV == 16 ? 4 : (NV == 8 ? 3 : 2);
  float v[NV];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    float s = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < H2; ++i) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&pk[g * H2 + i]));
      s += f.x + f.y;
      s2 = fmaf(f.x, f.x, fmaf(f.y, f.y, s2));
    }
    v[g] = s;
    v[G + g] = s2;
  }
#pragma unroll
  for (int lvl = 0; lvl < LG; ++lvl) {
    const int cnt = NV >> lvl;
    const int o = 16 >> lvl;
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < cnt / 2; ++i) {
      const float send = upper ? v[i] : v[i + cnt / 2];
      const float keep = upper ? v[i + cnt / 2] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  float x = v[0];
#pragma unroll
  for (int o = 16 >> LG; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

template <int BN, int CG>
__global__ void __launch_bounds__(320, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const KParams p) {
  using C = Cfg<BN, CG>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = ptx::warp_id();
  const uint32_t lane = ptx::lane_id();
  const uint32_t rank = (CG == 2) ? ptx::cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x / CG;
  const int nclusters = gridDim.x / CG;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&tmA);
    ptx::tma_prefetch(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], 8 * CG);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<CG>(tmem_slot, C::TMEM_COLS);
  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (ptx::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cluster_id; t < p.tiles; t += nclusters) {
        int m_tile, n_tile, ph;
        tile_coords(p, t, m_tile, n_tile, ph);
        const int m0 = m_tile * (128 * CG) + rank * 128;  // this CTA's first A row
        int img = 0, y0 = 0, x0 = 0;
        if (p.mode != GEMM_PLAIN) {
          const int hw = p.H * p.W;
          img = m0 / hw;
          const int rem = m0 - img * hw;
          y0 = rem / p.W;
          x0 = rem - y0 * p.W;
        }
        const int b_row = (p.mode == GEMM_SUBPIX ? ph * p.N : 0) + n_tile * BN + rank * C::B_ROWS;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* a_dst = sA + stage * C::A_BYTES;
          uint8_t* b_dst = sB + stage * C::B_BYTES;
          if (leader) ptx::mbar_arrive_expect_tx(&full[stage], C::TX_BYTES);
          if (p.mode == GEMM_PLAIN) {
            if constexpr (CG == 1) ptx::tma_load_2d(&tmA, &full[stage], a_dst, kb * 64, m0);
            else ptx::tma_load_2d_pair(&tmA, &full[stage], a_dst, kb * 64, m0);
          } else {
            const int tap = kb / p.cblocks;
            const int cb = kb - tap * p.cblocks;
            int dx, dy;
            if (p.mode == GEMM_CONV3X3) {
              dy = tap / 3 - 1;
              dx = tap % 3 - 1;
            } else {  // sub-pixel phase (a, b) = (ph >> 1, ph & 1): low-res offsets r + a - 1
              dy = (tap >> 1) + (ph >> 1) - 1;
              dx = (tap & 1) + (ph & 1) - 1;
            }
            if constexpr (CG == 1) ptx::tma_load_4d(&tmA, &full[stage], a_dst, cb * 64, x0 + dx, y0 + dy, img);
            else ptx::tma_load_4d_pair(&tmA, &full[stage], a_dst, cb * 64, x0 + dx, y0 + dy, img);
          }
          if constexpr (CG == 1) ptx::tma_load_2d(&tmB, &full[stage], b_dst, kb * 64, b_row);
          else ptx::tma_load_2d_pair(&tmB, &full[stage], b_dst, kb * 64, b_row);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA)
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = cluster_id; t < p.tiles; t += nclusters) {
        ptx::mbar_wait_cluster(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          if (ptx::elect_one()) {
            const uint64_t a_desc = ptx::sdesc_k_sw128(ptx::smem_u32(sA + stage * C::A_BYTES));
            const uint64_t b_desc = ptx::sdesc_k_sw128(ptx::smem_u32(sB + stage * C::B_BYTES));
#pragma unroll
            for (int k = 0; k < 4; ++k)  // 4 x K16 per 64-wide k-block; +32 B per step inside the swizzle atom
              ptx::mma_f16_ss<CG>(d_tmem, a_desc + 2 * k, b_desc + 2 * k, C::IDESC, (kb | k) != 0);
            ptx::mma_commit<CG>(&empty[stage]);
            if (kb == p.num_kb - 1) ptx::mma_commit<CG>(&tfull[acc]);
          }
          __syncwarp();
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..9)
    // Two warps per TMEM lane quarter; warp half `hsel` takes the even/odd 32-column chunks.
    const uint32_t q = warp & 3;
    const int hsel = (int)(warp - 2) >> 2;
    const int row = q * 32 + lane;
    constexpr int NCH = BN / 64;  // chunks per warp per tile
    // GroupNorm partials: after the per-chunk reduce-scatter each lane owns one (group, sum|sumsq)
    // value per chunk; lanes accumulate those across tiles in fp64 registers and flush with one
    // atomic per owned value only when the (image, n-tile) changes -- not once per tile.
    double gacc[NCH];
#pragma unroll
    for (int j = 0; j < NCH; ++j) gacc[j] = 0.0;
    int g_img = -1, g_ntile = -1;
    const int nv = p.gn_stats ? 64 / p.gn_cpg : 0;  // values per chunk: 2 * groups-per-chunk
    const int lg = nv == 16 ? 4 : (nv == 8 ? 3 : 2);
    const int own = nv ? (int)(lane >> (5 - lg)) & (nv - 1) : 0;
    const bool rep = nv ? (lane & ((1u << (5 - lg)) - 1u)) == 0 : false;
    auto flush = [&]() {
      if (g_img < 0) return;
      if (rep) {
        const int gpc = nv >> 1;  // groups per chunk
        const int kind = own >= gpc;
        const int g_in = own - kind * gpc;
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          const int c = hsel + 2 * j;
          const int grp = (g_ntile * BN + c * 32) / p.gn_cpg + g_in;
          atomicAdd(p.gn_stats + ((size_t)g_img * 32 + grp) * 2 + kind, gacc[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < NCH; ++j) gacc[j] = 0.0;
    };
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = cluster_id; t < p.tiles; t += nclusters) {
      int m_tile, n_tile, ph;
      tile_coords(p, t, m_tile, n_tile, ph);
      const int m = m_tile * (128 * CG) + rank * 128 + row;
      const int n0 = n_tile * BN;
      long long orow = m;
      if (p.mode == GEMM_SUBPIX) {
        const int hw = p.H * p.W;
        const int img = m / hw;
        const int rem = m - img * hw;
        const int i = rem / p.W, j = rem - (rem / p.W) * p.W;
        orow = ((long long)img * (2 * p.H) + (2 * i + (ph >> 1))) * (2 * p.W) + (2 * j + (ph & 1));
      }
      const float rs = p.alpha * (p.row_scale ? p.row_scale[m] : 1.f);
      if (p.gn_stats) {
        const int img = m / p.rows_per_img;  // warp-uniform: 32-row slices never straddle images
        if (img != g_img || n_tile != g_ntile) {
          flush();
          g_img = img;
          g_ntile = n_tile;
        }
      }

      // residual prefetch ring, two chunks deep, issued before waiting for the accumulator
      constexpr int PF = NCH < 2 ? NCH : 2;
      uint4 rr[PF][4];
      const __half* rbase = p.resid ? p.resid + orow * p.ldr + n0 + hsel * 32 : nullptr;
      if (p.resid) {
#pragma unroll
        for (int j = 0; j < PF; ++j)
#pragma unroll
          for (int i = 0; i < 4; ++i) rr[j][i] = __ldg(reinterpret_cast<const uint4*>(rbase + j * 64) + i);
      }
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const uint32_t t_row = tmem_base + ((q * 32u) << 16) + acc * BN;
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        const int c = hsel + 2 * j;
        const int n = n0 + c * 32;
        uint32_t r[32];
        ptx::tmem_ld32(t_row + c * 32, r);
        ptx::tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * rs;
        if (p.bias) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 b = __ldg(reinterpret_cast<const float4*>(p.bias + n + i));
            v[i] += b.x; v[i + 1] += b.y; v[i + 2] += b.z; v[i + 3] += b.w;
          }
        }
        if (p.resid) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint4 q4 = rr[j % PF][i];
            const uint32_t w4[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w4[k]));
              v[i * 8 + 2 * k] += f.x;
              v[i * 8 + 2 * k + 1] += f.y;
            }
          }
          if (j + PF < NCH) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              rr[j % PF][i] = __ldg(reinterpret_cast<const uint4*>(rbase + (j + PF) * 64) + i);
          }
        }
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const __half2 h = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
          pk[i] = *reinterpret_cast<const uint32_t*>(&h);
        }
        uint4* op = reinterpret_cast<uint4*>(p.out + orow * p.ldo + n);
#pragma unroll
        for (int i = 0; i < 4; ++i) op[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
        if (p.gn_stats) {
          float val;
          if (nv == 16) val = chunk_group_stats<16>(pk, lane);
          else if (nv == 8) val = chunk_group_stats<8>(pk, lane);
          else val = chunk_group_stats<4>(pk, lane);
          gacc[j] += (double)val;
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 1) ptx::mbar_arrive_relaxed(&tempty[acc]);
        else ptx::mbar_arrive_cluster_relaxed(&tempty[acc], 0);
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (p.gn_stats) flush();
  }

  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<CG>(tmem_base, C::TMEM_COLS);
  }
}

// ======================================================================= host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}

bool tma_available() { return get_encode() != nullptr; }

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static bool make_map(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                     const cuuint32_t* box) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, rank, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, int CG>
static cudaError_t launch_cfg(const GemmArgs& a, const KParams& kp, cudaStream_t stream) {
  using Cf = Cfg<BN, CG>;
  CUtensorMap tmA, tmB;
  if (a.mode == GEMM_PLAIN) {
    cuuint64_t dims[2] = {(cuuint64_t)a.K, (cuuint64_t)a.M};
    cuuint64_t strides[1] = {(cuuint64_t)a.lda * 2};
    cuuint32_t box[2] = {64, 128};
    if (!make_map(&tmA, a.A, 2, dims, strides, box)) return cudaErrorInvalidValue;
  } else {
    cuuint64_t dims[4] = {(cuuint64_t)a.C, (cuuint64_t)a.W, (cuuint64_t)a.H, (cuuint64_t)a.B_img};
    cuuint64_t strides[3] = {(cuuint64_t)a.C * 2, (cuuint64_t)a.W * a.C * 2, (cuuint64_t)a.H * a.W * a.C * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)kp.Wt, (cuuint32_t)kp.Ht, 1};
    if (!make_map(&tmA, a.A, 4, dims, strides, box)) return cudaErrorInvalidValue;
  }
  {
    const int brows = a.mode == GEMM_SUBPIX ? 4 * a.N : a.N;
    cuuint64_t dims[2] = {(cuuint64_t)a.K, (cuuint64_t)brows};
    cuuint64_t strides[1] = {(cuuint64_t)a.ldb * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)Cf::B_ROWS};
    if (!make_map(&tmB, a.Bw, 2, dims, strides, box)) return cudaErrorInvalidValue;
  }
  auto kern = gemm_tc_kernel<BN, CG>;
  const int sms = num_sms();
  int clusters = sms / CG;
  if (clusters > kp.tiles) clusters = kp.tiles;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(clusters * CG);
  cfg.blockDim = dim3(Cf::THREADS);
  cfg.dynamicSmemBytes = Cf::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, tmA, tmB, kp);
}

template <int BN, int CG>
static bool set_attr() {
  return cudaFuncSetAttribute(gemm_tc_kernel<BN, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              Cfg<BN, CG>::SMEM_BYTES) == cudaSuccess;
}

bool gemm_tc_prepare() {
  static int ok = -1;
  static std::mutex mu;
  std::lock_guard<std::mutex> g(mu);
  if (ok < 0) {
    ok = tma_available() && set_attr<256, 2>() && set_attr<128, 2>() && set_attr<256, 1>() && set_attr<128, 1>();
    num_sms();
  }
  return ok == 1;
}

cudaError_t gemm_tc_launch(const GemmArgs& a, cudaStream_t stream, int force_cg, int force_bn) {
  if (!gemm_tc_prepare()) return cudaErrorNotSupported;
  if (a.M <= 0 || a.N <= 0 || a.K <= 0 || a.K % 64) return cudaErrorInvalidValue;
  KParams kp = {};
  kp.mode = a.mode;
  kp.M = a.M; kp.N = a.N; kp.K = a.K;
  kp.num_kb = a.K / 64;
  if (a.mode != GEMM_PLAIN) {
    if (a.C % 64 || a.M != a.B_img * a.H * a.W) return cudaErrorInvalidValue;
    if (a.K != (a.mode == GEMM_CONV3X3 ? 9 : 4) * a.C) return cudaErrorInvalidValue;
    kp.cblocks = a.C / 64;
    kp.H = a.H; kp.W = a.W;
    kp.Wt = a.W < 128 ? a.W : 128;
    if (128 % kp.Wt || (a.W > 128 && a.W % 128)) return cudaErrorInvalidValue;
    kp.Ht = 128 / kp.Wt;
    if (a.H % kp.Ht) return cudaErrorInvalidValue;
  }
  kp.out = a.out; kp.ldo = a.ldo; kp.bias = a.bias; kp.resid = a.resid; kp.ldr = a.ldr;
  kp.row_scale = a.row_scale; kp.alpha = a.alpha;
  kp.gn_stats = a.gn_stats; kp.gn_cpg = a.gn_cpg; kp.rows_per_img = a.rows_per_img;
  if (a.gn_stats && (!(a.gn_cpg == 4 || a.gn_cpg == 8 || a.gn_cpg == 16) || a.N != 32 * a.gn_cpg ||
                     a.rows_per_img <= 0))
    return cudaErrorInvalidValue;
  if (a.mode == GEMM_SUBPIX && a.resid) return cudaErrorInvalidValue;

  int bn = force_bn ? force_bn : (a.N % 256 == 0 ? 256 : 128);
  if (a.N % bn) return cudaErrorInvalidValue;
  int cg = force_cg ? force_cg : ((a.M % 256 == 0) ? 2 : 1);
  if (a.M % (128 * cg)) return cudaErrorInvalidValue;
  kp.m_tiles = a.M / (128 * cg);
  kp.n_tiles = a.N / bn;
  kp.tiles = kp.m_tiles * kp.n_tiles * (a.mode == GEMM_SUBPIX ? 4 : 1);
  if (bn == 256 && cg == 2) return launch_cfg<256, 2>(a, kp, stream);
  if (bn == 128 && cg == 2) return launch_cfg<128, 2>(a, kp, stream);
  if (bn == 256 && cg == 1) return launch_cfg<256, 1>(a, kp, stream);
  return launch_cfg<128, 1>(a, kp, stream);
}

}  // namespace lbx
