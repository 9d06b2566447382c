// tcgen05 implicit-GEMM for the VAE decoder's dense contractions:
//   conv3x3 (pad 1, NHWC), conv1x1 / linear (plain GEMM, B K-major or MN-major), and nearest-2x
//   upsample fused with the following conv3x3 as four 2x2 sub-pixel convolutions (GEMM_SUBPIX; 4/9
//   of the FLOPs).
//
// Structure (persistent, warp-specialised, one CTA or one CTA pair per tile):
//   warp 0      A producer (TMA): one halo box per 64-channel block that every tap reads through a
//               row-shifted UMMA descriptor (TMA OOB zero-fill is the conv padding); plain 2-D boxes
//               in GEMM mode; the extra K segment (a folded 1x1 shortcut) from a second map.
//   warp 10     B producer (TMA): weight k-blocks into their own ring.
//   warp 1      TMEM allocator; in the leader CTA ONE thread issues every tcgen05.mma
//               (M = 128*CG, N = BN, K = 16) into a double-buffered TMEM accumulator.
//   warps 2..9  epilogue, two warps per TMEM lane quarter: tcgen05.ld -> (scale) + bias (+ residual)
//               in fp32 -> fp16, stored with STG.256 (convs) or staged in smem and TMA-stored (plain
//               GEMMs); GroupNorm-32 partial sums of the fp32 values (per lane, reduced at image
//               changes, exact fixed-point integer atomics, gnfix.cuh); at 128 output channels the residual of the tile that will
//               reuse the accumulator is preloaded into it (tcgen05.st) -- wider outputs add it here.
//   warps 11..14  (XF kernels only) GroupNorm + SiLU transform of each landed A halo.
// CG = 2 runs the tile on a CTA pair (cta_group::2): each CTA stages its 128 A rows and half of B
// (BN/2 rows); the leader's MMA reads both halves.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "act.cuh"
#include "gemm_tc.cuh"
#include "gnfix.cuh"
#include "ptx.cuh"

namespace lbx {

// Division by a launch-invariant divisor without the ~20-instruction IDIV sequence: q = n / d for
// 0 <= n < 2^31 as (umulhi(n, m) + n) >> s with s = ceil(log2 d), m = 2^32 (2^s - d) / d + 1.
struct FastDiv {
  uint32_t m = 1, s = 0;
  FastDiv() = default;
  explicit FastDiv(uint32_t d) {
    while ((1u << s) < d) ++s;
    m = (uint32_t)((((1ull << 32) * ((1ull << s) - d)) / d) + 1);
  }
};
__device__ __forceinline__ int fdiv(int n, FastDiv f) { return (int)((__umulhi((uint32_t)n, f.m) + (uint32_t)n) >> f.s); }

struct KParams {
  int mode;
  int M, N, K;
  int num_kb;          // K / 64
  int cblocks;         // conv: C / 64
  int H, W, Wt, Ht;    // conv geometry (per-tap A box = 64 x Wt x Ht x 1)
  int m_tiles, n_tiles, tiles;
  __half* out;
  int ldo;
  const float* bias;
  const __half* resid;
  int ldr;
  const float* row_scale;
  float alpha;
  unsigned long long* gn_stats;
  int gn_cpg;
  int rows_per_img;
  // operand staging (host-computed, see stage_plan())
  int halo;            // 1: one halo box per C-block feeds every tap (row-shifted UMMA descriptors)
  int halo_rows;       // 3 (conv3x3) or 2 (sub-pixel)
  int taps;            // 9 (conv3x3), 4 (sub-pixel)
  int a_stage_bytes;   // smem bytes per A stage (1024-aligned)
  int a_tx_bytes;      // bytes one CTA's A load lands per stage
  int a_stages, b_stages;
  int desc_base_mode;  // descriptor base-offset convention for row-shifted views (0 or 1)
  int msub;            // 128-row M sub-tiles per CTA sharing every B tile (1 or 2)
  int vsub;            // 1: the sub-tiles are vertically adjacent image rows sharing one halo box
  int b_mn;            // 1: B is MN-major in memory ([K][N], N contiguous), staged as 64-wide N atoms
  int rpf;             // 1: the residual is preloaded into the TMEM accumulator by the epilogue warps
  int a_hint;          // 1: conv A boxes loaded with an L2 evict_last policy (LBX_A_HINT, A/B)
  int rpf_pf;          // 1: L2-prefetch the next preload's rows before waiting for the accumulator
  int sched;           // 1: each cluster takes a contiguous block of tiles (conv modes), 0: round-robin
  int pdl;             // 1: launched as a programmatic dependent (wait before any global access)
  int rres;            // 1: residual preload through per-warp smem staging (line-covering loads)
  int epi_skip;        // diagnostics (debug bit 12): the epilogue only hands buffers back (wrong results)
  int rowred;          // attention row reductions (GemmArgs::rowred)
  const float* row_max;
  float* row_part;
  int* exp_flag;
  int exp_force;       // tests: flag every group (the exact-softmax fallback always runs)
  int exp_h2;          // rowred 2: fp16 exponent, two E per MUFU op (ex2.approx.f16x2)
  const int* run_if;   // per-image guards (GemmArgs::run_if): skip the tiles of unflagged images
  int run_if_n;
  int ld_skip;         // diagnostics (bits 27 / 28): after a CTA's first tile the B / A producer only
                       // arrives on the full barrier (no TMA; stale operands, wrong results) -- the
                       // energy and time of the operand traffic
  int store_mode;      // epilogue global stores: 0 STG.128, 1 STG.256, 2 streaming STG.128
  int tstore;          // 1: epilogue stages each 32x32 chunk in smem and TMA-stores it (tmO)
  int cmap;            // epilogue column chunks per warp: 1 contiguous (hsel*NCH + j), 0 interleaved
  int batch_m, batch_b;  // batched plain GEMM: rows per image of A, B offset per image
  int halo_sub_bytes;  // smem pitch of one sub-tile's halo box (1024-aligned)
  int tmem_cols;       // 2 accumulator buffers x msub x BN (power of two <= 512)
  int n_extra;         // extra plain k-blocks from the second A operand (K2 / 64)
  const float2* gn_ss; // fused GroupNorm+SiLU on A (XF kernels): per (image, channel) (scale, shift)
  int k_main;          // K of the main segment (B columns of the extra segment start here)
  int rbuf;            // 1: the extra K segment is staged k-block by k-block in its own buffer (msub x
                       // 16 KB), each k-block's MMAs interleaved between halo taps (rbuf_at), so its
                       // loads hide behind the taps instead of taking short A-ring stages
  int r_bytes;         // smem bytes of that buffer (0 without rbuf)
  // invariant divisors of the tile / row arithmetic
  FastDiv fd_ntiles;   // t / n_tiles
  FastDiv fd_segs;     // vsub: 128*CG-pixel segments per image row (W / (128 CG))
  FastDiv fd_per_img;  // vsub: tiles per image ((H / msub) * segs)
  FastDiv fd_rpi;      // m / rows_per_img (GroupNorm image index)
  int segs, per_img;
};

constexpr int kHaloW = 130;      // 128 output pixels + 1-pixel halo on each side
constexpr int kMaxStages = 16;   // barrier array capacity per ring
constexpr int kSmemBudget = 220 * 1024;

template <int BN, int CG>
struct Cfg {
  static constexpr int B_ROWS = BN / CG;             // B rows staged per CTA
  static constexpr int B_BYTES = B_ROWS * 64 * 2;    // one 64-wide k-block
  static constexpr int SMEM_MAX = 227 * 1024;
  // warp 0 A-producer, 1 MMA, 2..9 epilogue, 10 B-producer.  XF kernels are laid out by aligned
  // warpgroups so that registers can move to the epilogue (setmaxnreg): warps 0 A-producer,
  // 1 MMA, 2 B-producer, 3 idle | 4..11 epilogue | 12..15 A transform.
  static constexpr int THREADS = 352;
  static constexpr int THREADS_XF = 512;
  static constexpr uint32_t IDESC = ptx::idesc_f16(128 * CG, BN);
};

__device__ __forceinline__ int g_store_mode_dev(const KParams& p) { return p.store_mode; }
__device__ __forceinline__ int g_rpf_l2pf_dev(const KParams& p) { return p.rpf_pf; }

__device__ __forceinline__ void tile_coords(const KParams& p, int t, int& m_tile, int& n_tile, int& phase) {
  int r = fdiv(t, p.fd_ntiles);
  n_tile = t - r * p.n_tiles;
  if (p.mode == GEMM_SUBPIX) {
    phase = r & 3;
    m_tile = r >> 2;
  } else {
    phase = 0;
    m_tile = r;
  }
}

// First A row of sub-tile `sub` of this CTA's tile.  Horizontal sub-tiles (vsub = 0): the CTA's
// rows are contiguous, m0 + 128 sub.  Vertical sub-tiles (vsub = 1, conv halo mode): the CTA owns
// 128 pixels x msub image rows and the CTA pair covers 128 CG consecutive pixels of those rows,
// so both sub-tiles' taps read one (halo_rows + 1)-row halo box.
__device__ __forceinline__ int tile_row0(const KParams& p, int m_tile, int rank, int CG, int sub) {
  if (!p.vsub) return m_tile * (128 * p.msub * CG) + rank * (128 * p.msub) + sub * 128;
  const int img = fdiv(m_tile, p.fd_per_img);
  const int r = m_tile - img * p.per_img;
  const int yp = fdiv(r, p.fd_segs);
  const int x0 = (r - yp * p.segs) * 128 * CG + rank * 128;
  return (img * p.H + yp * p.msub + sub) * p.W + x0;
}

// Guarded launches (run_if): the tile belongs to an image whose flag is clear -- every warp role
// skips it, so the tile sequences of producers, MMA issuer and epilogue stay in step.
__device__ __forceinline__ bool tile_off(const KParams& p, int t, int CG) {
  if (!p.run_if) return false;
  int m_tile, n_tile, phase;
  tile_coords(p, t, m_tile, n_tile, phase);
  const long long m0 = (long long)m_tile * (128 * p.msub * CG);
  const int img = p.batch_m ? (int)(m0 / p.batch_m) : 0;
  return reinterpret_cast<const volatile int*>(p.run_if)[img] == 0;
}

// Per-lane GroupNorm partials of one chunk: NV = 2 * (groups per chunk) values -- the group sums,
// then the group sums of squares of this lane's 32 fp32 outputs -- added to the lane's running
// accumulators a[0..NV).  The cross-lane reduction happens once per flush (warp_flush_stats), not per
// chunk: it was two thirds of the epilogue's instructions.
// Even and odd elements are summed as packed pairs (FADD2 / FFMA2) and the pair folded at the end.
template <int NV>
__device__ __forceinline__ void lane_group_stats(const float (&xs)[32], float* a) {
  constexpr int G = NV / 2, E = 32 / G;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    float2 s = make_float2(xs[g * E], xs[g * E + 1]);
    float2 s2 = fmul2(s, s);
#pragma unroll
    for (int i = 2; i < E; i += 2) {
      const float2 x = make_float2(xs[g * E + i], xs[g * E + i + 1]);
      s = fadd2(s, x);
      s2 = ffma2(x, x, s2);
    }
    a[g] += s.x + s.y;
    a[G + g] += s2.x + s2.y;
  }
}

// Reduce-scatter 32 per-lane values across the warp (31 shuffles): lane L returns the warp total of
// value index L.
__device__ __forceinline__ float warp_reduce_scatter32(float (&x)[32], uint32_t lane) {
#pragma unroll
  for (int lvl = 0; lvl < 5; ++lvl) {
    const int cnt = 32 >> lvl, o = 16 >> lvl;
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < cnt / 2; ++i) {
      const float send = upper ? x[i] : x[i + cnt / 2];
      const float keep = upper ? x[i + cnt / 2] : x[i];
      x[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return x[0];
}

// rbuf: global tap index (halo stage j, tap tp -> j * taps + tp) before which extra k-block e of the
// tile is consumed -- spread evenly so every k-block's load hides behind whole taps of MMAs
__device__ __forceinline__ int rbuf_at(int e, int n_extra, int total_taps) { return (e * total_taps) / n_extra; }

// RR: the attention row-reduction epilogue (GemmArgs::rowred) is compiled in -- a separate
// instantiation, so the conv epilogue carries none of its branches or registers
template <int BN, int CG, bool XF, bool RR = false>
__global__ void __launch_bounds__(XF ? 512 : 352, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmO,
                   const KParams p) {
  using C = Cfg<BN, CG>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + p.a_stages * p.a_stage_bytes;
  uint8_t* sR = sB + p.b_stages * C::B_BYTES;  // rbuf: one extra-segment k-block of every sub-tile
  uint64_t* a_full = reinterpret_cast<uint64_t*>(sR + p.r_bytes);
  uint64_t* a_empty = a_full + kMaxStages;
  uint64_t* b_full = a_empty + kMaxStages;
  uint64_t* b_empty = b_full + kMaxStages;
  uint64_t* tfull = b_empty + kMaxStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* a_xform = tempty + 2;  // XF: halo transformed (GroupNorm + SiLU applied) and fenced
  uint64_t* r_full = a_xform + kMaxStages;  // rbuf: k-block landed / consumed
  uint64_t* r_empty = r_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(r_empty + 1);
  // 8 epilogue warps x (BN / 2) floats, 16-byte aligned for LDS.128
  float* sBias = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(tmem_slot + 4) + 15) & ~uintptr_t(15));
  // tstore: per epilogue warp, two 2 KB staging tiles (32 rows x 64 B, SWIZZLE_64B), 1 KB aligned
  uint8_t* sOut = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sBias + 8 * (BN / 2)) + 1023) & ~uintptr_t(1023));
  constexpr int EPI_WARPS = 8;
  constexpr uint32_t W_B = XF ? 2 : 10;        // B producer
  constexpr uint32_t W_EPI0 = XF ? 4 : 2;      // first epilogue warp
  constexpr uint32_t W_XF0 = 12;               // first A-transform warp (XF)

  const uint32_t warp = ptx::warp_id();
  const uint32_t lane = ptx::lane_id();
  const uint32_t rank = (CG == 2) ? ptx::cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x / CG;
  const int nclusters = gridDim.x / CG;
  // tile sequence of this cluster: a contiguous block (conv modes: a CTA walks down its own rows,
  // so the halo rows it shares with the row pair above were fetched by itself one tile-row earlier
  // and hit L2), or round-robin (plain GEMMs: concurrent clusters share A / B tiles through L2)
  const int t_first = p.sched ? (int)((long long)cluster_id * p.tiles / nclusters) : cluster_id;
  const int t_end = p.sched ? (int)((long long)(cluster_id + 1) * p.tiles / nclusters) : p.tiles;
  const int t_step = p.sched ? 1 : nclusters;
  // A stages per tile and taps (B stages) per A stage
  const int n_a = p.halo ? p.cblocks : p.num_kb;
  const int per_a = p.halo ? p.taps : 1;

  if (p.run_if) {  // uniform across the grid: every CTA reads the same flags before any barrier
    if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    int any = 0;
    for (int i = 0; i < p.run_if_n; ++i) any |= reinterpret_cast<const volatile int*>(p.run_if)[i];
    if (!any) return;
  }
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&tmA);
    ptx::tma_prefetch(&tmB);
    if (p.n_extra) ptx::tma_prefetch(&tmA2);
    for (int s = 0; s < kMaxStages; ++s) {
      ptx::mbar_init(&a_full[s], 1);
      ptx::mbar_init(&a_empty[s], 1);
      ptx::mbar_init(&b_full[s], 1);
      ptx::mbar_init(&b_empty[s], 1);
      ptx::mbar_init(&a_xform[s], 4 * CG);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], EPI_WARPS * CG);
    }
    ptx::mbar_init(r_full, 1);
    ptx::mbar_init(r_empty, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<CG>(tmem_slot, p.tmem_cols);
  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
  ptx::tc_fence_after();
  // programmatic dependent launch: the prologue above overlapped the previous kernel's tail; from
  // here on global memory is touched, so wait for that kernel to complete and flush
  if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;
  // XF: 512 threads start at 128 registers; each role branch re-sizes its warpgroup so that the
  // producers' registers go to the epilogue (4 x 56 + 8 x 176 + 4 x 96 warps' worth <= 64 K)

  if (warp == 0) {
    // ------------------------------------------------------------ A producer (TMA)
    if constexpr (XF) ptx::setmaxnreg_dec<56>();
    if (ptx::elect_one()) {
      int st = 0;
      uint32_t ph = 0, rph = 0;
      const int tot_taps = n_a * per_a;
      const uint64_t a_pol = p.a_hint ? ptx::l2_policy_evict_last() : 0ull;
      for (int t = t_first; t < t_end; t += t_step) {
        if (tile_off(p, t, CG)) continue;
        int m_tile, n_tile, phs;
        tile_coords(p, t, m_tile, n_tile, phs);
        const int rows_cta = 128 * p.msub;
        const int m0 = tile_row0(p, m_tile, rank, CG, 0);  // this CTA's first A row
        // rbuf: extra k-block e of every sub-tile into the dedicated buffer, once its previous
        // k-block has been consumed
        auto r_load = [&](int e) {
          ptx::mbar_wait(r_empty, rph ^ 1);
          if (leader) ptx::mbar_arrive_expect_tx(r_full, CG * rows_cta * 64 * 2);
          for (int sub = 0; sub < p.msub; ++sub) {
            const int ms = p.vsub ? tile_row0(p, m_tile, rank, CG, sub) : m0 + sub * 128;
            if constexpr (CG == 1) ptx::tma_load_2d(&tmA2, r_full, sR + sub * 16384, e * 64, ms);
            else ptx::tma_load_2d_pair(&tmA2, r_full, sR + sub * 16384, e * 64, ms);
          }
          rph ^= 1;
        };
        int e_next = 0;
        int img = 0, y0 = 0, x0 = 0;
        if (p.mode != GEMM_PLAIN) {
          const int hw = p.H * p.W;
          img = m0 / hw;
          const int rem = m0 - img * hw;
          y0 = rem / p.W;
          x0 = rem - y0 * p.W;
        }
        for (int j = 0; j < n_a; ++j) {
          if (p.rbuf && e_next < p.n_extra && rbuf_at(e_next, p.n_extra, tot_taps) == j * per_a) r_load(e_next++);
          ptx::mbar_wait(&a_empty[st], ph ^ 1);
          if ((p.ld_skip & 2) && t != t_first && !XF) {  // diagnostics: no A traffic
            if (leader) ptx::mbar_arrive(&a_full[st]);
            if (++st == p.a_stages) { st = 0; ph ^= 1; }
            continue;
          }
          uint8_t* dst = sA + st * p.a_stage_bytes;
          // XF: each CTA's transform warps wait for their own halo, so A lands on the local barrier
          if (XF) ptx::mbar_arrive_expect_tx(&a_full[st], p.a_tx_bytes);
          else if (leader) ptx::mbar_arrive_expect_tx(&a_full[st], CG * p.a_tx_bytes);
          int c0 = 0, c1 = 0, c2 = 0, c3 = img;
          if (p.mode == GEMM_PLAIN) {
            c0 = j * 64;
            c1 = m0;
          } else if (p.halo) {  // per sub-tile: rows [y_top, y_top + halo_rows) x cols [x-1, x+129) x 64 ch
            c0 = j * 64;
            c1 = x0 - 1;
            c2 = p.mode == GEMM_CONV3X3 ? y0 - 1 : y0 + (phs >> 1) - 1;
            for (int sub = 1; sub < (p.vsub ? 1 : p.msub); ++sub) {
              if constexpr (CG == 1 || XF) ptx::tma_load_4d(&tmA, &a_full[st], dst + sub * p.halo_sub_bytes, c0, c1 + sub * 128, c2, c3);
              else ptx::tma_load_4d_pair(&tmA, &a_full[st], dst + sub * p.halo_sub_bytes, c0, c1 + sub * 128, c2, c3);
            }
          } else {
            const int tap = j / p.cblocks;
            const int cb = j - tap * p.cblocks;
            int dx, dy;
            if (p.mode == GEMM_CONV3X3) {
              dy = tap / 3 - 1;
              dx = tap % 3 - 1;
            } else {  // sub-pixel phase (a, b): low-res offsets r + a - 1
              dy = (tap >> 1) + (phs >> 1) - 1;
              dx = (tap & 1) + (phs & 1) - 1;
            }
            c0 = cb * 64;
            c1 = x0 + dx;
            c2 = y0 + dy;
          }
          if (p.mode == GEMM_PLAIN) {
            if constexpr (CG == 1) ptx::tma_load_2d(&tmA, &a_full[st], dst, c0, c1);
            else ptx::tma_load_2d_pair(&tmA, &a_full[st], dst, c0, c1);
          } else if (p.a_hint) {  // halo rows: keep them in L2 for the vertically adjacent tiles
            if constexpr (CG == 1 || XF) ptx::tma_load_4d_hint(&tmA, &a_full[st], dst, c0, c1, c2, c3, a_pol);
            else ptx::tma_load_4d_pair_hint(&tmA, &a_full[st], dst, c0, c1, c2, c3, a_pol);
          } else {
            if constexpr (CG == 1 || XF) ptx::tma_load_4d(&tmA, &a_full[st], dst, c0, c1, c2, c3);
            else ptx::tma_load_4d_pair(&tmA, &a_full[st], dst, c0, c1, c2, c3);
          }
          if (++st == p.a_stages) { st = 0; ph ^= 1; }
          if (p.rbuf)  // the k-blocks consumed between this stage's later taps
            while (e_next < p.n_extra && rbuf_at(e_next, p.n_extra, tot_taps) < (j + 1) * per_a) r_load(e_next++);
        }
        for (int e = 0; e < (p.rbuf ? 0 : p.n_extra); ++e) {  // second operand: plain [M][K2] rows of this tile
          ptx::mbar_wait(&a_empty[st], ph ^ 1);
          uint8_t* dst = sA + st * p.a_stage_bytes;
          if (XF) ptx::mbar_arrive_expect_tx(&a_full[st], rows_cta * 64 * 2);
          else if (leader) ptx::mbar_arrive_expect_tx(&a_full[st], CG * rows_cta * 64 * 2);
          for (int sub = 0; sub < p.msub; ++sub) {
            const int ms = p.vsub ? tile_row0(p, m_tile, rank, CG, sub) : m0 + sub * 128;
            if constexpr (CG == 1 || XF) ptx::tma_load_2d(&tmA2, &a_full[st], dst + sub * 16384, e * 64, ms);
            else ptx::tma_load_2d_pair(&tmA2, &a_full[st], dst + sub * 16384, e * 64, ms);
          }
          if (++st == p.a_stages) { st = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == W_B) {
    // ------------------------------------------------------------ B producer (TMA, weights)
    if constexpr (XF) ptx::setmaxnreg_dec<56>();
    if (ptx::elect_one()) {
      int st = 0;
      uint32_t ph = 0;
      for (int t = t_first; t < t_end; t += t_step) {
        if (tile_off(p, t, CG)) continue;
        int m_tile, n_tile, phs;
        tile_coords(p, t, m_tile, n_tile, phs);
        const int bimg = p.batch_m ? (m_tile * 128 * p.msub * CG) / p.batch_m : 0;  // batched: image of the tile
        const int b_row = (p.mode == GEMM_SUBPIX ? phs * p.N : 0) + n_tile * BN + rank * C::B_ROWS +
                          (p.b_mn ? 0 : bimg * p.batch_b);
        const int k_img = p.b_mn ? bimg * p.batch_b : 0;
        int e_next = 0;
        for (int j = 0; j < n_a; ++j) {
          for (int tp = 0; tp < per_a; ++tp) {
            if (p.rbuf && e_next < p.n_extra && rbuf_at(e_next, p.n_extra, n_a * per_a) == j * per_a + tp) {
              ptx::mbar_wait(&b_empty[st], ph ^ 1);  // the extra k-block's B rows, in MMA order
              if (leader) ptx::mbar_arrive_expect_tx(&b_full[st], CG * C::B_BYTES);
              uint8_t* dst = sB + st * C::B_BYTES;
              if constexpr (CG == 1) ptx::tma_load_2d(&tmB, &b_full[st], dst, p.k_main + e_next * 64, b_row);
              else ptx::tma_load_2d_pair(&tmB, &b_full[st], dst, p.k_main + e_next * 64, b_row);
              if (++st == p.b_stages) { st = 0; ph ^= 1; }
              ++e_next;
            }
            ptx::mbar_wait(&b_empty[st], ph ^ 1);
            if ((p.ld_skip & 1) && t != t_first) {  // diagnostics: no B traffic
              if (leader) ptx::mbar_arrive(&b_full[st]);
              if (++st == p.b_stages) { st = 0; ph ^= 1; }
              continue;
            }
            if (leader) ptx::mbar_arrive_expect_tx(&b_full[st], CG * C::B_BYTES);
            const int k0 = p.halo ? tp * (p.cblocks * 64) + j * 64 : j * 64;  // K = (tap, channel)
            uint8_t* dst = sB + st * C::B_BYTES;
            if (p.b_mn) {  // B_ROWS / 64 boxes of (64 N) x (64 K), one per 64-wide N atom
              for (int na = 0; na < C::B_ROWS / 64; ++na) {
                if constexpr (CG == 1) ptx::tma_load_2d(&tmB, &b_full[st], dst + na * 8192, b_row + na * 64, k0 + k_img);
                else ptx::tma_load_2d_pair(&tmB, &b_full[st], dst + na * 8192, b_row + na * 64, k0 + k_img);
              }
            } else if constexpr (CG == 1) {
              ptx::tma_load_2d(&tmB, &b_full[st], dst, k0, b_row);
            } else {
              ptx::tma_load_2d_pair(&tmB, &b_full[st], dst, k0, b_row);
            }
            if (++st == p.b_stages) { st = 0; ph ^= 1; }
          }
        }
        for (int e = 0; e < (p.rbuf ? 0 : p.n_extra); ++e) {
          ptx::mbar_wait(&b_empty[st], ph ^ 1);
          if (leader) ptx::mbar_arrive_expect_tx(&b_full[st], CG * C::B_BYTES);
          uint8_t* dst = sB + st * C::B_BYTES;
          if constexpr (CG == 1) ptx::tma_load_2d(&tmB, &b_full[st], dst, p.k_main + e * 64, b_row);
          else ptx::tma_load_2d_pair(&tmB, &b_full[st], dst, p.k_main + e * 64, b_row);
          if (++st == p.b_stages) { st = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA)
    // One thread runs the whole issue loop (no per-tap elect / reconvergence).  Descriptors are
    // built once and advanced by adding (byte offset >> 4) to the address field: every smem
    // address is < 256 KB, so the 14-bit field never carries.
    if constexpr (XF) ptx::setmaxnreg_dec<56>();
    if (leader && ptx::elect_one()) {
      int as = 0, bs = 0;
      uint32_t aph = 0, bph = 0, rph = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const uint64_t a_desc0 = ptx::sdesc_k_sw128(ptx::smem_u32(sA));
      // MN-major B (SW128 canonical ((8,n),(8,k)) in 16-byte units): LBO = 8 KB between 64-wide N
      // atoms, SBO = 1 KB between 8-row K groups; a K16 step is two K groups (+2 KB)
      const uint64_t b_desc0 = p.b_mn ? ptx::sdesc_mn_sw128(ptx::smem_u32(sB), 8192, 1024)
                                      : ptx::sdesc_k_sw128(ptx::smem_u32(sB));
      const uint32_t b_k16 = p.b_mn ? (2048 >> 4) : 2;
      const uint32_t idesc = C::IDESC | (p.b_mn ? (1u << 16) : 0u);
      const uint32_t a_stage16 = (uint32_t)p.a_stage_bytes >> 4, sub16 = (uint32_t)p.halo_sub_bytes >> 4;
      const int msub = p.msub;
      const bool conv = p.mode == GEMM_CONV3X3, halo = p.halo != 0, dbm = p.desc_base_mode != 0;
      const uint64_t r_desc0 = ptx::sdesc_k_sw128(ptx::smem_u32(sR));
      const uint32_t rb = (p.rbuf && p.n_extra) ? 1u : 0u;  // the tile's first MMA is an extra k-block's
      const int tot_taps = n_a * per_a;
      for (int t = t_first; t < t_end; t += t_step) {
        if (tile_off(p, t, CG)) continue;
        int m_tile, n_tile, phs;
        tile_coords(p, t, m_tile, n_tile, phs);
        // rpf: every use of a buffer (the first included) waits for the epilogue's residual preload
        ptx::mbar_wait_cluster(&tempty[acc], p.rpf ? acc_phase : acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * (msub * BN);
        const uint32_t acc0 = (p.rpf ? 1u : 0u) | rb;  // accumulate onto the preloaded residual / k-block 0
        int e_next = 0;
        for (int j = 0; j < n_a; ++j) {
          uint64_t a_stage = 0;
          int r0 = halo && !conv ? (phs & 1) : 0;  // the tap's 128 A rows start r0 rows into the halo
          for (int tp = 0; tp < per_a; ++tp) {
            if (rb && e_next < p.n_extra && rbuf_at(e_next, p.n_extra, tot_taps) == j * per_a + tp) {
              ptx::mbar_wait(r_full, rph);  // extra k-block e_next (its B rows are next in the ring)
              ptx::mbar_wait(&b_full[bs], bph);
              ptx::tc_fence_after();
              const uint64_t b_desc = b_desc0 + (uint64_t)(bs * (C::B_BYTES >> 4));
#pragma unroll
              for (int sub = 0; sub < 2; ++sub) {
                if (sub < msub) {
                  const uint64_t a_desc = r_desc0 + (uint64_t)(sub * (16384 >> 4));
#pragma unroll
                  for (int k = 0; k < 4; ++k)
                    ptx::mma_f16_ss<CG>(d_tmem + sub * BN, a_desc + 2 * k, b_desc + b_k16 * k, idesc, (e_next | k) != 0);
                }
              }
              ptx::mma_commit<CG>(&b_empty[bs]);
              ptx::mma_commit<CG>(r_empty);
              if (++bs == p.b_stages) { bs = 0; bph ^= 1; }
              rph ^= 1;
              ++e_next;
            }
            if (tp == 0) {
              if (XF) ptx::mbar_wait_cluster(&a_xform[as], aph);
              else ptx::mbar_wait(&a_full[as], aph);
              a_stage = a_desc0 + (uint64_t)(as * a_stage16);
            }
            ptx::mbar_wait(&b_full[bs], bph);
            ptx::tc_fence_after();
            const uint64_t b_desc = b_desc0 + (uint64_t)(bs * (C::B_BYTES >> 4));
#pragma unroll
            for (int sub = 0; sub < 2; ++sub) {  // sub-tiles share this B tile
              if (sub < msub) {
                uint64_t a_desc = a_stage + (uint64_t)(sub * sub16 + r0 * 8);
                if (dbm) a_desc |= (uint64_t)(r0 & 7) << 49;
#pragma unroll
                for (int k = 0; k < 4; ++k)  // 4 x K16 per 64-wide k-block; +32 B per step inside the swizzle atom
                  ptx::mma_f16_ss<CG>(d_tmem + sub * BN, a_desc + 2 * k, b_desc + b_k16 * k, idesc, (acc0 | j | tp | k) != 0);
              }
            }
            ptx::mma_commit<CG>(&b_empty[bs]);
            if (++bs == p.b_stages) { bs = 0; bph ^= 1; }
            if (halo) {  // conv3x3: r0 = ky*130 + kx; sub-pixel: (tap >> 1)*130 + (tap & 1) + (phase & 1)
              if (conv) r0 += (tp % 3 == 2) ? 128 : 1;
              else r0 += (tp & 1) ? 129 : 1;
            }
          }
          ptx::mma_commit<CG>(&a_empty[as]);
          if (j == n_a - 1 && (p.n_extra == 0 || p.rbuf)) ptx::mma_commit<CG>(&tfull[acc]);
          if (++as == p.a_stages) { as = 0; aph ^= 1; }
        }
        for (int e = 0; e < (p.rbuf ? 0 : p.n_extra); ++e) {
          if (XF) ptx::mbar_wait_cluster(&a_xform[as], aph);
          else ptx::mbar_wait(&a_full[as], aph);
          ptx::mbar_wait(&b_full[bs], bph);
          ptx::tc_fence_after();
          const uint64_t b_desc = b_desc0 + (uint64_t)(bs * (C::B_BYTES >> 4));
          const uint64_t a_stage = a_desc0 + (uint64_t)(as * a_stage16);
#pragma unroll
          for (int sub = 0; sub < 2; ++sub) {
            if (sub < msub) {
              const uint64_t a_desc = a_stage + (uint64_t)(sub * (16384 >> 4));
#pragma unroll
              for (int k = 0; k < 4; ++k)
                ptx::mma_f16_ss<CG>(d_tmem + sub * BN, a_desc + 2 * k, b_desc + b_k16 * k, idesc, 1u);
            }
          }
          ptx::mma_commit<CG>(&b_empty[bs]);
          ptx::mma_commit<CG>(&a_empty[as]);
          if (e == p.n_extra - 1) ptx::mma_commit<CG>(&tfull[acc]);
          if (++bs == p.b_stages) { bs = 0; bph ^= 1; }
          if (++as == p.a_stages) { as = 0; aph ^= 1; }
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (XF && warp == 3) {
    ptx::setmaxnreg_dec<56>();  // idle (keeps the warpgroups aligned)
  } else if (XF && warp >= W_XF0) {
    // ------------------------------------------------------------ fused GroupNorm + SiLU on A
    // Warps 12..15 rewrite each landed halo in place: y = SiLU(x * a_c + b_c) (fp32 affine, SiLU
    // on packed halves as in act.cuh gn_act8_h2, one fp16 rounding) for pixels inside the image;
    // out-of-image positions keep TMA's zero fill (the conv pads after the activation).  Thread t
    // owns logical 16-byte chunk t & 7 (8 channels) of every 16th halo row, so its 8 (a, b) pairs
    // load once per C-block; the physical chunk is (chunk ^ row & 7) (128B swizzle).
    if constexpr (XF) ptx::setmaxnreg_dec<96>();
    const int tid = (int)(warp - W_XF0) * 32 + (int)lane;
    const int cq = tid & 7;
    const int nbox = p.vsub ? 1 : p.msub;
    const int box_rows = p.vsub ? p.halo_rows + p.msub - 1 : p.halo_rows;
    const int rows = box_rows * 130;
    int st = 0;
    uint32_t ph = 0;
    for (int t = t_first; t < t_end; t += t_step) {
      if (tile_off(p, t, CG)) continue;
      int m_tile, n_tile, phs;
      tile_coords(p, t, m_tile, n_tile, phs);
      const int m0 = tile_row0(p, m_tile, (int)rank, CG, 0);
      const int hw = p.H * p.W;
      const int img = m0 / hw;
      const int rem = m0 - img * hw;
      const int y0 = rem / p.W, x0 = rem - (rem / p.W) * p.W;
      for (int j = 0; j < n_a + p.n_extra; ++j) {
        float ca[8], cb[8];
        if (j < n_a) {
          const float4* cp = reinterpret_cast<const float4*>(p.gn_ss + (size_t)img * p.cblocks * 64 + j * 64 + cq * 8);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float4 v = __ldg(cp + k);  // halved for gn_silu8_h2_half
            ca[2 * k] = 0.5f * v.x; cb[2 * k] = 0.5f * v.y; ca[2 * k + 1] = 0.5f * v.z; cb[2 * k + 1] = 0.5f * v.w;
          }
        }
        ptx::mbar_wait(&a_full[st], ph);
        if (j < n_a) {
          uint8_t* base = sA + st * p.a_stage_bytes;
          for (int bx = 0; bx < nbox; ++bx) {
            const uint32_t hb = ptx::smem_u32(base + bx * p.halo_sub_bytes);
            const int xs = x0 - 1 + bx * 128;
            // validity of halo row r = (hr, px): vertical from a per-box row mask, horizontal only
            // at the image's left / right edge (px 0 / 129); invalid rows keep TMA's zero fill
            uint32_t vmask = 0;
            for (int k = 0; k < box_rows; ++k)
              if (y0 - 1 + k >= 0 && y0 - 1 + k < p.H) vmask |= 1u << k;
            const bool ledge = xs < 0, redge = xs + 129 >= p.W;
            int hr = 0, px = tid >> 3;  // row r = tid/8 + 16 i, as (halo row, pixel)
            // four rows per iteration: independent LDS -> affine -> MUFU chains per thread
            for (int r = tid >> 3; r < rows; r += 64) {
              uint4 u[4];
              bool v[4];
              uint32_t q[4];
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                int pk = px + 16 * k, hk = hr;
                if (pk >= 130) { pk -= 130; ++hk; }
                const int rk = r + 16 * k;
                v[k] = rk < rows && ((vmask >> hk) & 1u) && !(ledge && pk == 0) && !(redge && pk == 129);
                q[k] = hb + rk * 128 + ((cq ^ (rk & 7)) << 4);
                u[k] = v[k] ? ptx::lds128(q[k]) : make_uint4(0, 0, 0, 0);
              }
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const uint4 w = gn_silu8_h2_half(u[k], ca, cb);
                if (v[k]) ptx::sts128(q[k], w);
              }
              px += 64;
              if (px >= 130) { px -= 130; ++hr; }
            }
          }
          ptx::fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
        }
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 1) ptx::mbar_arrive(&a_xform[st]);
          else ptx::mbar_arrive_cluster(&a_xform[st], 0);
        }
        if (++st == p.a_stages) { st = 0; ph ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..9; XF: 4..11)
    if constexpr (XF) ptx::setmaxnreg_inc<176>();
    // Two warps per TMEM lane quarter; warp half `hsel` takes the even/odd 32-column chunks.
    const uint32_t q = warp & 3;
    const int ew = (int)(warp - W_EPI0);  // epilogue warp index 0..7
    const int hsel = ew >> 2;
    const int row = q * 32 + lane;
    constexpr int NCH = BN / 32 / (EPI_WARPS / 4);  // chunks per warp per tile
    // 32-column chunk j of this warp: contiguous (the warp owns whole 128-byte row segments, so a
    // lane's consecutive stores complete a cache line) or interleaved with the other column half
    const int cbase = p.cmap ? hsel * NCH : hsel, cstep = p.cmap ? 1 : (EPI_WARPS / 4);
    // GroupNorm partials: each lane accumulates its own per-chunk (group sum, group sumsq) values in
    // fp32 registers across tiles (NCH x NV <= 32 of them); at a flush -- when the (image, n-tile)
    // changes -- the warp reduce-scatters them (lane L owns value L) and adds them as one exact
    // fixed-point integer pair per value (gnfix.cuh).  Which tiles a lane sums in fp32 is fixed by
    // the tile index within its image (residue class mod the cluster count, see gemm_tc_launch), so
    // together with the order-independent integer totals an image's statistics do not depend on
    // its position in the batch or on the batch size.
    float sacc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) sacc[i] = 0.f;
    // bias of this warp's chunks, staged once per n-tile in the warp's own smem slice and read back
    // as broadcast LDS.128 (an LDG per chunk put the L1 latency on the epilogue's critical path)
    // shared-space address: the pointer arithmetic on the dynamic smem base makes the compiler emit
    // generic LD.E/ST.E for plain dereferences (long-scoreboard stalls in ncu), so use LDS/STS
    const uint32_t wbias = ptx::smem_u32(sBias) + ew * (NCH * 32) * 4;
    int bias_ntile = -1;
    const bool scaled = p.row_scale != nullptr || p.alpha != 1.f;
    int g_img = -1, g_ntile = -1;
    const int nv = p.gn_stats ? 64 / p.gn_cpg : 0;  // values per chunk: 2 * groups-per-chunk
    auto flush = [&]() {
      if (g_img < 0) return;
      const float tot = warp_reduce_scatter32(sacc, lane);
      if ((int)lane < nv * NCH) {
        const int j = (int)lane / nv, i = (int)lane - j * nv;
        const int gpc = nv >> 1;  // groups per chunk
        const int kind = i >= gpc;
        const int c = cbase + cstep * j;
        const int grp = (g_ntile * BN + c * 32) / p.gn_cpg + (i - kind * gpc);
        gnfix_add(p.gn_stats + (((size_t)g_img * 32 + grp) * 2 + kind) * 2, tot);  // order-independent
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) sacc[i] = 0.f;
    };
    // Residual preload (rpf): the residual of tile tn goes into accumulator buffer `buf` (fp16 ->
    // fp32, tcgen05.st) before its MMAs start, which then accumulate onto it; the release of the
    // buffer to the MMA issuer is the arrival after the preload.  It replaces the folded extra K
    // (4-8 short k-blocks of MMAs) and the epilogue's late residual reads.
    auto prefill = [&](int tn, int buf) {
      if (tn < t_end && p.rres) {
        // line-covering loads: instruction k reads pixels 8k..8k+7 of the warp's 32 rows, 64 B each
        // (lane l: pixel 8k + l/4, quarter l%4), transposed through the warp's 2 KB swizzled stage
        int mt, nt, phn;
        tile_coords(p, tn, mt, nt, phn);
        const uint32_t stage = ptx::smem_u32(sOut + ew * 2 * 2048);
        for (int sub = 0; sub < p.msub; ++sub) {
          const long long prow0 = tile_row0(p, mt, (int)rank, CG, sub) + q * 32;  // the warp's first pixel row
          const uint32_t tb = tmem_base + ((q * 32u) << 16) + buf * (p.msub * BN) + sub * BN;
#pragma unroll
          for (int j = 0; j < NCH; ++j) {
            const __half* rb0 = p.resid + prow0 * p.ldr + nt * BN + (cbase + cstep * j) * 32;
            uint4 u[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int px = 8 * k + (int)(lane >> 2);
              u[k] = __ldg(reinterpret_cast<const uint4*>(rb0 + (long long)px * p.ldr) + (lane & 3));
            }
            __syncwarp();  // the stage's previous contents are consumed
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int px = 8 * k + (int)(lane >> 2);
              ptx::sts128(stage + px * 64 + ((((int)lane & 3) ^ ((px >> 1) & 3)) << 4), u[k]);
            }
            __syncwarp();
            uint32_t r[32];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint4 v = ptx::lds128(stage + lane * 64 + ((i ^ ((lane >> 1) & 3)) << 4));
              const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w4[k]));
                r[i * 8 + 2 * k] = __float_as_uint(f.x);
                r[i * 8 + 2 * k + 1] = __float_as_uint(f.y);
              }
            }
            ptx::tmem_st32(tb + (cbase + cstep * j) * 32, r);
          }
        }
        ptx::tmem_st_wait();
      } else if (tn < t_end) {
        int mt, nt, phn;
        tile_coords(p, tn, mt, nt, phn);
        const long long mrow0 = tile_row0(p, mt, (int)rank, CG, 0) + row;
        for (int sub = 0; sub < p.msub; ++sub) {
          const long long mrow = mrow0 + sub * (p.vsub ? p.W : 128);
          const __half* rb = p.resid + mrow * p.ldr + nt * BN + cbase * 32;
          const uint32_t tb = tmem_base + ((q * 32u) << 16) + buf * (p.msub * BN) + sub * BN;
#pragma unroll
          for (int j = 0; j < NCH; ++j) {
            uint4 u[4];
            if (p.ld_skip & 4) {  // diagnostics (bit 4 of ld_skip): preload zeros, no residual loads
#pragma unroll
              for (int i = 0; i < 4; ++i) u[i] = make_uint4(0, 0, 0, 0);
            } else if (p.ld_skip & 8) {  // diagnostics: the residual rows of tile 0 (L2-resident)
              const __half* r0 = p.resid + (long long)row * p.ldr + cbase * 32;
#pragma unroll
              for (int i = 0; i < 4; ++i) u[i] = __ldg(reinterpret_cast<const uint4*>(r0 + j * 32 * cstep) + i);
            } else {
#pragma unroll
              for (int i = 0; i < 4; ++i) u[i] = __ldg(reinterpret_cast<const uint4*>(rb + j * 32 * cstep) + i);
            }
            uint32_t r[32];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint32_t w4[4] = {u[i].x, u[i].y, u[i].z, u[i].w};
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w4[k]));
                r[i * 8 + 2 * k] = __float_as_uint(f.x);
                r[i * 8 + 2 * k + 1] = __float_as_uint(f.y);
              }
            }
            ptx::tmem_st32(tb + (cbase + cstep * j) * 32, r);
          }
        }
        ptx::tmem_st_wait();
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 1) ptx::mbar_arrive_relaxed(&tempty[buf]);
        else ptx::mbar_arrive_cluster_relaxed(&tempty[buf], 0);
      }
    };
    // L2 prefetch of the rows the next preload reads, issued before the wait for the accumulator
    auto prefetch_resid = [&](int tn) {
      if (tn >= t_end || !g_rpf_l2pf_dev(p)) return;
      int mt, nt, phn;
      tile_coords(p, tn, mt, nt, phn);
      for (int sub = 0; sub < p.msub; ++sub) {
        const long long mrow = tile_row0(p, mt, (int)rank, CG, sub) + row;
        const __half* rb = p.resid + mrow * p.ldr + nt * BN + cbase * 32;
#pragma unroll
        for (int j = 0; j < NCH; ++j) asm volatile("prefetch.global.L2 [%0];" ::"l"(rb + j * 32 * cstep));
      }
    };
    if (p.rpf) {
      prefill(t_first, 0);
      prefill(t_first + t_step, 1);
    }
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t ochunk = 0;  // tstore: staged chunks so far (selects the staging buffer)
    for (int t = t_first; t < t_end; t += t_step) {
      if (tile_off(p, t, CG)) continue;
      int m_tile, n_tile, ph;
      tile_coords(p, t, m_tile, n_tile, ph);
      const int n0 = n_tile * BN;
      if (p.bias && n_tile != bias_ntile) {
        __syncwarp();
#pragma unroll
        for (int j = 0; j < NCH; ++j)
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(wbias + (j * 32 + lane) * 4),
                       "f"(p.bias[n0 + (cbase + cstep * j) * 32 + lane])
                       : "memory");
        __syncwarp();
        bias_ntile = n_tile;
      }
      if (p.rpf) prefetch_resid(t + 2 * t_step);
      const int mrow0 = tile_row0(p, m_tile, (int)rank, CG, 0) + row;  // sub-tile s: + s * sub_stride
      const int sub_stride = p.vsub ? p.W : 128;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      for (int sub = 0; sub < (p.epi_skip == 1 ? 0 : p.msub); ++sub) {
      const int m = mrow0 + sub * sub_stride;
      long long orow = m;
      if (p.mode == GEMM_SUBPIX) {
        const int hw = p.H * p.W;
        const int img = m / hw;
        const int rem = m - img * hw;
        const int i = rem / p.W, j = rem - (rem / p.W) * p.W;
        orow = ((long long)img * (2 * p.H) + (2 * i + (ph >> 1))) * (2 * p.W) + (2 * j + (ph & 1));
      }
      const float rs = scaled ? p.alpha * (p.row_scale ? p.row_scale[m] : 1.f) : 1.f;
      if (p.gn_stats) {
        const int img = fdiv(m, p.fd_rpi);  // warp-uniform: 32-row slices never straddle images
        if (img != g_img || n_tile != g_ntile) {
          flush();
          g_img = img;
          g_ntile = n_tile;
        }
      }

      // attention row reductions: this lane's row, this warp's column half of the tile
      float racc = RR && p.rowred == 1 ? -INFINITY : 0.f;
      bool rbig = false;  // rowred 2: a chunk's E sum reached the fp16 range limit (possible overflow)
      float2 esc = make_float2(0.f, 0.f), eoff = esc;  // E = 2^(acc * esc - eoff): alpha log2(e), r_m log2(e)
      if (RR && p.rowred == 2) {
        const float rref = fmaxf(__ldg(p.row_max + 2 * (size_t)m), __ldg(p.row_max + 2 * (size_t)m + 1));
        esc = make_float2(p.alpha * 1.4426950408889634f, p.alpha * 1.4426950408889634f);
        eoff = make_float2(-rref * 1.4426950408889634f, -rref * 1.4426950408889634f);
      }

      // residual prefetch ring, two chunks deep, issued before waiting for the accumulator
      constexpr int PF = NCH < 2 ? NCH : 2;
      uint4 rr[PF][4];
      const bool eresid = p.resid && !p.rpf;  // residual added here (not preloaded into TMEM)
      const __half* rbase = eresid ? p.resid + orow * p.ldr + n0 + cbase * 32 : nullptr;
      const int RSTRIDE = 32 * cstep;  // columns between this warp's chunks
      if (eresid) {
#pragma unroll
        for (int j = 0; j < PF; ++j)
#pragma unroll
          for (int i = 0; i < 4; ++i) rr[j][i] = __ldg(reinterpret_cast<const uint4*>(rbase + j * RSTRIDE) + i);
      }
      const uint32_t t_row = tmem_base + ((q * 32u) << 16) + acc * (p.msub * BN) + sub * BN;
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        const int c = cbase + cstep * j;
        const int n = n0 + c * 32;
        uint32_t r[32];
        ptx::tmem_ld32(t_row + c * 32, r);
        ptx::tmem_ld_wait();
        if (p.epi_skip == 2) {  // diagnostics: TMEM reads only
          if (r[0] == 0x7fc00001u && r[31] == 0x7fc00001u) p.out[0] = __float2half(0.f);  // keep the load
          continue;
        }
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        if (RR && p.rowred == 2 && p.exp_h2) {
          // E = exp(alpha acc - r_m): the exponent u = log2(e) (alpha acc - r_m) in fp32 (one FFMA2
          // per pair), rounded to fp16 -- its error is relative to |S - r_m|, not to |S| -- then two
          // E per MUFU op (ex2.approx.f16x2), already the fp16 values P.V multiplies; their fp32 sum
          float2 cs = make_float2(0.f, 0.f);
          uint32_t e2[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 u = ffma2(make_float2(v[2 * i], v[2 * i + 1]), esc, eoff);
            const __half2 uh = __floats2half2_rn(u.x, u.y);
            e2[i] = ptx::ex2_approx_h2(*reinterpret_cast<const uint32_t*>(&uh));
            cs = fadd2(cs, __half22float2(*reinterpret_cast<const __half2*>(&e2[i])));
          }
          const float csum = cs.x + cs.y;
          racc += csum;
          rbig |= !(csum < 65504.f);  // an E of the chunk may be inf (or NaN): flag the group
          uint4* op = reinterpret_cast<uint4*>(p.out + orow * p.ldo + n);
          uint4 pk[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) pk[i] = make_uint4(e2[4 * i], e2[4 * i + 1], e2[4 * i + 2], e2[4 * i + 3]);
          if (p.tstore) {
            uint8_t* buf = sOut + (ew * 2 + (ochunk & 1)) * 2048;
            if (lane == 0) ptx::bulk_wait_read<1>();
            __syncwarp();
            const uint32_t base = ptx::smem_u32(buf) + lane * 64;
#pragma unroll
            for (int i = 0; i < 4; ++i) ptx::sts128(base + ((i ^ ((lane >> 1) & 3)) << 4), pk[i]);
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) ptx::tma_store_2d(&tmO, buf, n, (int)(orow - lane));
            ++ochunk;
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) op[i] = pk[i];
          }
          continue;
        }
        if (RR && p.rowred == 2) {  // E = exp(alpha acc - r_m): one FFMA2 per pair, the exponential in fp32
          float2 cs = make_float2(0.f, 0.f);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 u = ffma2(make_float2(v[2 * i], v[2 * i + 1]), esc, eoff);
            v[2 * i] = ptx::ex2_approx(u.x);
            v[2 * i + 1] = ptx::ex2_approx(u.y);
            cs = fadd2(cs, make_float2(v[2 * i], v[2 * i + 1]));
          }
          const float csum = cs.x + cs.y;
          racc += csum;
          rbig |= !(csum < 65504.f);  // some E of the chunk may not fit fp16 (or NaN): flag the group
        } else if (scaled) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 t = fmul2(make_float2(v[2 * i], v[2 * i + 1]), make_float2(rs, rs));
            v[2 * i] = t.x; v[2 * i + 1] = t.y;
          }
        }
        if (RR && p.rowred == 1) {  // row maximum only, nothing stored
#pragma unroll
          for (int i = 0; i < 32; ++i) racc = fmaxf(racc, v[i]);
          continue;
        }
        if (p.bias) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float4 b;
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                         : "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                         : "r"(wbias + (j * 32 + 4 * i) * 4));
            const float2 t0 = fadd2(make_float2(v[4 * i], v[4 * i + 1]), make_float2(b.x, b.y));
            const float2 t1 = fadd2(make_float2(v[4 * i + 2], v[4 * i + 3]), make_float2(b.z, b.w));
            v[4 * i] = t0.x; v[4 * i + 1] = t0.y; v[4 * i + 2] = t1.x; v[4 * i + 3] = t1.y;
          }
        }
        if (eresid) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint4 q4 = rr[j % PF][i];
            const uint32_t w4[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float2 t = fadd2(make_float2(v[i * 8 + 2 * k], v[i * 8 + 2 * k + 1]),
                                     __half22float2(*reinterpret_cast<const __half2*>(&w4[k])));
              v[i * 8 + 2 * k] = t.x;
              v[i * 8 + 2 * k + 1] = t.y;
            }
          }
          if (j + PF < NCH) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              rr[j % PF][i] = __ldg(reinterpret_cast<const uint4*>(rbase + (j + PF) * RSTRIDE) + i);
          }
        }
        // pack straight into four aligned register quads (no MOVs into a shared staging quad,
        // whose reuse serialised each STG.128 behind the previous one's operand read)
        uint4 pk[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          __half2 h0 = __floats2half2_rn(v[8 * i], v[8 * i + 1]), h1 = __floats2half2_rn(v[8 * i + 2], v[8 * i + 3]);
          __half2 h2 = __floats2half2_rn(v[8 * i + 4], v[8 * i + 5]), h3 = __floats2half2_rn(v[8 * i + 6], v[8 * i + 7]);
          pk[i] = make_uint4(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1),
                             *reinterpret_cast<uint32_t*>(&h2), *reinterpret_cast<uint32_t*>(&h3));
        }
        uint4* op = reinterpret_cast<uint4*>(p.out + orow * p.ldo + n);
        if (p.tstore) {
          // stage the warp's 32 x 32 chunk (conflict-free under the 64B swizzle) and TMA-store it:
          // 16 smem wavefronts instead of 64 L1 wavefronts for two STG.256 with 32 distinct rows
          uint8_t* buf = sOut + (ew * 2 + (ochunk & 1)) * 2048;
          if (lane == 0) ptx::bulk_wait_read<1>();  // the store that used this buffer has read it
          __syncwarp();
          const uint32_t base = ptx::smem_u32(buf) + lane * 64;
#pragma unroll
          for (int i = 0; i < 4; ++i) ptx::sts128(base + ((i ^ ((lane >> 1) & 3)) << 4), pk[i]);
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) ptx::tma_store_2d(&tmO, buf, n, (int)(orow - lane));
          ++ochunk;
        } else if (p.epi_skip == 3) {  // diagnostics: no stores
          if (pk[0].x == 0x7fc07fc1u && pk[3].w == 0x7fc07fc1u) op[0] = pk[0];
        } else if (g_store_mode_dev(p) == 1) {  // two 256-bit stores (STG.256)
#pragma unroll
          for (int i = 0; i < 2; ++i)
            asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(op + 2 * i), "r"(pk[2 * i].x),
                         "r"(pk[2 * i].y), "r"(pk[2 * i].z), "r"(pk[2 * i].w), "r"(pk[2 * i + 1].x),
                         "r"(pk[2 * i + 1].y), "r"(pk[2 * i + 1].z), "r"(pk[2 * i + 1].w)
                         : "memory");
        } else if (g_store_mode_dev(p) == 2) {  // streaming stores
#pragma unroll
          for (int i = 0; i < 4; ++i) __stcs(op + i, pk[i]);
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) op[i] = pk[i];
        }
        if (p.gn_stats && p.epi_skip != 4) {  // NCH * nv <= 32 always (nv = 16 only with 128-wide tiles, NCH = 2)
          if (nv == 16) {
            if constexpr (NCH <= 2) lane_group_stats<16>(v, sacc + j * 16);
          } else if (nv == 8) {
            if constexpr (NCH <= 4) lane_group_stats<8>(v, sacc + j * 8);
          } else {
            lane_group_stats<4>(v, sacc + j * 4);
          }
        }
      }
      if (RR && p.rowred) {
        p.row_part[(size_t)m * (2 * p.n_tiles) + n_tile * 2 + hsel] = racc;
        if (p.rowred == 2 && (rbig || p.exp_force)) atomicOr(p.exp_flag + (p.batch_m ? m / p.batch_m : 0), 1);
      }
      }  // sub-tiles
      if (p.rpf) {
        prefill(t + 2 * t_step, acc);  // this buffer's next tile: preload, then release
      } else {
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 1) ptx::mbar_arrive_relaxed(&tempty[acc]);
          else ptx::mbar_arrive_cluster_relaxed(&tempty[acc], 0);
        }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (p.gn_stats) flush();
    if (p.tstore && lane == 0) ptx::bulk_wait_all();
  }

  if (p.pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // this CTA's work is done
  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<CG>(tmem_base, p.tmem_cols);
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
                     const cuuint32_t* box, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, rank, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tensor_map_f16(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                         const uint32_t* box) {
  cuuint64_t d[5], st[4];
  cuuint32_t bx[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    bx[i] = box[i];
    if (i + 1 < rank) st[i] = strides[i];
  }
  return make_map(m, base, rank, d, st, bx);
}

static int g_halo_policy = 1;      // 1: use halo staging whenever the geometry allows
static int g_msub_policy = 1;      // 1: two M sub-tiles per CTA for BN = 128 halo convs
static int g_fuse_policy = 0;      // fused GroupNorm+SiLU on A: off by default (measured slower)
static int g_desc_base_mode = 0;   // descriptor base-offset convention for row-shifted A views
static int g_stage_policy = 0;     // 1: two A halo stages, the rest of smem to B (bit 5 sets; measured
                                   // equal for c128, ~3% slower for the 256-wide c512 / sub-pixel tiles)
static int g_vsub_policy = 1;      // 1: vertical sub-tiles sharing one halo box (bit 6 clears)
static int g_fold_always = 0;      // 1: fold identity residuals into K at every width (bit 7)
static int g_vt_legacy = 0;        // 1: attention V transposed by a kernel instead of MN-major B (bit 9)
static int g_eadd_all = 0;         // bit 29: identity residuals added in the epilogue at every width
static int g_rbuf_policy = 0;      // bit 24: extra K segments (1x1 shortcut, folded identity residual)
                                   // staged through their own buffer between halo taps (rbuf)
static int g_rpf_policy = 1;       // preload conv residuals into the TMEM accumulator: 1 for 128-wide
                                   // outputs (default; 256-wide: the epilogue read measured 10% faster
                                   // on c256), 0 never (bit 10), 2 at every width (bit 20)
static int g_gemm_max_sms = 0;     // diagnostics: cap on the SMs a GEMM grid uses (0 = all)
static int g_rres_policy = 0;      // 1: residual preload via per-warp smem staging (bit 25; half the
                                   // LSU wavefronts, measured neutral: same ms and J/TFLOP sustained)
static int g_pdl_policy = 0;       // 1: programmatic dependent launch of the GEMM kernels (bit 23)
static int g_sched_policy = 0;     // 1: contiguous tile blocks per cluster for conv modes (bit 22 sets;
                                   // measured worse: c128 conv reads 25.5 vs 23.0 GB from DRAM, the
                                   // vertical halo reuse distance outlives L2; decode time neutral)
static int g_rpf_pf = 0;           // 1: L2 prefetch ahead of the residual preload (bit 21 sets;
                                   // measured neutral under the power cap)
static int g_epi_skip = 0;         // diagnostics only (bit 12): skip the epilogue's work
static int g_attn_exp = 1;          // attention softmax fused into the score GEMM (bit 3 clears)
static int g_attn_fallback = 0;     // bit 11: force the fused path's exact-softmax fallback (tests)
static int g_ld_skip = 0;
static int g_small_bn = 1;          // 128-wide tiles for small grids (LBX_SMALL_BN=0 disables; A/B)          // diagnostics only (bits 27 / 28): skip B / A operand loads
static int g_cmap_policy = 1;      // 1: contiguous epilogue column chunks per warp (bit 19 clears)
static int g_tstore_policy = 2;    // TMA-store epilogue: 2 (default) plain GEMMs only -- the attention
                                   // GEMMs gain 13-26% (scores 9.5 -> 8.3 ms per step) -- 1 every
                                   // eligible GEMM (bit 18), 0 none (bit 26); convs keep STG.256, for
                                   // which it measured equal and costs 33 KB of operand stages
static int g_store_mode = 1;       // epilogue stores (bits 16-17 = mode + 1 override): 0 STG.128,
                                   // 1 STG.256 (default: full 32-byte sectors per lane; 3% on c128
                                   // convs, 17% on the score GEMM), 2 streaming STG.128
void gemm_tc_set_debug(int halo_policy, int desc_base_mode) {
  g_halo_policy = halo_policy & 1;
  g_msub_policy = ((halo_policy >> 1) & 1) ? 0 : 1;  // bit 1 disables the two-sub-tile variant
  g_fuse_policy = (halo_policy >> 2) & 1;  // bit 2 enables fused GroupNorm on A in the decoder
  g_desc_base_mode = desc_base_mode;
  g_stage_policy = (halo_policy >> 5) & 1;
  g_vsub_policy = ((halo_policy >> 6) & 1) ? 0 : 1;
  g_fold_always = (halo_policy >> 7) & 1;
  g_vt_legacy = (halo_policy >> 9) & 1;
  g_rpf_policy = ((halo_policy >> 10) & 1) || ((halo_policy >> 29) & 1) ? 0 : ((halo_policy >> 20) & 1) ? 2 : 1;
  g_eadd_all = (halo_policy >> 29) & 1;
  g_rbuf_policy = (halo_policy >> 24) & 1;
  g_rpf_pf = (halo_policy >> 21) & 1;
  g_sched_policy = (halo_policy >> 22) & 1;
  g_pdl_policy = (halo_policy >> 23) & 1;
  g_rres_policy = (halo_policy >> 25) & 1;
  g_tstore_policy = ((halo_policy >> 26) & 1) ? 0 : ((halo_policy >> 18) & 1) ? 1 : 2;
  g_cmap_policy = ((halo_policy >> 19) & 1) ? 0 : 1;
  g_attn_exp = ((halo_policy >> 3) & 1) ? 0 : ((halo_policy >> 30) & 1) ? 2 : 1;  // bit 30: f16x2 exp
  g_attn_fallback = (halo_policy >> 11) & 1;
  g_ld_skip = ((halo_policy >> 27) & 1) | (((halo_policy >> 28) & 1) << 1);
  if (const char* e = std::getenv("LBX_RESID_DIAG")) g_ld_skip |= (std::atoi(e) & 3) << 2;  // 1 zeros, 2 L2 rows
  g_store_mode = ((halo_policy >> 16) & 3) ? (((halo_policy >> 16) & 3) - 1) : 1;
  g_epi_skip = ((halo_policy >> 12) & 1) ? 1 : ((halo_policy >> 13) & 1) ? 2 : ((halo_policy >> 14) & 1) ? 3
                                                                     : ((halo_policy >> 15) & 1) ? 4 : 0;
}

template <int BN, int CG, bool XF, bool RR = false>
static cudaError_t launch_cfg(const GemmArgs& a, KParams kp, cudaStream_t stream) {
  using Cf = Cfg<BN, CG>;
  // ---- operand staging plan (tstore: 32 KB of the budget go to the output staging tiles)
  const int budget = kSmemBudget - ((kp.tstore || kp.rres) ? 33 * 1024 : 0) - kp.r_bytes;
  if (kp.halo) {
    if (kp.vsub) {  // one box of halo_rows + msub - 1 rows; sub-tile s starts 130 s rows in
      kp.halo_sub_bytes = 130 * 128;
      kp.a_tx_bytes = 64 * 130 * (kp.halo_rows + kp.msub - 1) * 2;
      kp.a_stage_bytes = (kp.a_tx_bytes + 1023) & ~1023;
    } else {
      kp.halo_sub_bytes = (64 * 130 * kp.halo_rows * 2 + 1023) & ~1023;
      kp.a_tx_bytes = kp.msub * 64 * 130 * kp.halo_rows * 2;
      kp.a_stage_bytes = kp.msub * kp.halo_sub_bytes;
    }
    // policy 1: a halo stage feeds >= 36 MMAs, so two are enough and the rest of the budget goes to
    // B; policy 0 (default): three A stages when the B tile is small and there is one sub-tile
    if (g_stage_policy || kp.rbuf || ((kp.tstore || kp.rres) && Cf::B_BYTES >= 16384)) kp.a_stages = 2;
    else kp.a_stages = (Cf::B_BYTES >= 32768 || kp.msub > 1) ? 2 : 3;
    kp.b_stages = (budget - kp.a_stages * kp.a_stage_bytes) / Cf::B_BYTES;
  } else {
    kp.a_tx_bytes = kp.a_stage_bytes = 128 * 64 * 2;
    kp.a_stages = kp.b_stages = budget / (kp.a_stage_bytes + Cf::B_BYTES);
  }
  if (kp.a_stages > kMaxStages) kp.a_stages = kMaxStages;
  if (kp.b_stages > kMaxStages) kp.b_stages = kMaxStages;
  if (kp.a_stages < 2 || kp.b_stages < 2) return cudaErrorInvalidValue;
  const int smem = 1024 + kp.a_stages * kp.a_stage_bytes + kp.b_stages * Cf::B_BYTES + kp.r_bytes + (5 * kMaxStages + 6) * 8 + 16 +
                   16 + 8 * (BN / 2) * 4 + ((kp.tstore || kp.rres) ? 1024 + 8 * 2 * 2048 : 0);
  if (smem > Cf::SMEM_MAX) return cudaErrorInvalidValue;

  CUtensorMap tmA, tmB;
  if (a.mode == GEMM_PLAIN) {
    cuuint64_t dims[2] = {(cuuint64_t)a.K, (cuuint64_t)a.M};
    cuuint64_t strides[1] = {(cuuint64_t)a.lda * 2};
    cuuint32_t box[2] = {64, 128};
    if (!make_map(&tmA, a.A, 2, dims, strides, box)) return cudaErrorInvalidValue;
  } else {
    cuuint64_t dims[4] = {(cuuint64_t)a.C, (cuuint64_t)a.W, (cuuint64_t)a.H, (cuuint64_t)a.B_img};
    cuuint64_t strides[3] = {(cuuint64_t)a.C * 2, (cuuint64_t)a.W * a.C * 2, (cuuint64_t)a.H * a.W * a.C * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)(kp.halo ? 130 : kp.Wt),
                         (cuuint32_t)(kp.halo ? kp.halo_rows + (kp.vsub ? kp.msub - 1 : 0) : kp.Ht), 1};
    if (!make_map(&tmA, a.A, 4, dims, strides, box)) return cudaErrorInvalidValue;
  }
  CUtensorMap tmA2;
  if (kp.n_extra) {
    cuuint64_t dims[2] = {(cuuint64_t)a.K2, (cuuint64_t)a.M};
    cuuint64_t strides[1] = {(cuuint64_t)a.lda2 * 2};
    cuuint32_t box[2] = {64, 128};
    if (!make_map(&tmA2, a.A2, 2, dims, strides, box)) return cudaErrorInvalidValue;
  } else {
    tmA2 = tmA;
  }
  CUtensorMap tmO = tmA;
  if (kp.tstore) {  // output [M][N] (row stride ldo): boxes of 32 columns x 32 rows, 64B swizzle
    cuuint64_t dims[2] = {(cuuint64_t)a.N, (cuuint64_t)a.M};
    cuuint64_t strides[1] = {(cuuint64_t)a.ldo * 2};
    cuuint32_t box[2] = {32, 32};
    if (!make_map(&tmO, a.out, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_64B)) return cudaErrorInvalidValue;
  }
  if (kp.b_mn) {  // B stored [K][N] (row stride ldb): boxes of 64 N x 64 K
    cuuint64_t dims[2] = {(cuuint64_t)a.N, (cuuint64_t)(a.b_rows_total ? a.b_rows_total : a.K)};
    cuuint64_t strides[1] = {(cuuint64_t)a.ldb * 2};
    cuuint32_t box[2] = {64, 64};
    if (!make_map(&tmB, a.Bw, 2, dims, strides, box)) return cudaErrorInvalidValue;
  } else {
    const int brows = a.mode == GEMM_SUBPIX ? 4 * a.N : (a.b_rows_total ? a.b_rows_total : a.N);
    cuuint64_t dims[2] = {(cuuint64_t)(a.K + a.K2), (cuuint64_t)brows};
    cuuint64_t strides[1] = {(cuuint64_t)a.ldb * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)Cf::B_ROWS};
    if (!make_map(&tmB, a.Bw, 2, dims, strides, box)) return cudaErrorInvalidValue;
  }
  auto kern = gemm_tc_kernel<BN, CG, XF, RR>;
  const int sms = num_sms();
  int clusters = (g_gemm_max_sms > 0 && g_gemm_max_sms < sms ? g_gemm_max_sms : sms) / CG;
  if (kp.gn_stats && !kp.sched) {
    // GroupNorm statistics are summed per lane over the tiles of one image that a cluster visits:
    // tile j of an image goes to cluster (img * T + j) mod G, so the tiles summed together are a
    // residue class of j mod G -- the same for every image as long as G does not change with the
    // batch.  G = the full grid when an image has >= that many tiles; otherwise a multiple of T
    // (each cluster then sees at most one tile per image, exactly as a solo decode does).
    const long long imgs = (long long)a.M / a.rows_per_img;
    const int T = imgs > 0 ? (int)(kp.tiles / imgs) : kp.tiles;
    if (T > 0 && T < clusters) clusters = T * (clusters / T);
  }
  if (clusters > kp.tiles) clusters = kp.tiles;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(clusters * CG);
  cfg.blockDim = dim3(XF ? Cf::THREADS_XF : Cf::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (kp.pdl) {
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = 2;
  }
  return cudaLaunchKernelEx(&cfg, kern, tmA, tmB, tmA2, tmO, kp);
}

template <int BN, int CG>
static bool set_attr() {
  return ensure_smem_attr(reinterpret_cast<const void*>(gemm_tc_kernel<BN, CG, false>), Cfg<BN, CG>::SMEM_MAX) &&
         ensure_smem_attr(reinterpret_cast<const void*>(gemm_tc_kernel<BN, CG, true>), Cfg<BN, CG>::SMEM_MAX) &&
         (BN != 256 || ensure_smem_attr(reinterpret_cast<const void*>(gemm_tc_kernel<256, CG, false, true>),
                                        Cfg<256, CG>::SMEM_MAX));
}

bool ensure_smem_attr(const void* func, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  std::lock_guard<std::mutex> g(mu);
  int& have = done[{dev, func}];
  if (have >= bytes) return true;
  if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return false;
  have = bytes;
  return true;
}

bool gemm_tc_prepare() {  // per device (a multi-GPU batcher drives several from one process)
  num_sms();
  static const bool env_read = [] {
    if (const char* e = std::getenv("LBX_SMALL_BN")) g_small_bn = std::atoi(e);
    return true;
  }();
  (void)env_read;
  return tma_available() && set_attr<256, 2>() && set_attr<128, 2>() && set_attr<256, 1>() && set_attr<128, 1>();
}

bool resid_fold_always() { return g_fold_always != 0; }
bool v_transpose_legacy() { return g_vt_legacy != 0; }
bool attn_fused_exp() { return g_attn_exp != 0; }
bool attn_force_fallback() { return g_attn_fallback != 0; }
bool resid_preload() { return g_rpf_policy != 0; }
bool resid_epilogue_all() { return g_eadd_all != 0; }
bool resid_rbuf() { return g_rbuf_policy != 0; }
bool pdl_enabled() { return g_pdl_policy != 0; }
void gemm_tc_set_max_sms(int n) { g_gemm_max_sms = n; }

bool gemm_tc_can_fuse_gn(const GemmArgs& a) {
  // halo staging (128-pixel row segments); four extra warps transform each landed halo
  // LBX_FUSE_C (diagnostics): with bit 2, fuse only the convs with this many input channels
  static const int fuse_c = std::getenv("LBX_FUSE_C") ? std::atoi(std::getenv("LBX_FUSE_C")) : 0;
  if (fuse_c && a.C != fuse_c) return false;
  return g_fuse_policy && g_halo_policy && a.mode == GEMM_CONV3X3 && a.W >= 128 && a.W % 128 == 0 &&
         a.N % 128 == 0 && a.C % 64 == 0 && a.M % 256 == 0;
}

cudaError_t gemm_tc_launch(const GemmArgs& a, cudaStream_t stream, int force_cg, int force_bn) {
  if (!gemm_tc_prepare()) return cudaErrorNotSupported;
  if (a.M <= 0 || a.N <= 0 || a.K <= 0 || a.K % 64) return cudaErrorInvalidValue;
  KParams kp = {};
  kp.mode = a.mode;
  kp.M = a.M; kp.N = a.N; kp.K = a.K;
  kp.num_kb = a.K / 64;
  kp.k_main = a.K;
  if (a.K2) {
    if (a.K2 % 64 || !a.A2 || a.lda2 < a.K2 || a.mode == GEMM_SUBPIX) return cudaErrorInvalidValue;
    kp.n_extra = a.K2 / 64;
  }
  if (a.mode != GEMM_PLAIN) {
    if (a.C % 64 || a.M != a.B_img * a.H * a.W) return cudaErrorInvalidValue;
    if (a.K != (a.mode == GEMM_CONV3X3 ? 9 : 4) * a.C) return cudaErrorInvalidValue;
    kp.cblocks = a.C / 64;
    kp.H = a.H; kp.W = a.W;
    kp.Wt = a.W < 128 ? a.W : 128;
    if (128 % kp.Wt || (a.W > 128 && a.W % 128)) return cudaErrorInvalidValue;
    kp.Ht = 128 / kp.Wt;
    if (a.H % kp.Ht) return cudaErrorInvalidValue;
    kp.taps = a.mode == GEMM_CONV3X3 ? 9 : 4;
    kp.halo_rows = a.mode == GEMM_CONV3X3 ? 3 : 2;
    kp.halo = (g_halo_policy && kp.Ht == 1) ? 1 : 0;  // a tap's 128 rows must be contiguous in the halo
    kp.desc_base_mode = g_desc_base_mode;
  }
  if (a.batch_m) {  // batched plain GEMM: tiles never straddle images
    if (a.mode != GEMM_PLAIN || a.K2 || a.batch_m % 256 || a.M % a.batch_m || a.b_rows_total <= 0)
      return cudaErrorInvalidValue;
    kp.batch_m = a.batch_m;
    kp.batch_b = a.batch_b;
  }
  if (a.b_mn_major) {  // plain GEMM only, no extra K segment
    if (a.mode != GEMM_PLAIN || a.K2 || a.N % 64) return cudaErrorInvalidValue;
    kp.b_mn = 1;
  }
  kp.out = a.out; kp.ldo = a.ldo; kp.bias = a.bias; kp.resid = a.resid; kp.ldr = a.ldr;
  // residual preload into TMEM: conv mode, unscaled outputs (the preload would be scaled too)
  kp.epi_skip = g_epi_skip;
  kp.ld_skip = g_ld_skip;
  kp.store_mode = g_store_mode;
  kp.cmap = g_cmap_policy;
  if (kp.store_mode == 1 && ((reinterpret_cast<uintptr_t>(a.out) & 31) || (a.ldo % 16))) kp.store_mode = 0;
  // TMA-store epilogue: rows of a warp's chunk are contiguous output rows (not the sub-pixel
  // phases), 16-byte aligned rows, no XF transform warps
  kp.tstore = (g_tstore_policy && (g_tstore_policy == 1 || a.mode == GEMM_PLAIN) && a.mode != GEMM_SUBPIX && !a.gn_ss && !(reinterpret_cast<uintptr_t>(a.out) & 15) &&
               a.ldo % 8 == 0) ? 1 : 0;
  kp.rpf = (a.resid && a.mode == GEMM_CONV3X3 && !a.row_scale && a.alpha == 1.f && !a.gn_ss && g_rpf_policy &&
            (g_rpf_policy == 2 || a.N <= 128)) ? 1 : 0;
  kp.rpf_pf = g_rpf_pf;
  static const int a_hint = std::getenv("LBX_A_HINT") ? std::atoi(std::getenv("LBX_A_HINT")) : 0;
  kp.a_hint = (a_hint && a.mode != GEMM_PLAIN) ? 1 : 0;
  kp.sched = (g_sched_policy && a.mode != GEMM_PLAIN) ? 1 : 0;
  kp.pdl = g_pdl_policy;
  kp.rres = (kp.rpf && g_rres_policy && !kp.tstore && a.ldr % 8 == 0) ? 1 : 0;
  kp.row_scale = a.row_scale; kp.alpha = a.alpha;
  kp.run_if = a.run_if;
  kp.run_if_n = a.run_if ? std::max(1, a.run_if_n) : 0;
  if (a.rowred) {  // plain GEMM, 256-wide tiles (two column halves per tile), nothing else in the epilogue
    if (a.mode != GEMM_PLAIN || a.bias || a.resid || a.gn_stats || a.row_scale || !a.row_part ||
        (a.rowred == 2 && (!a.row_max || !a.exp_flag)) || a.rowred > 2 || a.N % 256 || force_bn == 128)
      return cudaErrorInvalidValue;
    kp.rowred = a.rowred; kp.row_max = a.row_max; kp.row_part = a.row_part; kp.exp_flag = a.exp_flag;
    kp.exp_force = a.exp_force;
    kp.exp_h2 = g_attn_exp == 2 ? 1 : 0;
  }
  kp.gn_stats = a.gn_stats; kp.gn_cpg = a.gn_cpg; kp.rows_per_img = a.rows_per_img;
  if (a.gn_stats && (!(a.gn_cpg == 4 || a.gn_cpg == 8 || a.gn_cpg == 16) || a.N != 32 * a.gn_cpg ||
                     a.rows_per_img <= 0))
    return cudaErrorInvalidValue;
  if (a.mode == GEMM_SUBPIX && a.resid) return cudaErrorInvalidValue;

  int bn = force_bn ? force_bn : (a.N % 256 == 0 ? 256 : 128);
  if (a.N % bn) return cudaErrorInvalidValue;
  int cg = force_cg ? force_cg : ((a.M % 256 == 0) ? 2 : 1);
  if (!force_bn && bn == 256 && !a.rowred && g_small_bn) {
    // small grids (the 64x64 layers and the attention of a 512^2 decode): when 256-wide tiles
    // would leave clusters idle, 128-wide ones double the tiles.  With GroupNorm statistics the
    // rule looks at one image's tiles, so the choice -- and with it which values a lane sums in
    // fp32 -- does not depend on the batch (decodes stay bit-identical across batch sizes); plain
    // GEMM outputs do not depend on the tile width at all (same K order per element).
    const long long rows = a.gn_stats ? (long long)a.rows_per_img : (long long)a.M;
    const long long t256 = rows / (128 * cg) * (a.N / 256) * (a.mode == GEMM_SUBPIX ? 4 : 1);
    if (t256 < num_sms() / cg) bn = 128;
  }
  if (a.M % (128 * cg)) return cudaErrorInvalidValue;
  kp.msub = (kp.halo && g_msub_policy && bn == 128 && cg == 2 && a.mode == GEMM_CONV3X3 && a.W % 256 == 0 &&
             a.M % (512 * cg) == 0) ? 2 : 1;
  kp.vsub = (kp.msub == 2 && g_vsub_policy && a.H % 2 == 0 && a.W % (128 * cg) == 0) ? 1 : 0;
  kp.tmem_cols = 2 * bn * kp.msub;
  kp.m_tiles = a.M / (128 * cg * kp.msub);
  if (kp.vsub) {
    kp.segs = a.W / (128 * cg);
    kp.per_img = (a.H / kp.msub) * kp.segs;
    kp.fd_segs = FastDiv((uint32_t)kp.segs);
    kp.fd_per_img = FastDiv((uint32_t)kp.per_img);
  }
  kp.n_tiles = a.N / bn;
  kp.fd_ntiles = FastDiv((uint32_t)kp.n_tiles);
  kp.fd_rpi = FastDiv((uint32_t)(a.rows_per_img > 0 ? a.rows_per_img : 1));
  kp.tiles = kp.m_tiles * kp.n_tiles * (a.mode == GEMM_SUBPIX ? 4 : 1);
  // rbuf: conv halo mode with an extra segment of at most one k-block per tap (not with XF)
  kp.rbuf = (g_rbuf_policy && kp.n_extra && kp.halo && a.mode == GEMM_CONV3X3 && !a.gn_ss &&
             kp.n_extra <= kp.cblocks * kp.taps) ? 1 : 0;
  kp.r_bytes = kp.rbuf ? kp.msub * 16384 : 0;
  if (a.gn_ss) {  // fused GroupNorm + SiLU on the A operand: conv3x3 halo staging only
    if (a.mode != GEMM_CONV3X3 || !kp.halo) return cudaErrorInvalidValue;
    kp.gn_ss = a.gn_ss;
    if (bn == 256 && cg == 2) return launch_cfg<256, 2, true>(a, kp, stream);
    if (bn == 128 && cg == 2) return launch_cfg<128, 2, true>(a, kp, stream);
    if (bn == 256 && cg == 1) return launch_cfg<256, 1, true>(a, kp, stream);
    return launch_cfg<128, 1, true>(a, kp, stream);
  }
  if (kp.rowred) {  // bn == 256 (checked above)
    if (cg == 2) return launch_cfg<256, 2, false, true>(a, kp, stream);
    return launch_cfg<256, 1, false, true>(a, kp, stream);
  }
  if (bn == 256 && cg == 2) return launch_cfg<256, 2, false>(a, kp, stream);
  if (bn == 128 && cg == 2) return launch_cfg<128, 2, false>(a, kp, stream);
  if (bn == 256 && cg == 1) return launch_cfg<256, 1, false>(a, kp, stream);
  return launch_cfg<128, 1, false>(a, kp, stream);
}

}  // namespace lbx
