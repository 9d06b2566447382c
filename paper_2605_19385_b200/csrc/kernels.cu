// HBM-bound kernels of the reconstruction path (SURVEY.md 2.4 K1/K5/K7 and the attention glue).
// All are vectorised (16-byte global accesses), grid-stride, sized in multiples of the SM count.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "act.cuh"
#include "gemm_tc.cuh"
#include "gnfix.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace lbx {

static inline int grid_for(long long work, int threads, int per_sm = 8) {
  long long g = (work + threads - 1) / threads;
  long long cap = (long long)num_sms() * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// ----------------------------------------------------------------------------- latent prep
__global__ void latent_prep_kernel(const __half* __restrict__ lat, __half* __restrict__ out, int n, int cl, int h,
                                   int w, float scaling, float shift, const float* __restrict__ pq_w,
                                   const float* __restrict__ pq_b) {
  const long long pix = (long long)n * h * w;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < pix; p += (long long)gridDim.x * blockDim.x) {
    const long long img = p / (h * w);
    const int rem = (int)(p - img * h * w);
    float z[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      if (c < cl) {
        const float v = __half2float(lat[(img * cl + c) * h * w + rem]);
        z[c] = __fadd_rn(__fdiv_rn(v, scaling), shift);
      } else {
        z[c] = 0.f;
      }
    }
    if (pq_w) {
      float y[16];
#pragma unroll
      for (int o = 0; o < 16; ++o) {
        if (o < cl) {
          float a = pq_b[o];
          for (int c = 0; c < cl; ++c) a = fmaf(pq_w[o * cl + c], z[c], a);
          y[o] = a;
        } else {
          y[o] = 0.f;
        }
      }
#pragma unroll
      for (int o = 0; o < 16; ++o) z[o] = y[o];
    }
    uint4 pk[8];
    __half2* h2 = reinterpret_cast<__half2*>(pk);
#pragma unroll
    for (int i = 0; i < 8; ++i) h2[i] = __floats2half2_rn(z[2 * i], z[2 * i + 1]);
#pragma unroll
    for (int i = 2; i < 8; ++i) pk[i] = make_uint4(0, 0, 0, 0);
    uint4* o4 = reinterpret_cast<uint4*>(out + p * 64);
#pragma unroll
    for (int i = 0; i < 8; ++i) o4[i] = pk[i];
  }
}

void launch_latent_prep(const __half* lat, __half* out, int n, int cl, int h, int w, float scaling, float shift,
                        const float* pq_w, const float* pq_b, cudaStream_t s) {
  const long long pix = (long long)n * h * w;
  latent_prep_kernel<<<grid_for(pix, 256), 256, 0, s>>>(lat, out, n, cl, h, w, scaling, shift, pq_w, pq_b);
}

// ----------------------------------------------------------------------------- GroupNorm
__global__ void gn_finalize_kernel(const unsigned long long* __restrict__ stats, const float* __restrict__ gamma,
                                   const float* __restrict__ beta, float2* __restrict__ ss, int n, int C,
                                   double inv_count, float eps) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * C) return;
  const int img = i / C, c = i - img * C;
  const int g = c / (C / 32);
  const unsigned long long* st = stats + ((size_t)img * 32 + g) * kGnStatWords;
  ss[i] = gn_affine(gnfix_value(st), gnfix_value(st + 2), inv_count, gamma[c], beta[c], eps);
}

void launch_gn_finalize(const unsigned long long* stats, const float* gamma, const float* beta, float2* ss, int n, int C,
                        double count, float eps, cudaStream_t s) {
  gn_finalize_kernel<<<(n * C + 255) / 256, 256, 0, s>>>(stats, gamma, beta, ss, n, C, 1.0 / count, eps);
}

// The apply kernels finalize the statistics themselves (the same gn_affine arithmetic as
// gn_finalize_kernel, so results are bit-identical): one launch per GroupNorm site instead of two.
__device__ __forceinline__ float2 site_affine(const GnSrc& g, int img, int c, int cpg) {
  const unsigned long long* st = g.stats + ((size_t)img * 32 + c / cpg) * kGnStatWords;
  const unsigned long long w[4] = {__ldg(st), __ldg(st + 1), __ldg(st + 2), __ldg(st + 3)};
  return gn_affine(gnfix_value(w), gnfix_value(w + 2), g.inv_count, __ldg(g.gamma + c), __ldg(g.beta + c), g.eps);
}

// y = act(x * a_c + b_c).  The launch is exactly one resident wave; block b covers a contiguous
// range of the flattened (image, pixel) space, split at image boundaries.  Thread t owns channel
// octet t % (C/8) for every pixel it visits, so its 8 affine pairs are reloaded only per image.
template <bool SILU, int CV, bool H2>
__global__ void __launch_bounds__(256) gn_apply_kernel(const __half* x, __half* y, const GnSrc g, int hw,
                                                       long long total, long long pix_per_block) {
  constexpr int PSTEP = 256 / CV;  // pixels advanced per iteration of the block
  const int cvec = threadIdx.x % CV;
  const long long end = min(total, (blockIdx.x + 1) * pix_per_block);
  long long p = blockIdx.x * pix_per_block + threadIdx.x / CV;
  const uint4* xv = reinterpret_cast<const uint4*>(x) + cvec;
  uint4* yv = reinterpret_cast<uint4*>(y) + cvec;
  while (p < end) {
    const int img = (int)(p / hw);
    const long long seg_end = min(end, (long long)(img + 1) * hw);
    float a[8], b[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float2 t = site_affine(g, img, cvec * 8 + k, CV / 4);
      a[k] = (SILU && H2) ? 0.5f * t.x : t.x;  // halved for gn_silu8_h2_half
      b[k] = (SILU && H2) ? 0.5f * t.y : t.y;
    }
    auto apply = [&](uint4 u) { return (SILU && H2) ? gn_silu8_h2_half(u, a, b) : gn_act8<SILU>(u, a, b); };
    constexpr int U = 8;  // 16-byte loads in flight per thread (latency x bandwidth needs ~100 KB/SM)
    for (; p + (U - 1) * PSTEP < seg_end; p += U * PSTEP) {
      uint4 u[U];
#pragma unroll
      for (int i = 0; i < U; ++i) u[i] = __ldcs(xv + (size_t)(p + i * PSTEP) * CV);
#pragma unroll
      for (int i = 0; i < U; ++i) __stcs(yv + (size_t)(p + i * PSTEP) * CV, apply(u[i]));
    }
    for (; p < seg_end; p += PSTEP) __stcs(yv + (size_t)p * CV, apply(__ldcs(xv + (size_t)p * CV)));
  }
}

// Bulk-copy form of the same apply (default): one persistent CTA per SM streams 32 KB chunks
// through a 4-stage smem ring with 1-D TMA (cp.async.bulk global -> smem, mbarrier completion),
// all 256 threads rewrite the chunk in smem, and one thread writes it back with a bulk store
// (cp.async.bulk smem -> global, bulk_group).  Three loads stay in flight per SM without holding
// registers, so the stream runs closer to copy bandwidth than the register-staged kernel above.
// A chunk never straddles an image (every image is a multiple of 32 KB), and thread t always
// owns channel octet t mod CV (256 is a multiple of CV), so its 8 affine pairs change only with
// the image.
#ifndef LBX_AP_STAGES
#define LBX_AP_STAGES 4
#endif
constexpr int kApChunk = 32768, kApStages = LBX_AP_STAGES;

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   ptx::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(ptx::smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(ptx::smem_u32(src)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

template <bool SILU, int CV, bool H2>
__global__ void __launch_bounds__(256, 1) gn_apply_bulk_kernel(const __half* x, __half* y, const GnSrc g,
                                                              long long img_bytes, long long chunks) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* ring = smem_raw;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kApStages * kApChunk);
  const int tid = threadIdx.x;
  const int cvec = tid % CV;
  if (tid == 0) {
    for (int i = 0; i < kApStages; ++i) ptx::mbar_init(&full[i], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");  // no-op unless launched as a PDL dependent
  const uint8_t* src = reinterpret_cast<const uint8_t*>(x);
  uint8_t* dst = reinterpret_cast<uint8_t*>(y);
  const long long first = blockIdx.x, step = gridDim.x;
  const long long mine = first < chunks ? (chunks - first + step - 1) / step : 0;
  constexpr int P = kApStages - 1;  // loads in flight
  if (tid == 0) {
    for (long long k = 0; k < P && k < mine; ++k) {
      ptx::mbar_arrive_expect_tx(&full[k], kApChunk);
      bulk_load(ring + k * kApChunk, src + (first + k * step) * kApChunk, kApChunk, &full[k]);
    }
  }
  int cur_img = -1, pf_img = -1;
  float a[8], b[8], na[8], nb[8];
  // the next image's statistics: loaded while the current chunk is rewritten, finalized after it,
  // so an image change no longer stalls on dependent L2 loads (small images change every few chunks)
  unsigned long long pw[8][4];
  float pg[8], pb[8];
  // chunk -> image with 32-bit arithmetic (a 64-bit divide per chunk was a measurable share of the
  // issue slots): the chunk count stays far below 2^32 and an image is a whole number of chunks
  const uint32_t cpi = (uint32_t)(img_bytes / kApChunk);
  for (long long k = 0; k < mine; ++k) {
    const int st = (int)(k % kApStages);
    const long long c = first + k * step;
    const int img = (int)((uint32_t)c / cpi);
    if (img != cur_img) {  // this thread's 8 channels of the new image
      if (img == pf_img) {
#pragma unroll
        for (int j = 0; j < 8; ++j) { a[j] = na[j]; b[j] = nb[j]; }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float2 t = site_affine(g, img, cvec * 8 + j, CV / 4);
          a[j] = (SILU && H2) ? 0.5f * t.x : t.x;  // halved for gn_silu8_h2_half
          b[j] = (SILU && H2) ? 0.5f * t.y : t.y;
        }
      }
      cur_img = img;
    }
    const int img_n = k + 1 < mine ? (int)((uint32_t)(c + step) / cpi) : -1;
    const bool pf = img_n >= 0 && img_n != img && img_n != pf_img;
    if (pf) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int ch = cvec * 8 + j;
        const unsigned long long* stp = g.stats + ((size_t)img_n * 32 + ch / (CV / 4)) * kGnStatWords;
#pragma unroll
        for (int w = 0; w < 4; ++w) pw[j][w] = __ldg(stp + w);
        pg[j] = __ldg(g.gamma + ch);
        pb[j] = __ldg(g.beta + ch);
      }
    }
    ptx::mbar_wait(&full[st], (uint32_t)((k / kApStages) & 1));
    uint4* q = reinterpret_cast<uint4*>(ring + st * kApChunk);
#pragma unroll
    for (int i = 0; i < kApChunk / 16 / 256; ++i) {
      const uint4 u = q[tid + 256 * i];
      q[tid + 256 * i] = (SILU && H2) ? gn_silu8_h2_half(u, a, b) : gn_act8<SILU>(u, a, b);
    }
    if (pf) {  // the same gn_affine arithmetic as site_affine (bit-identical)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float2 t = gn_affine(gnfix_value(pw[j]), gnfix_value(pw[j] + 2), g.inv_count, pg[j], pb[j], g.eps);
        na[j] = (SILU && H2) ? 0.5f * t.x : t.x;
        nb[j] = (SILU && H2) ? 0.5f * t.y : t.y;
      }
      pf_img = img_n;
    }
    ptx::fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the bulk store
    __syncthreads();
    if (tid == 0) {
      bulk_store(dst + c * kApChunk, ring + st * kApChunk, kApChunk);
      if (k + P < mine) {
        // the refill targets the stage of chunk k-1: its store must have finished reading smem
        bulk_wait_read<1>();
        const int ns = (int)((k + P) % kApStages);
        ptx::mbar_arrive_expect_tx(&full[ns], kApChunk);
        bulk_load(ring + ns * kApChunk, src + (first + (k + P) * step) * kApChunk, kApChunk, &full[ns]);
      }
    }
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

static int g_apply_max_sms = 0;  // diagnostics: cap on the SMs a bulk GroupNorm apply uses
void kernels_set_apply_max_sms(int n) { g_apply_max_sms = n; }
static bool g_apply_bulk = true;  // bulk-copy apply (debug bit 8 selects the register-staged one)
void kernels_set_apply_bulk(bool on) { g_apply_bulk = on; }

template <bool SILU, int CV, bool H2>
static bool gn_apply_bulk_launch(const __half* x, __half* y, const GnSrc& g, int n, int hw, cudaStream_t s) {
  const long long img_bytes = (long long)hw * CV * 16;
  // 6.3-6.45 TB/s at 128/256/512 channels alone (97% of the measured copy rate) vs 5.9-6.0 for
  // the register-staged kernel (scripts/op_bench.py gn)
  if (!g_apply_bulk || img_bytes % kApChunk) return false;
  constexpr int smem = kApStages * kApChunk + kApStages * 8;
  if (!ensure_smem_attr(reinterpret_cast<const void*>(gn_apply_bulk_kernel<SILU, CV, H2>), smem)) return false;
  const long long chunks = (long long)n * img_bytes / kApChunk;
  const int sms = g_apply_max_sms > 0 && g_apply_max_sms < num_sms() ? g_apply_max_sms : num_sms();
  const int grid = (int)(chunks < sms ? chunks : sms);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, gn_apply_bulk_kernel<SILU, CV, H2>, x, y, g, img_bytes, chunks);
  return true;
}

static bool g_conv_out_legacy = false;  // CUDA-core conv_out instead of the tensor-core tail
void kernels_set_conv_out_legacy(bool on) { g_conv_out_legacy = on; }
bool kernels_conv_out_legacy() { return g_conv_out_legacy; }

template <bool SILU, int CV, bool H2>
static void gn_apply_launch(const __half* x, __half* y, const GnSrc& g, int n, int hw, cudaStream_t s) {
  if (gn_apply_bulk_launch<SILU, CV, H2>(x, y, g, n, hw, s)) return;
  static int occ = 0;
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gn_apply_kernel<SILU, CV, H2>, 256, 0);
    if (occ <= 0) occ = 4;
  }
  constexpr int PSTEP = 256 / CV;
  const long long total = (long long)n * hw;
  const long long blocks = (long long)num_sms() * occ;
  long long ppb = (total + blocks - 1) / blocks;
  ppb = (ppb + PSTEP - 1) / PSTEP * PSTEP;
  const int grid = (int)((total + ppb - 1) / ppb);
  gn_apply_kernel<SILU, CV, H2><<<grid, 256, 0, s>>>(x, y, g, hw, total, ppb);
}

template <bool SILU, bool H2>
static void gn_apply_dispatch(const __half* x, __half* y, const GnSrc& g, int n, int hw, int C, cudaStream_t s) {
  switch (C / 8) {
    case 16: gn_apply_launch<SILU, 16, H2>(x, y, g, n, hw, s); break;
    case 32: gn_apply_launch<SILU, 32, H2>(x, y, g, n, hw, s); break;
    case 64: gn_apply_launch<SILU, 64, H2>(x, y, g, n, hw, s); break;
    default: break;  // C validated by callers (128 / 256 / 512)
  }
}

void launch_gn_apply(const __half* x, __half* y, const GnSrc& g, long long rows, int hw, int C, bool silu, bool h2,
                     cudaStream_t s) {
  const int n = (int)(rows / hw);
  if (silu) {
    if (h2) gn_apply_dispatch<true, true>(x, y, g, n, hw, C, s);
    else gn_apply_dispatch<true, false>(x, y, g, n, hw, C, s);
  } else {
    gn_apply_dispatch<false, false>(x, y, g, n, hw, C, s);
  }
}

// Deterministic: each thread sums a fixed pixel subset of one channel octet in fp32, the block
// combines its threads in a fixed order through shared memory, and the block totals are added as
// exact fixed-point integers (gnfix.cuh) -- bit-identical across runs and schedules.
__global__ void __launch_bounds__(256) gn_stats_kernel(const __half* __restrict__ x, unsigned long long* stats,
                                                       int hw, int C) {
  __shared__ float part[256][17];
  const int img = blockIdx.y;
  const int cpg = C / 32;
  const int cv = C / 8;
  const long long vecs = (long long)hw * cv;
  const uint4* xv = reinterpret_cast<const uint4*>(x + (size_t)img * hw * C);
  float s[8], s2[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { s[j] = 0.f; s2[j] = 0.f; }
  // each thread keeps a fixed channel octet so its partial sums stay per channel
  const int stride = gridDim.x * blockDim.x;  // a multiple of C/8 (see launch_gn_stats)
  const int first = blockIdx.x * blockDim.x + threadIdx.x;
  for (long long v = first; v < vecs; v += stride) {
    uint4 u = xv[v];
    const __half2* h2 = reinterpret_cast<const __half2*>(&u);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = __half22float2(h2[j]);
      s[2 * j] += f.x; s2[2 * j] += f.x * f.x;
      s[2 * j + 1] += f.y; s2[2 * j + 1] += f.y * f.y;
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    part[threadIdx.x][j] = s[j];
    part[threadIdx.x][8 + j] = s2[j];
  }
  __syncthreads();
  if (threadIdx.x < 64) {  // value (group g, kind k): fixed-order sum over the block's threads
    const int g = threadIdx.x >> 1, k = threadIdx.x & 1;
    float acc = 0.f;
    for (int t = 0; t < 256; ++t) {
      const int c0 = ((blockIdx.x * blockDim.x + t) % cv) * 8;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if ((c0 + j) / cpg == g) acc += part[t][8 * k + j];
    }
    gnfix_add(stats + ((size_t)img * 32 + g) * kGnStatWords + 2 * k, acc);
  }
}

void launch_gn_stats(const __half* x, unsigned long long* stats, int n, int hw, int C, cudaStream_t s) {
  // 256 threads x 64 blocks per image: stride 16384 vectors, a multiple of C/8 for C <= 512
  dim3 grid(64, n);
  gn_stats_kernel<<<grid, 256, 0, s>>>(x, stats, hw, C);
}

// ----------------------------------------------------------------------------- softmax
// One 256-thread block per row; the row (<= 16384 fp16 = 32 KiB) is held in registers.
template <int VPT>  // 16-byte vectors per thread
__global__ void __launch_bounds__(256) softmax_rows_kernel(__half* S, float* row_scale, int rows, int cols,
                                                           const int* run_if) {
  if (run_if && *reinterpret_cast<const volatile int*>(run_if) == 0) return;
  __shared__ float red[8];
  for (int rix = blockIdx.x; rix < rows; rix += gridDim.x) {  // grid = rows, or one wave when guarded
  __syncthreads();  // red[] of the previous row is consumed
  __half* row = S + (size_t)rix * cols;
  const int nvec = cols / 8;
  uint4 u[VPT];
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int v = threadIdx.x + i * 256;
    if (v < nvec) {
      u[i] = reinterpret_cast<const uint4*>(row)[v];
      const __half2* h2 = reinterpret_cast<const __half2*>(&u[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 f = __half22float2(h2[j]);
        mx = fmaxf(mx, fmaxf(f.x, f.y));
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = red[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) mx = fmaxf(mx, red[i]);
  __syncthreads();
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int v = threadIdx.x + i * 256;
    if (v < nvec) {
      __half2* h2 = reinterpret_cast<__half2*>(&u[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 f = __half22float2(h2[j]);
        const float e0 = __expf(f.x - mx), e1 = __expf(f.y - mx);
        const __half2 e = __floats2half2_rn(e0, e1);
        const float2 er = __half22float2(e);
        sum += er.x + er.y;  // sum the values actually used by P*V
        h2[j] = e;
      }
      reinterpret_cast<uint4*>(row)[v] = u[i];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int i = 0; i < 8; ++i) t += red[i];
    row_scale[rix] = 1.0f / t;
  }
  }
}

void launch_softmax_rows(__half* S, float* row_scale, int rows, int cols, cudaStream_t s, const int* run_if) {
  const int nvec = cols / 8;
  // guarded (fallback) launches are one wave of row-looping blocks, so the usual early exit is cheap
  const int grid = run_if ? std::min(rows, num_sms() * 8) : rows;
  if (nvec <= 256 * 2) softmax_rows_kernel<2><<<grid, 256, 0, s>>>(S, row_scale, rows, cols, run_if);
  else if (nvec <= 256 * 4) softmax_rows_kernel<4><<<grid, 256, 0, s>>>(S, row_scale, rows, cols, run_if);
  else softmax_rows_kernel<8><<<grid, 256, 0, s>>>(S, row_scale, rows, cols, run_if);
}

// Row sums of the fused-exp score GEMM (GemmArgs::rowred 2): row_scale[r] = 1 / (sum of the row's
// nparts partial sums).  One warp per row; lane l adds parts l, l + 32, ... in order and the lanes
// combine through a fixed butterfly, so the result does not depend on the batch or the grid.
// MAX = true: out[2r] = max of the row's parts, out[2r + 1] = -inf (the exact row maximum of the
// fallback, in the sampled-maximum layout the score GEMM reads).  Guarded launches (run_if) are one
// wave of row-looping warps that exit at once unless the group was flagged.
template <bool MAX>
__global__ void __launch_bounds__(256) attn_rowred_kernel(const float* __restrict__ part, int nparts,
                                                          float* __restrict__ out, int rows, const int* run_if,
                                                          int rows_per_img) {
  const int lane = threadIdx.x & 31;
  if (run_if) {  // per-image guards: nothing to do unless some image of the launch is flagged
    int any = 0;
    for (int i = 0; i < rows / rows_per_img; ++i) any |= reinterpret_cast<const volatile int*>(run_if)[i];
    if (!any) return;
  }
  for (int r = blockIdx.x * 8 + (threadIdx.x >> 5); r < rows; r += gridDim.x * 8) {
    if (run_if && reinterpret_cast<const volatile int*>(run_if)[r / rows_per_img] == 0) continue;
    const float* pr = part + (size_t)r * nparts;
    float t = MAX ? -INFINITY : 0.f;
    for (int i = lane; i < nparts; i += 32) t = MAX ? fmaxf(t, pr[i]) : t + pr[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float u = __shfl_xor_sync(0xffffffffu, t, o);
      t = MAX ? fmaxf(t, u) : t + u;
    }
    if (lane == 0) {
      if (MAX) {
        out[2 * (size_t)r] = t;
        out[2 * (size_t)r + 1] = -INFINITY;
      } else {
        out[r] = 1.0f / t;
      }
    }
  }
}

void launch_attn_rowsum(const float* part, int nparts, float* row_scale, int rows, cudaStream_t s, const int* run_if,
                        int rows_per_img) {
  const int grid = run_if ? std::min((rows + 7) / 8, num_sms() * 8) : (rows + 7) / 8;
  attn_rowred_kernel<false><<<grid, 256, 0, s>>>(part, nparts, row_scale, rows, run_if, rows_per_img);
}

// counter += number of flagged images (the decoder's lbx_decoder_counters.attn_fallbacks)
__global__ void attn_count_kernel(const int* __restrict__ flags, int groups, unsigned long long* counter) {
  unsigned long long c = 0;
  for (int i = 0; i < groups; ++i) c += flags[i] != 0;
  if (c) atomicAdd(counter, c);
}

void launch_attn_count(const int* flags, int groups, unsigned long long* counter, cudaStream_t s) {
  attn_count_kernel<<<1, 1, 0, s>>>(flags, groups, counter);
}

void launch_attn_rowmax(const float* part, int nparts, float* row_max2, int rows, cudaStream_t s, const int* run_if,
                        int rows_per_img) {
  const int grid = run_if ? std::min((rows + 7) / 8, num_sms() * 8) : (rows + 7) / 8;
  attn_rowred_kernel<true><<<grid, 256, 0, s>>>(part, nparts, row_max2, rows, run_if, rows_per_img);
}

// ----------------------------------------------------------------------------- transpose
__global__ void transpose_kernel(const __half* __restrict__ in, int ldi, __half* __restrict__ out, int ldo, int R,
                                 int Cc) {
  __shared__ __half tile[32][33];
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    if (r < R && c < Cc) tile[i][threadIdx.x] = in[(size_t)r * ldi + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (r < R && c < Cc) out[(size_t)c * ldo + r] = tile[threadIdx.x][i];
  }
}

void launch_transpose(const __half* in, int ldi, __half* out, int ldo, int R, int Cc, cudaStream_t s) {
  dim3 grid((Cc + 31) / 32, (R + 31) / 32);
  transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(in, ldi, out, ldo, R, Cc);
}

// ----------------------------------------------------------------------------- conv_out -> uint8
// Tile: 16 rows x 64 columns of output pixels per 256-thread block; each thread owns 4 horizontally
// adjacent pixels, so one 6-wide input window per (row, channel) feeds all 3 taps x 4 pixels
// (6 LDS + 9 broadcast LDS.128 of weights per 108 FMAs).  Channels stream in chunks of 8 through
// a GN+SiLU-transformed fp32 halo tile; the padding taps are exact zeros (padding after SiLU).
constexpr int CO_TH = 16, CO_TW = 64, CO_CC = 8, CO_PW = 68;  // halo row pitch (>= 66, float4-aligned)

__global__ void __launch_bounds__(256) conv_out_u8_kernel(const __half* __restrict__ x, const float2* __restrict__ ss,
                                                          const float* __restrict__ w, const float* __restrict__ b,
                                                          uint8_t* __restrict__ rgb, int H, int W) {
  __shared__ __align__(16) float tile[CO_CC][CO_TH + 2][CO_PW];
  __shared__ float4 wsm[9][CO_CC];  // (co0, co1, co2, 0) per tap and channel
  const int img = blockIdx.z;
  const int y0 = blockIdx.y * CO_TH, x0 = blockIdx.x * CO_TW;
  const int ty = threadIdx.x >> 4, tx4 = (threadIdx.x & 15) * 4;
  float acc[4][3];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    acc[p][0] = b[0];
    acc[p][1] = b[1];
    acc[p][2] = b[2];
  }
  const float2* ssi = ss + (size_t)img * 128;
  for (int c0 = 0; c0 < 128; c0 += CO_CC) {
    __syncthreads();
    for (int pix = threadIdx.x; pix < (CO_TH + 2) * (CO_TW + 2); pix += 256) {
      const int py = pix / (CO_TW + 2), px = pix - py * (CO_TW + 2);
      const int gy = y0 + py - 1, gx = x0 + px - 1;
      float v[8];
      if (gy >= 0 && gy < H && gx >= 0 && gx < W) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(x + (((size_t)img * H + gy) * W + gx) * 128 + c0));
        const uint32_t wd[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&wd[j]));
          const float2 a = ssi[c0 + 2 * j], bb = ssi[c0 + 2 * j + 1];
          v[2 * j] = silu_f(fmaf(f.x, a.x, a.y));
          v[2 * j + 1] = silu_f(fmaf(f.y, bb.x, bb.y));
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) tile[j][py][px] = v[j];
    }
    if (threadIdx.x < 9 * CO_CC) {
      const int tap = threadIdx.x / CO_CC, ci = threadIdx.x % CO_CC;
      wsm[tap][ci] = make_float4(w[(0 * 9 + tap) * 128 + c0 + ci], w[(1 * 9 + tap) * 128 + c0 + ci],
                                 w[(2 * 9 + tap) * 128 + c0 + ci], 0.f);
    }
    __syncthreads();
#pragma unroll
    for (int ci = 0; ci < CO_CC; ++ci) {
#pragma unroll
      for (int ky = 0; ky < 3; ++ky) {
        const float* row = &tile[ci][ty + ky][tx4];
        const float4 i4 = *reinterpret_cast<const float4*>(row);
        const float2 i2 = *reinterpret_cast<const float2*>(row + 4);
        const float in[6] = {i4.x, i4.y, i4.z, i4.w, i2.x, i2.y};
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {
          const float4 wv = wsm[ky * 3 + kx][ci];
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            acc[p][0] = fmaf(in[p + kx], wv.x, acc[p][0]);
            acc[p][1] = fmaf(in[p + kx], wv.y, acc[p][1]);
            acc[p][2] = fmaf(in[p + kx], wv.z, acc[p][2]);
          }
        }
      }
    }
  }
  const int gy = y0 + ty, gx = x0 + tx4;
  if (gy < H && gx + 3 < W) {
    uint32_t q[3] = {0, 0, 0};
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        float t = __fadd_rn(__fmul_rn(acc[p][k], 0.5f), 0.5f);
        t = fminf(fmaxf(t, 0.f), 1.f);
        const uint32_t u8 = (uint32_t)__float2int_rn(__fmul_rn(t, 255.f));  // round-half-even
        const int byte = p * 3 + k;
        q[byte >> 2] |= u8 << (8 * (byte & 3));
      }
    uint32_t* o = reinterpret_cast<uint32_t*>(rgb + (((size_t)img * H + gy) * W + gx) * 3);  // 4-byte aligned
    o[0] = q[0];
    o[1] = q[1];
    o[2] = q[2];
  }
}

void launch_conv_out_u8(const __half* x, const float2* ss, const float* w, const float* b, uint8_t* rgb, int n,
                        int H, int W, cudaStream_t s) {
  dim3 grid((W + CO_TW - 1) / CO_TW, (H + CO_TH - 1) / CO_TH, n);
  conv_out_u8_kernel<<<grid, 256, 0, s>>>(x, ss, w, b, rgb, H, W);
}

}  // namespace lbx
