// Host-visible description of one tcgen05 implicit-GEMM launch (conv3x3 / conv1x1 / plain GEMM).
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace lbx {

enum GemmMode : int {
  GEMM_PLAIN = 0,    // A = 2-D [M][K] (row stride lda), K-major
  GEMM_CONV3X3 = 1,  // A = NHWC activation, 3x3 taps, pad 1 (TMA OOB zero-fill supplies the halo)
  GEMM_SUBPIX = 2,   // nearest-2x upsample fused with 3x3 conv: 4 output phases, 2x2 taps each
};

// C[m, n] = alpha * row_scale[m] * sum_k A[m, k] B[n, k] + bias[n] + resid[m, n]     (fp32 math,
// one rounding to fp16), optional GroupNorm(32) partial sums of the stored fp16 values.
struct GemmArgs {
  int mode = GEMM_PLAIN;
  int M = 0, N = 0, K = 0;
  // A operand
  const __half* A = nullptr;
  int lda = 0;                    // plain: row stride (elements)
  int B_img = 0, H = 0, W = 0, C = 0;  // conv: NHWC input geometry (M = B_img*H*W, K = 9*C)
  // optional extra K segment from a second, plain operand whose rows match the output rows:
  // C += A2[m, :] . B[n, K : K + K2].  Used to fold a residual (B = identity) or a 1x1 shortcut
  // conv (B = W_sc) into the tensor-core accumulation instead of the epilogue.
  const __half* A2 = nullptr;
  int lda2 = 0, K2 = 0;
  // optional fused GroupNorm + SiLU on the A operand (conv3x3 halo mode): A' = SiLU(A * a_c + b_c),
  // (a_c, b_c) = gn_ss[image][channel]; out-of-image padding stays zero (applied after SiLU).
  const float2* gn_ss = nullptr;
  // B operand: weights [N][K + K2] K-major (conv: K index = (ky*3+kx)*C + ci); with b_mn_major
  // (plain GEMM) B is [K][N] with N contiguous (row stride ldb), e.g. V of the attention for P.V
  const __half* Bw = nullptr;
  int ldb = 0;
  int b_mn_major = 0;
  // batched plain GEMM over images: A / out rows of image i are [i*batch_m, (i+1)*batch_m) and
  // image i's B starts batch_b rows (K-major: N rows; MN-major: K rows) further; b_rows_total is
  // then the extent of B's row dimension (e.g. attention scores / P.V of a group of images)
  int batch_m = 0, batch_b = 0, b_rows_total = 0;
  // epilogue
  __half* out = nullptr;
  int ldo = 0;
  const float* bias = nullptr;
  const __half* resid = nullptr;
  int ldr = 0;
  const float* row_scale = nullptr;
  float alpha = 1.f;
  unsigned long long* gn_stats = nullptr;  // [img][32][2][2] fixed point (gnfix.cuh); zeroed by the caller
  int gn_cpg = 0;                 // channels per group = N / 32
  int rows_per_img = 0;           // M rows per image (GN image index = m / rows_per_img)
  // attention row reductions (plain GEMM with alpha, no bias / residual / GroupNorm), per output
  // row m and (n tile, epilogue column half) h -> row_part[m * 2 * n_tiles + h]:
  //   rowred 1: the maximum of the scaled values; nothing is stored
  //   rowred 2: E = exp(v - r_m) is stored (fp16), r_m = max(row_max[2m], row_max[2m + 1]) (a
  //             rowred-1 pass over a sample of the keys); row_part gets the fp32 sums of E.  A
  //             32-column chunk whose sum reaches 65504 (an E may overflow fp16) sets the flag of
  //             its image, exp_flag[m / batch_m], and the caller recomputes that image's softmax
  //             (exp_force: every image).
  int rowred = 0;
  const float* row_max = nullptr;
  float* row_part = nullptr;
  int* exp_flag = nullptr;
  int exp_force = 0;
  // per-image guard (the fallback of the fused softmax): run_if[i] for the launch's images
  // i < run_if_n (rows m / batch_m); tiles of images whose flag is 0 are skipped, and a launch with
  // no flag set exits at once
  const int* run_if = nullptr;
  int run_if_n = 1;
};

// Launch on `stream`.  Returns cudaSuccess or the launch error.  Chooses tile / CTA-pair config.
cudaError_t gemm_tc_launch(const GemmArgs& a, cudaStream_t stream, int force_cg = 0, int force_bn = 0);

// True when a conv3x3 launch of this geometry can fuse GroupNorm + SiLU into its A operand.
bool gemm_tc_can_fuse_gn(const GemmArgs& a);

// Diagnostics: halo_policy 0 forces per-tap A staging; desc_base_mode selects the UMMA descriptor
// base-offset convention for row-shifted (non-1024-aligned) halo views.
void gemm_tc_set_debug(int halo_policy, int desc_base_mode);
// Debug bit 7: fold identity residuals into the K loop at every width (default: only at 128 channels).
bool resid_fold_always();
// Debug bit 9: transpose V with a kernel for P.V (default: V read in place as an MN-major B).
bool v_transpose_legacy();
// Attention softmax fused into the score GEMM (exp in the epilogue against a sampled row maximum,
// exact-softmax fallback on overflow); debug bit 3 clears.  Bit 11 forces the fallback (tests).
bool attn_fused_exp();
bool attn_force_fallback();
// Debug bit 10 clears: conv residuals preloaded into the TMEM accumulator (default on).
bool resid_preload();
bool resid_rbuf();          // debug bit 24: extra K segments through their own buffer (rbuf); the
                            // 128-wide identity residual is then folded into K instead of preloaded
bool resid_epilogue_all();  // debug bit 29: identity residuals added in the epilogue at every width

// Resolve the TMA encoder and set kernel attributes up front (never during stream capture).
bool gemm_tc_prepare();
// programmatic dependent launch of the decode's kernels (debug bit 23); kernels that support it wait
// (griddepcontrol.wait) before their first global access and trigger their dependents when done
bool pdl_enabled();
void gemm_tc_set_max_sms(int n);  // diagnostics: GEMM grids use at most n SMs (0 = all)

// fp16 tiled TMA descriptor with 128-byte swizzle (dims innermost first; strides in bytes for
// dims 1..rank-1).  Out-of-bounds boxes are zero-filled.
bool make_tensor_map_f16(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                         const uint32_t* box);

// Number of SMs (cached) and the driver entry point used to encode TMA descriptors.
int num_sms();
bool tma_available();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: set it for the current device the
// first time a kernel is launched there (again if a larger size is needed).  Thread-safe.
bool ensure_smem_attr(const void* func, int bytes);

}  // namespace lbx
