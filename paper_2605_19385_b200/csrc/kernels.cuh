// Launch wrappers for the HBM-bound kernels of the reconstruction path.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace lbx {

// fp16 NCHW latents -> prescale z/scaling + shift -> [post_quant 1x1, fp32] -> fp16 NHWC, channels
// zero-padded to 64 (conv_in then runs as an ordinary tcgen05 conv with C = 64).
void launch_latent_prep(const __half* lat, __half* out, int n, int cl, int h, int w, float scaling, float shift,
                        const float* pq_w, const float* pq_b, cudaStream_t s);

// GroupNorm-32 finalize: stats [n][32][2][2] (sum, sumsq of `count` values per group, gnfix.cuh
// fixed point) -> per-channel affine ss[n][C] = (gamma*rstd, beta - mean*gamma*rstd).
void launch_gn_finalize(const unsigned long long* stats, const float* gamma, const float* beta, float2* ss, int n, int C,
                        double count, float eps, cudaStream_t s);

// One GroupNorm site: fixed-point statistics [n][32][2][2] (gnfix.cuh) over 1/inv_count values per
// group, affine, eps.
struct GnSrc {
  const unsigned long long* stats;
  const float* gamma;
  const float* beta;
  double inv_count;
  float eps;
};

// y = act(GN(x)), x/y fp16 [n*hw][C] (y may alias x), act = SiLU if silu else identity; the kernel
// finalizes the statistics itself (same arithmetic as launch_gn_finalize).  h2: packed-half SiLU
// (act.cuh gn_act8_h2) instead of the fp32 one (gn_act8).
void launch_gn_apply(const __half* x, __half* y, const GnSrc& g, long long rows, int hw, int C, bool silu, bool h2,
                     cudaStream_t s);

// Row softmax numerator in place: P = exp(S - rowmax(S)) (fp16), row_scale = 1 / sum(P) (fp32).
// With run_if set the launch does nothing unless *run_if != 0 (the fused-exp path's fallback).
void launch_softmax_rows(__half* S, float* row_scale, int rows, int cols, cudaStream_t s, const int* run_if = nullptr);
// Fused-exp attention scores: row_scale[r] = 1 / sum(part[r][0 .. nparts)) in a fixed order, and
// (fallback) row_max2[2r] = max(part[r][..]), row_max2[2r + 1] = -inf.  With run_if set only the
// rows of flagged images (run_if[r / rows_per_img] != 0) are computed.
void launch_attn_rowsum(const float* part, int nparts, float* row_scale, int rows, cudaStream_t s,
                        const int* run_if = nullptr, int rows_per_img = 1);
void launch_attn_rowmax(const float* part, int nparts, float* row_max2, int rows, cudaStream_t s,
                        const int* run_if = nullptr, int rows_per_img = 1);
void launch_attn_count(const int* flags, int groups, unsigned long long* counter, cudaStream_t s);

// out[c][r] = in[r][c] for an R x Cc block with input row stride ldi and output row stride ldo.
void launch_transpose(const __half* in, int ldi, __half* out, int ldo, int R, int Cc, cudaStream_t s);

// Fused tail: GroupNorm(128) + SiLU -> conv3x3 128->3 (+bias) -> (x/2+0.5).clamp(0,1)*255 ->
// round-half-even -> uint8 HWC.  x fp16 NHWC [n][H][W][128]; w fp32 [3][3][3][128]; rgb [n][H][W][3].
void launch_conv_out_u8(const __half* x, const float2* ss, const float* w, const float* b, uint8_t* rgb, int n,
                        int H, int W, cudaStream_t s);

// Same tail on the tensor cores (csrc/conv_out_tc.cu): each input row loaded once by TMA, GN +
// SiLU applied in shared memory (packed-half SiLU when h2), 72 tcgen05.mma (M=128, N=16) per
// 128-pixel output row.  W must be a multiple of 128.
cudaError_t launch_conv_out_tc(const __half* x, const float2* ss, const float* w, const float* b, uint8_t* rgb,
                               int n, int H, int W, bool h2, cudaStream_t s);
void kernels_set_conv_out_legacy(bool on);
void kernels_set_apply_bulk(bool on);
void kernels_set_apply_max_sms(int n);
bool kernels_conv_out_legacy();

// GroupNorm-32 statistics (sum, sumsq per image and group) of x [n][hw][C] fp16 into stats
// [n][32][2][2] (gnfix.cuh fixed point, accumulated; zero it first).  Standalone form of what the
// conv epilogue fuses.
void launch_gn_stats(const __half* x, unsigned long long* stats, int n, int hw, int C, cudaStream_t s);

// LBLP v1 device unpack (include/lbx/lblp.h).  `blobs` is one device buffer holding n blobs at
// byte offsets `offs[i]` (device array); output fp16 NCHW [n][C][H][W].  Any malformed blob sets
// *err (device int) to a nonzero code; the output of that latent is then unspecified (zeros).
void kernels_set_unpack_rows(bool on);  // debug bit 24: the row-per-warp unpack kernel
void launch_lblp_unpack(const uint8_t* blobs, const unsigned long long* offs, const unsigned int* sizes, int n,
                        int C, int H, int W, __half* out, int* err, cudaStream_t s);

// Mid-block attention without the L x L scores (csrc/attn_fa.cu): out[n][L][512] =
// softmax(Q K^T / sqrt(512)) V with Q, K, V the column blocks of qkv [n][L][1536]; L % 128 == 0.
cudaError_t launch_attn_fa(const __half* qkv, __half* out, int n, int L, cudaStream_t s);

// LBLP mode-1 pack of n device latents (fp16 NCHW [n][C][H][W], W % 32 == 0) into out + i*stride
// (stride >= lblp_pack_bound, multiple of 4); sizes[i] = blob bytes.  Temporaries: widths_tmp
// [n*C*H*W/32] bytes, row_bytes_tmp [n*C*H] uint32.  Byte-identical to the host packer.
size_t lblp_pack_bound(int C, int H, int W);
cudaError_t launch_lblp_pack(const uint16_t* x, int n, int C, int H, int W, uint8_t* out, long long stride,
                             uint32_t* sizes, uint8_t* widths_tmp, uint32_t* row_bytes_tmp, cudaStream_t s);

// PNG encode (csrc/png.cu) of n uint8 RGB images [n][H][W][3] into out + i*stride (stride >=
// png_bound(H, W)) or, when `contiguous`, back to back from out (image i at the sum of the earlier
// sizes; out must hold n * png_bound); sizes[i] = PNG bytes.  `work` >= png_workspace(n, H, W)
// bytes of device scratch.
size_t png_bound(int H, int W);
size_t png_workspace(int n, int H, int W);
cudaError_t launch_png_encode(const uint8_t* rgb, int n, int H, int W, uint8_t* out, long long stride,
                              uint32_t* sizes, uint8_t* work, cudaStream_t s, bool contiguous = false);

}  // namespace lbx
