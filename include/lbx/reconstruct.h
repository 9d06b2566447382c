/*
 * lbx/reconstruct.h -- C ABI of the B200-native decode-on-miss reconstruction path.
 *
 * What this replaces.  In the reference, a cache miss that needs pixels becomes a GPU job whose
 * service time is the constant LatencyModel::decode_ms = 40 (proj/include/latentbox/sim.hpp:19):
 *   Engine::on_job_ready  (proj/src/sim.cpp:409-429)  least-loaded GPU, start = max(t, free_at),
 *                                                      free_at = start + decode_ms   (:414)
 *   Engine::on_job_done   (proj/src/sim.cpp:431-442)  depth--, observe_latency(Decode, queue+decode)
 *   observe_latency       (proj/include/latentbox/tuner.hpp:57-58, proj/src/tuner.cpp:48-59)
 * called for LatentHit / FullMiss from Engine::on_arrival (proj/src/sim.cpp:364-405) and for the
 * off-path promotion decode (:376-377).  There is no callable decode function in the reference
 * (SPEC.md:8 scopes real decoding out); this header is the callable boundary those call sites get:
 * lbx_reconstruct() is the "decode" of on_job_ready, its measured duration is the sample that
 * on_job_done feeds to observe_latency, and lbx_batcher_* replaces least_loaded_gpu (sim.cpp:238-243)
 * with real per-GPU queues.  INTEGRATION.md shows the call-site binding.
 *
 * Conventions mirrored from the reference:
 *   - status codes instead of exceptions; LBX_E_CONFIG plays the role of ConfigError naming the bad
 *     field (proj/include/latentbox/error.hpp:8-11), LBX_E_RUNTIME of std::runtime_error; the
 *     message is available from lbx_last_error() (thread-local).
 *   - single-owner state: one lbx_decoder per GPU, calls on it serialised by its owner thread
 *     (proj/include/latentbox/dual_cache.hpp:46; the paper serialises each device behind
 *     a lock).  Different decoders run concurrently from different threads.
 *   - the caller owns inputs and outputs; the decoder owns weights, activation arena and CUDA graphs.
 * No exceptions cross this boundary; no torch types appear in it.
 */
#ifndef LBX_RECONSTRUCT_H
#define LBX_RECONSTRUCT_H

#include <stddef.h>
#include <stdint.h>

#include "lbx/lblp.h"

/* The library is built with hidden visibility: exactly the functions declared LBX_API are exported
 * (its C++ internals never clash with a host program's symbols). */
#ifndef LBX_API
#if defined(__GNUC__)
#define LBX_API __attribute__((visibility("default")))
#else
#define LBX_API
#endif
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LBX_OK = 0,
  LBX_E_RUNTIME = 1, /* runtime failure (std::runtime_error in the reference) */
  LBX_E_CONFIG = 2,  /* invalid descriptor / argument (ConfigError, error.hpp:8-11) */
  LBX_E_CUDA = 3,    /* CUDA error or no sm_100 device */
  LBX_E_FORMAT = 4   /* malformed LBLP blob */
} lbx_status;

typedef enum { LBX_FAMILY_SD15 = 0, LBX_FAMILY_SD3 = 1, LBX_FAMILY_FLUX = 2 } lbx_family;

/* Decoder descriptor.  Latent shapes: 4x64x64 (-> 512^2), 4x128x128 / 16x128x128 (-> 1024^2). */
typedef struct {
  int family;                 /* lbx_family: sets latent channels, scaling/shift, post_quant_conv */
  uint32_t latent_h, latent_w; /* latent spatial size, output 8x larger: latent_w 64 or a multiple of
                                  128, latent_h even, both in [8, 512] (LBX_E_CONFIG otherwise) */
  uint64_t weight_seed;       /* used when weights == NULL (deterministic generator) */
  const float* weights;       /* optional: all parameters, fp32, canonical order (lbx_param_count) */
  size_t weights_count;       /* number of floats in `weights` */
  int device;                 /* CUDA device ordinal */
  uint32_t max_batch;         /* largest n passed to decode/reconstruct (arena is sized for it) */
  int precise_activations;    /* 0 (default): SiLU of every GroupNorm apply on packed halves (one
                                 MUFU.TANH per two elements, fp16-engine numerics);
                                 1: fp32 SiLU (~0.7 dB higher PSNR vs the fp32 oracle, ~2% slower) */
} lbx_decoder_desc;

typedef struct lbx_decoder lbx_decoder;
typedef void* lbx_stream; /* cudaStream_t; NULL = the decoder's own stream */

/* Number of fp32 parameters of a family's decoder (49,490,199 for SD1.5, 49,545,475 for SD3/FLUX). */
LBX_API size_t lbx_param_count(int family);

/* The deterministic parameters a seed selects (fp32, canonical order; `out` holds count floats). */
LBX_API lbx_status lbx_generate_params(int family, uint64_t seed, float* out, size_t count);

LBX_API lbx_status lbx_decoder_create(const lbx_decoder_desc* desc, lbx_decoder** out);
LBX_API lbx_status lbx_decoder_destroy(lbx_decoder* dec);
/* Capture (without running) the CUDA graphs for every batch size 1..n_max, so the first request of
 * each size does not pay graph capture (~tens of ms).  Graphs run on the decoder's own latent / RGB
 * buffers; every entry point (including lbx_decode on caller device buffers) reuses them. */
LBX_API lbx_status lbx_decoder_prepare(lbx_decoder* dec, uint32_t n_max);

/* Packed LBLP blobs (HOST memory) -> fp16 NCHW latents on the device, bit-exact.  Blob shapes must
 * equal the decoder's (C, latent_h, latent_w).  Asynchronous on `stream`; a malformed blob is
 * reported as LBX_E_FORMAT (host-side header validation) or at the next synchronising call. */
LBX_API lbx_status lbx_unpack(lbx_decoder* dec, const uint8_t* const* blobs, const size_t* nbytes, uint32_t n,
                      void* latents_dev, lbx_stream stream);

/* fp16 NCHW latents (device) -> uint8 RGB NHWC (device), n x 8h x 8w x 3.  Asynchronous. */
LBX_API lbx_status lbx_decode(lbx_decoder* dec, const void* latents_dev, uint32_t n, uint8_t* rgb_dev,
                      lbx_stream stream);

/* The call the cache tiers make on a miss: host blobs -> H2D -> unpack -> decode (CUDA graph) ->
 * D2H into rgb_host (n x 8h x 8w x 3).  Synchronous: returns when rgb_host is filled. */
LBX_API lbx_status lbx_reconstruct(lbx_decoder* dec, const uint8_t* const* blobs, const size_t* nbytes, uint32_t n,
                           uint8_t* rgb_host, lbx_stream stream);

/* Vectored form: image i lands in rgb_hosts[i] (8h x 8w x 3 bytes each).  Synchronous. */
LBX_API lbx_status lbx_reconstruct_v(lbx_decoder* dec, const uint8_t* const* blobs, const size_t* nbytes, uint32_t n,
                             uint8_t* const* rgb_hosts, lbx_stream stream);

/* Asynchronous, pipelined form of lbx_reconstruct_v (what lbx_batcher's workers use).  Stages the
 * batch and enqueues H2D + unpack, the decode graph and the D2H on three streams of the decoder,
 * then returns a ticket without waiting.  Up to two batches may be in flight: batch k+1's host
 * staging, H2D and unpack and batch k-1's D2H overlap batch k's decode (PAPER.md:667-670 runs
 * decompression and encoding in pools around GPU inference).  A third submit before the oldest
 * ticket is waited for returns LBX_E_RUNTIME.  Blob headers are validated before anything is
 * enqueued (LBX_E_FORMAT, no ticket).  rgb_hosts[i] must stay valid until the wait returns. */
LBX_API lbx_status lbx_reconstruct_submit(lbx_decoder* dec, const uint8_t* const* blobs, const size_t* nbytes, uint32_t n,
                                  uint8_t* const* rgb_hosts, uint64_t* ticket);
/* Block until the batch of `ticket` is in rgb_hosts; its status (LBX_E_FORMAT if the device unpack
 * found a malformed blob).  Each ticket is waited for exactly once. */
LBX_API lbx_status lbx_reconstruct_wait(lbx_decoder* dec, uint64_t ticket);

/* CUDA graphs this decoder has captured (one per batch size; caller buffers never cause one). */
LBX_API uint64_t lbx_graph_captures(lbx_decoder* dec);

/* Same pipeline for blobs resident in GPU memory (an HBM latent tier): blob i is nbytes[i] bytes at
 * device pointer blobs_dev[i] on CUDA device blob_devices[i] (-1: host memory, handled as in
 * lbx_reconstruct_submit, so one batch may mix both).  A blob on this decoder's device is
 * copied D2D; a blob on another GPU is fetched with a peer copy over NVLink -- the latent shipping
 * of a spilled decode, which the reference models as LatencyModel::intra_cluster_ms = 5
 * (proj/include/latentbox/sim.hpp:20, proj/src/sim.cpp:369-373, proj/src/router.cpp:99-114).  Blob
 * headers are validated by the device unpack (LBX_E_FORMAT at the wait). */
LBX_API lbx_status lbx_reconstruct_submit_dev(lbx_decoder* dec, const uint8_t* const* blobs_dev, const int* blob_devices,
                                      const size_t* nbytes, uint32_t n, uint8_t* const* rgb_hosts, uint64_t* ticket);

typedef struct {
  uint64_t graph_captures; /* CUDA graphs captured (one per batch size) */
  uint64_t peer_copies;    /* blobs fetched from another GPU (lbx_reconstruct_submit_dev) */
  uint64_t peer_bytes;     /* their bytes */
  double peer_ms;          /* device time of the batches' peer-copy phases, summed (CUDA events) */
  uint64_t attn_fallbacks; /* images whose sampled-maximum attention softmax could overflow fp16 and
                              was recomputed against the exact row maximum (normally 0) */
} lbx_decoder_counters;
LBX_API lbx_status lbx_decoder_get_counters(lbx_decoder* dec, lbx_decoder_counters* out);

/* Same path from fp16 NCHW latents in HOST memory (no codec): H2D -> decode -> D2H.  Synchronous. */
LBX_API lbx_status lbx_reconstruct_latents(lbx_decoder* dec, const void* latents_host, uint32_t n, uint8_t* rgb_host,
                                   lbx_stream stream);

/* Host-side LBLP packer (the write path).  `latent` is one fp16 NCHW latent (c*h*w values).
 * Returns the blob size; writes it when out != NULL and cap is large enough. */
LBX_API lbx_status lbx_pack(const uint16_t* latent, int mode, uint32_t c, uint32_t h, uint32_t w, uint8_t* out,
                    size_t cap, size_t* out_bytes);

/* Device-side write path: LBLP mode-1 (lossless) pack of n fp16 NCHW latents already on the GPU
 * (latents_dev, c x h x w each, w % 32 == 0).  Blob i is written at out_dev + i * stride (stride >=
 * lbx_pack_bound(c, h, w), multiple of 4) and its size to sizes_dev[i] (uint32, device).  The bytes
 * equal lbx_pack(..., mode 1, ...).  Asynchronous on `stream` (NULL = default stream). */
LBX_API size_t lbx_pack_bound(uint32_t c, uint32_t h, uint32_t w);
LBX_API lbx_status lbx_pack_device(const void* latents_dev, uint32_t n, uint32_t c, uint32_t h, uint32_t w, uint8_t* out_dev,
                           size_t stride, uint32_t* sizes_dev, lbx_stream stream);

/* Return path (the paper PNG-encodes on CPU): PNG encode of n
 * uint8 RGB images already on the GPU (rgb_dev, [n][h][w][3], e.g. lbx_decode's output).  PNG i is
 * written at out_dev + i * stride (stride >= lbx_png_bound(h, w)) and its size to sizes_dev[i]
 * (uint32, device).  8-bit RGB, per-row adaptive filter, zlib/DEFLATE with dynamic Huffman codes
 * (stored where smaller); lossless: any PNG decoder returns rgb exactly.  w <= 8192, h <= 65535.
 * Asynchronous on `stream`. */
LBX_API size_t lbx_png_bound(uint32_t h, uint32_t w);
/* lbx_reconstruct with the return path on the GPU: host blobs -> unpack -> decode -> PNG encode ->
 * only the PNG bytes cross PCIe.  PNG i is written at png_host + (png_sizes[0] + ... + png_sizes[i-1])
 * and its length to png_sizes[i].  cap = bytes available at png_host; n * lbx_png_bound(8*latent_h,
 * 8*latent_w) always suffices; if the PNGs need more, LBX_E_CONFIG (sizes still returned). */
LBX_API lbx_status lbx_reconstruct_png(lbx_decoder* dec, const uint8_t* const* blobs, const size_t* nbytes, uint32_t n,
                               uint8_t* png_host, size_t cap, size_t* png_sizes, lbx_stream stream);
LBX_API lbx_status lbx_png_encode_device(const uint8_t* rgb_dev, uint32_t n, uint32_t h, uint32_t w, uint8_t* out_dev,
                                 size_t stride, uint32_t* sizes_dev, lbx_stream stream);

/* Unpack of LBLP blobs already in device memory (e.g. an HBM-resident latent tier): blob i at
 * blobs_dev + offs_dev[i] (8-byte aligned), sizes_dev[i] bytes; out_dev = n fp16 NCHW latents of
 * c x h x w.  A malformed blob sets *err_dev (device int, zero it first) to a nonzero code and leaves
 * that latent unspecified.  Bit-exact with lbx_unpack.  Asynchronous on `stream`. */
LBX_API lbx_status lbx_op_unpack(const uint8_t* blobs_dev, const unsigned long long* offs_dev, const uint32_t* sizes_dev,
                         uint32_t n, uint32_t c, uint32_t h, uint32_t w, void* out_dev, int* err_dev,
                         lbx_stream stream);

/* Page-locked host memory for blobs and outputs (cudaMallocHost): copies to and from it run at full
 * PCIe rate, where pageable memory goes through a staging copy.  NULL on failure. */
LBX_API void* lbx_host_alloc(size_t bytes);
LBX_API void lbx_host_free(void* p);

/* Thread-local description of the last error on this thread ("" if none). */
LBX_API const char* lbx_last_error(void);

/* ------------------------------------------------------------------ profiling
 * Run one decode of n latents (internal buffers) eagerly with a CUDA event after every launch and
 * report per-launch device time.  flops = executed tensor FLOPs, algo_flops = the standard
 * algorithmic FLOPs the launch stands for (a sub-pixel launch stands for nearest-2x + conv3x3),
 * bytes = algorithmic HBM bytes.  Fills up to cap entries, *count = entries written. */
typedef struct {
  char name[96];
  double ms;
  double flops;
  double algo_flops;
  double bytes;
} lbx_prof_entry;
LBX_API lbx_status lbx_profile(lbx_decoder* dec, uint32_t n, lbx_prof_entry* out, int cap, int* count);

/* Kernel launches in one decode of batch n (after the first lbx_decode/reconstruct of that n), or -1. */
LBX_API int lbx_launch_count(lbx_decoder* dec, uint32_t n);

/* ------------------------------------------------------------------ diagnostics / op-level entry
 * Individual kernels of the path, for op-level parity tests and benchmarks.  Device pointers,
 * fp16 = uint16 storage.  All asynchronous on `stream`. */

/* tcgen05 GEMM / conv: out[m, n] = alpha*rs[m]*sum_k A[m,k]*B[n,k] + bias[n] + resid[m,n].
 * mode 0 plain (A [M][K], row stride lda); mode 1 conv3x3 pad 1 (A NHWC [b][h][w][c], K = 9c);
 * mode 2 nearest-2x upsample + conv3x3 as 4 sub-pixel 2x2 convs (B = [4][N][4c], out 2h x 2w).
 * gn_stats (optional, uint64 [b][32][2][2], accumulated) gets GroupNorm-32 partial sums of out as
 * exact fixed-point pairs: value = (int64)hi * 4 + lo * 2^-30 (order-independent, see gnfix.cuh).
 * cta_group/bn: 0 = auto, else force 1|2 and 128|256. */
LBX_API lbx_status lbx_op_gemm(int mode, int M, int N, int K, const void* A, int lda, int b, int h, int w, int c,
                       const void* Bw, int ldb, void* out, int ldo, const float* bias, const void* resid, int ldr,
                       const float* row_scale, float alpha, uint64_t* gn_stats, int cta_group, int bn,
                       lbx_stream stream);
/* Same op with an optional extra K segment from a second plain operand A2 [M][K2] (row stride lda2):
 * out += A2 . B[:, K:K+K2]^T inside the tensor-core accumulation (B then has K + K2 columns).  The
 * decoder folds each resnet's residual (B = identity) or 1x1 shortcut (B = W_sc) into conv2 this way. */
typedef struct {
  int mode, M, N, K;
  const void* A;
  int lda, b, h, w, c;
  const void* A2;
  int lda2, K2;
  const void* B;
  int ldb;
  void* out;
  int ldo;
  const float* bias;
  const void* resid;
  int ldr;
  const float* row_scale;
  float alpha;
  uint64_t* gn_stats;
  int cta_group, bn;
  const float* gn_ss; /* optional: fused A' = SiLU(A * ss[img][c].x + ss[img][c].y) (conv3x3), float pairs */
  int b_mn_major;     /* plain GEMM: B is [K][N] with N contiguous (row stride ldb) instead of [N][K] */
} lbx_gemm_desc;
LBX_API lbx_status lbx_op_gemm_desc(const lbx_gemm_desc* d, lbx_stream stream);
/* Diagnostics.  halo_policy bits: 0 = halo staging when possible (else per-tap A staging); 1 disables
 * the two-sub-tile variant; 2 enables the fused GroupNorm A-operand transform (XF) in the decoder;
 * 4 selects the CUDA-core conv_out tail; 5 gives halo convs two A stages and the rest of smem to B;
 * 6 uses horizontally (instead of vertically) adjacent sub-tiles for the two-sub-tile variant; 7 folds
 * identity residuals into the K loop at every width (default: epilogue add at >= 256 channels); 8
 * selects the register-staged GroupNorm apply instead of the bulk-copy (1-D TMA) one; 9 transposes the
 * attention's V with a kernel instead of reading it in place as an MN-major B operand; 10 adds conv
 * residuals in the epilogue instead of preloading them into the TMEM accumulator (default: preload for
 * 128-wide outputs, epilogue add for wider ones; bit 20 preloads at every width; bit 21 L2-prefetches
 * the next preload's rows; bit 22 gives each conv cluster a contiguous block of tiles instead of
 * round-robin; bit 23 launches the GEMM and GroupNorm-apply kernels as programmatic dependents; bit 25 routes
 * the residual preload through per-warp shared-memory staging with line-covering loads);
 * 12-15 are
 * epilogue ablations (wrong results: skip all work / keep only TMEM loads / no stores / no
 * statistics); bits 16-17 = 1 + epilogue store mode (0 STG.128, 1 STG.256 = default, 2 streaming); 18
 * stages every eligible GEMM's epilogue chunks in smem and TMA-stores them (default: plain GEMMs
 * only, i.e. the attention projections and scores), 26 disables the TMA-store epilogue.
 * desc_base_mode selects the UMMA descriptor base-offset convention for row-shifted halo views. */
LBX_API lbx_status lbx_op_set_debug(int halo_policy, int desc_base_mode);
/* Diagnostics: GEMM grids use at most gemm_sms SMs and bulk GroupNorm applies at most apply_sms
 * (0 = all), so that two kernels can share the GPU on different streams. */
LBX_API lbx_status lbx_op_set_grid_limits(int gemm_sms, int apply_sms);
/* Decoder tail: rgb = u8(conv3x3_{128->3}(SiLU(x * ss.x + ss.y)) + b) with x fp16 NHWC [n][H][W][128],
 * ss float pairs [n][128], w fp32 [3][3][3][128] ([out][ky][kx][in]), rgb [n][H][W][3].  impl 0 =
 * tensor cores (fp32 SiLU), 2 = tensor cores with packed-half SiLU, 1 = CUDA cores (fp32). */
LBX_API lbx_status lbx_op_conv_out(const void* x, const float* ss, const float* w, const float* b, uint8_t* rgb, int n,
                           int H, int W, int impl, lbx_stream stream);
/* Mid-block attention core without the L x L scores (csrc/attn_fa.cu): out [n][L][512] =
 * softmax(Q K^T / sqrt(512)) V, Q/K/V = column blocks 0/512/1024 of qkv [n][L][1536] fp16; L % 128 == 0. */
LBX_API lbx_status lbx_op_attention(const void* qkv, void* out, int n, int L, lbx_stream stream);
/* Fold a 3x3 conv weight [N][3][3][C] (fp32, host) into the 4 sub-pixel 2x2 kernels, fp16 [4][N][2][2][C]. */
LBX_API lbx_status lbx_subpixel_weights(const float* w3x3, int N, int C, uint16_t* out);
/* GroupNorm finalize + apply; silu 0 = identity, 1 = fp32 SiLU, 2 = packed-half SiLU; y may alias x. */
LBX_API lbx_status lbx_op_groupnorm(const void* x, void* y, const uint64_t* stats, const float* gamma, const float* beta,
                            int b, int hw, int c, int silu, float eps, lbx_stream stream);
/* GroupNorm-32 statistics of x ([b][hw][c] fp16) into stats (uint64 [b][32][2][2] fixed point, zeroed
 * here). */
LBX_API lbx_status lbx_op_gn_stats(const void* x, uint64_t* stats, int b, int hw, int c, lbx_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* LBX_RECONSTRUCT_H */
