// Device-side activation / GroupNorm helpers shared by the standalone HBM kernels (kernels.cu) and the
// deferred GroupNorm apply inside the tcgen05 conv (gemm_tc.cu), so both paths round identically.
#pragma once
#include <cuda_fp16.h>
#include <cstdint>

namespace lbx {

// Packed fp32 pairs (sm_100 FFMA2 / FADD2 / FMUL2): two IEEE fp32 operations per instruction, each
// rounded once, so bit-identical to the scalar forms with half the issue slots.
__device__ __forceinline__ uint64_t f2_pack(float2 a) {
  uint64_t u;
  asm("mov.b64 %0, {%1, %2};" : "=l"(u) : "f"(a.x), "f"(a.y));
  return u;
}
__device__ __forceinline__ float2 f2_unpack(uint64_t u) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(u));
  return r;
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2_pack(a)), "l"(f2_pack(b)), "l"(f2_pack(c)));
  return f2_unpack(d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_pack(a)), "l"(f2_pack(b)));
  return f2_unpack(d);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_pack(a)), "l"(f2_pack(b)));
  return f2_unpack(d);
}

// SiLU with one MUFU op per element: ex2 on the SFU, the reciprocal of (1 + e) on the FMA pipe
// (bit-trick seed, 3 Newton steps -> fp32-accurate).  The SFU (16 ops/clk/SM) is what bounded the
// GroupNorm-apply pass at ~3.5 TB/s with ex2 + rcp; the FMA pipe has 8x its throughput.
__device__ __forceinline__ float silu_f(float x) {
  const float xc = fmaxf(x, -80.0f);  // keeps 1 + e finite and normal for the seed trick
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(xc * -1.4426950408889634f));
  const float d = 1.0f + e;
  float r = __int_as_float(0x7EF311C3 - __float_as_int(d));
  r = r * fmaf(-d, r, 2.0f);
  r = r * fmaf(-d, r, 2.0f);
  r = r * fmaf(-d, r, 2.0f);
  return x * r;
}

// GroupNorm affine of one channel from fp64 (sum, sumsq) over 1/inv_count values -- the single
// definition of the finalize arithmetic: y = x * a + b with a = gamma * rstd, b = beta - mean * a.
// Mean and variance stay fp64 (the E[x^2] - mean^2 cancellation), but only multiplies: the fp64
// divide / sqrt sequences cost too much when every apply thread finalizes its own channels;
// rstd is an IEEE fp32 sqrt + divide of the fp32-rounded variance.
__device__ __forceinline__ float2 gn_affine(double s, double s2, double inv_count, float gamma, float beta,
                                            float eps) {
  const double inv = inv_count;  // 1 / values per group, computed once on the host
  const double mean = s * inv;
  double var = fma(s2, inv, -mean * mean);
  if (var < 0) var = 0;
  const float rstd = 1.0f / sqrtf((float)var + eps);
  const float a = gamma * rstd;
  return make_float2(a, (float)fma(-mean, (double)a, (double)beta));
}

// 8 packed fp16 -> act(x * a + b) -> 8 packed fp16 (fp32 math, one rounding).
template <bool SILU>
__device__ __forceinline__ uint4 gn_act8(uint4 u, const float (&a)[8], const float (&b)[8]) {
  uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 y = ffma2(__half22float2(*reinterpret_cast<const __half2*>(&w[j])), make_float2(a[2 * j], a[2 * j + 1]),
                           make_float2(b[2 * j], b[2 * j + 1]));
    float y0 = y.x, y1 = y.y;
    if (SILU) { y0 = silu_f(y0); y1 = silu_f(y1); }
    const __half2 h = __floats2half2_rn(y0, y1);
    w[j] = *reinterpret_cast<const uint32_t*>(&h);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// Packed-half variant: affine in fp32, one rounding to fp16, then SiLU(y) = h + h*tanh(h), h = y/2,
// on half2 (HMUL2, one MUFU.TANH per two elements, HFMA2): ~4 instructions per element instead of
// ~13.  tanh.approx.f16x2 has ~2^-11 absolute error, so the result carries up to ~|y|*2^-11 more
// error than the fp32 path (about one extra fp16 ulp); opt-in, judged end to end (tests/).
__device__ __forceinline__ uint32_t tanh_f16x2(uint32_t x) {
  uint32_t r;
  asm("tanh.approx.f16x2 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}
template <bool SILU>
__device__ __forceinline__ uint4 gn_act8_h2(uint4 u, const float (&a)[8], const float (&b)[8]) {
  uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    __half2 y = __float22half2_rn(ffma2(__half22float2(*reinterpret_cast<const __half2*>(&w[j])),
                                        make_float2(a[2 * j], a[2 * j + 1]), make_float2(b[2 * j], b[2 * j + 1])));
    if (SILU) {
      const __half2 h = __hmul2(y, __float2half2_rn(0.5f));
      const uint32_t hb = *reinterpret_cast<const uint32_t*>(&h);
      const uint32_t tb = tanh_f16x2(hb);
      y = __hfma2(h, *reinterpret_cast<const __half2*>(&tb), h);
    }
    w[j] = *reinterpret_cast<const uint32_t*>(&y);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// The same packed-half SiLU with the 1/2 folded into the affine: ah = a/2, bh = b/2 (exact in fp32),
// so h = fp16(x*ah + bh) = fp16(x*a + b)/2 without the HMUL2 (3 instead of 4 instructions per two
// elements; identical to gn_act8_h2<true> except where y/2 is an fp16 subnormal).  Hot transforms
// (GroupNorm applies, the fused A operand, the tail) halve their coefficients once when loading them.
__device__ __forceinline__ uint4 gn_silu8_h2_half(uint4 u, const float (&ah)[8], const float (&bh)[8]) {
  uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const __half2 h = __float22half2_rn(ffma2(__half22float2(*reinterpret_cast<const __half2*>(&w[j])),
                                              make_float2(ah[2 * j], ah[2 * j + 1]), make_float2(bh[2 * j], bh[2 * j + 1])));
    const uint32_t hb = *reinterpret_cast<const uint32_t*>(&h);
    const uint32_t tb = tanh_f16x2(hb);
    const __half2 y = __hfma2(h, *reinterpret_cast<const __half2*>(&tb), h);
    w[j] = *reinterpret_cast<const uint32_t*>(&y);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

}  // namespace lbx
