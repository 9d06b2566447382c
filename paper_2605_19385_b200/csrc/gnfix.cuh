// GroupNorm statistics as exact fixed-point integers.
//
// Each (sum, sumsq) value of a GroupNorm site is accumulated by many CTAs.  With floating-point
// atomics the result depends on the order the partials arrive in, so an image decoded inside a
// batch could differ by an LSB from the same image decoded alone.  Here every partial (an fp32
// value) is rounded once to a multiple of 2^-30 and split into two integer words
//     v * 2^30 = hi * 2^32 + lo,   lo in [0, 2^32]
// which are added with 64-bit integer atomics.  Integer addition is associative, so the totals are
// the same for any arrival order, grid size or batch composition.  hi holds magnitudes up to
// 2^63 * 4 (far beyond any fp16 activation sum) and lo up to 2^31 partials.
//
// Layout of one site: unsigned long long [img][32 groups][2: sum, sumsq][2: hi, lo], zeroed by the
// caller before the producing kernel runs.
#pragma once
#include <cstdint>

namespace lbx {

constexpr int kGnStatWords = 4;  // per (image, group): sum hi, sum lo, sumsq hi, sumsq lo

__device__ __forceinline__ void gnfix_add(unsigned long long* p, float v) {
  const double d = (double)v * 1073741824.0;                 // v * 2^30, exact
  const double hf = floor(d * 2.3283064365386963e-10);       // floor(d / 2^32)
  const long long hi = (long long)hf;
  const long long lo = __double2ll_rn(d - hf * 4294967296.0);  // in [0, 2^32]
  atomicAdd(p, (unsigned long long)hi);
  atomicAdd(p + 1, (unsigned long long)lo);
}

// The accumulated (hi, lo) pair as a double: one rounding, so the same integers give the same value.
__host__ __device__ __forceinline__ double gnfix_value(const unsigned long long* p) {
  return (double)(long long)p[0] * 4.0 + (double)p[1] * 9.313225746154785e-10;  // hi*2^2 + lo*2^-30
}

}  // namespace lbx
