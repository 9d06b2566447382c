// Decoder parameter specs and the deterministic weight generator (product side).
// Architecture: AutoencoderKL decoder pinned by PAPER.md:386-391 (49,490,199 / 49,545,475 params,
// reproduced exactly by param_specs) and SURVEY.md Appendix A.  Generator contract: DESIGN.md 3.
#include "model.h"

#include <cmath>
#include <cstring>

namespace lbx {

bool family_info(int family, FamilyInfo* out) {
  switch (family) {
    case 0: *out = {4, 0.18215f, 0.0f, true}; return true;     // SD1.5
    case 1: *out = {16, 1.5305f, 0.0609f, false}; return true; // SD3 / SD3.5
    case 2: *out = {16, 0.3611f, 0.1159f, false}; return true; // FLUX.1
    default: return false;
  }
}

std::vector<ParamSpec> param_specs(int cl, bool post_quant) {
  std::vector<ParamSpec> v;
  auto conv = [&](const std::string& n, int cin, int cout, int k) {
    v.push_back({n + ".weight", {cout, cin, k, k}, 'w', cin * k * k});
    v.push_back({n + ".bias", {cout}, 'b', cin * k * k});
  };
  auto linear = [&](const std::string& n, int cin, int cout) {
    v.push_back({n + ".weight", {cout, cin}, 'w', cin});
    v.push_back({n + ".bias", {cout}, 'b', cin});
  };
  auto norm = [&](const std::string& n, int c) {
    v.push_back({n + ".weight", {c}, 'g', 0});
    v.push_back({n + ".bias", {c}, 'e', 0});
  };
  auto resnet = [&](const std::string& n, int cin, int cout) {
    norm(n + ".norm1", cin);
    conv(n + ".conv1", cin, cout, 3);
    norm(n + ".norm2", cout);
    conv(n + ".conv2", cout, cout, 3);
    if (cin != cout) conv(n + ".conv_shortcut", cin, cout, 1);
  };
  const int chans[4] = {512, 512, 256, 128};  // reversed block_out_channels
  if (post_quant) conv("post_quant_conv", cl, cl, 1);
  conv("decoder.conv_in", cl, 512, 3);
  resnet("decoder.mid_block.resnets.0", 512, 512);
  const std::string a = "decoder.mid_block.attentions.0";
  norm(a + ".group_norm", 512);
  linear(a + ".to_q", 512, 512);
  linear(a + ".to_k", 512, 512);
  linear(a + ".to_v", 512, 512);
  linear(a + ".to_out.0", 512, 512);
  resnet("decoder.mid_block.resnets.1", 512, 512);
  int prev = 512;
  for (int i = 0; i < 4; ++i) {
    for (int j = 0; j < 3; ++j)
      resnet("decoder.up_blocks." + std::to_string(i) + ".resnets." + std::to_string(j), j == 0 ? prev : chans[i],
             chans[i]);
    if (i < 3) conv("decoder.up_blocks." + std::to_string(i) + ".upsamplers.0.conv", chans[i], chans[i], 3);
    prev = chans[i];
  }
  norm("decoder.conv_norm_out", 128);
  conv("decoder.conv_out", 128, 3, 3);
  return v;
}

uint16_t f32_to_f16_bits(float f) {
  uint32_t b;
  std::memcpy(&b, &f, 4);
  const uint32_t sign = (b >> 16) & 0x8000u;
  const int32_t e = (int32_t)((b >> 23) & 0xFF);
  uint32_t m = b & 0x7FFFFFu;
  if (e == 0xFF) return (uint16_t)(sign | 0x7C00u | (m ? 0x200u : 0u));
  int32_t he = e - 127 + 15;
  if (he >= 31) return (uint16_t)(sign | 0x7C00u);
  if (he <= 0) {
    if (he < -10) return (uint16_t)sign;
    m |= 0x800000u;
    const int shift = 14 - he;
    uint32_t q = m >> shift;
    const uint32_t rem = m & ((1u << shift) - 1u), half = 1u << (shift - 1);
    if (rem > half || (rem == half && (q & 1u))) ++q;
    return (uint16_t)(sign | q);
  }
  uint32_t q = ((uint32_t)he << 10) | (m >> 13);
  const uint32_t rem = m & 0x1FFFu;
  if (rem > 0x1000u || (rem == 0x1000u && (q & 1u))) ++q;  // carry may roll into the exponent (correct)
  return (uint16_t)(sign | q);
}

float f16_bits_to_f32(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const uint32_t e = (h >> 10) & 31u, m = h & 1023u;
  uint32_t b;
  if (e == 0) {
    if (m == 0) b = sign;
    else {
      float f = std::ldexp((float)m, -24);
      std::memcpy(&b, &f, 4);
      b |= sign;
    }
  } else if (e == 31) {
    b = sign | 0x7F800000u | (m << 13);
  } else {
    b = sign | ((e - 15 + 127) << 23) | (m << 13);
  }
  float f;
  std::memcpy(&f, &b, 4);
  return f;
}

// splitmix64 finalizer -- the same mix64 the reference uses for its hash ring
// (proj/src/router.cpp:30-37).
static inline uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

std::vector<float> generate_params(int family, uint64_t seed) {
  FamilyInfo fi;
  if (!family_info(family, &fi)) return {};
  const auto specs = param_specs(fi.latent_channels, fi.post_quant);
  size_t total = 0;
  for (const auto& s : specs) total += s.count();
  std::vector<float> out(total);
  size_t pos = 0;
  for (size_t tid = 0; tid < specs.size(); ++tid) {
    const auto& s = specs[tid];
    const uint64_t base = ((seed + 1) * 0x9E3779B97F4A7C15ull) ^ ((uint64_t)(tid + 1) * 0xC2B2AE3D27D4EB4Full);
    const double root = s.fan_in ? std::sqrt((double)s.fan_in) : 1.0;  // divide (not multiply by 1/root)
    const size_t n = s.count();
    for (size_t i = 0; i < n; ++i) {
      const uint64_t z = mix64(base + (uint64_t)(i + 1) * 0xD1B54A32D192ED03ull);
      const double u = (double)(z >> 11) * (1.0 / 9007199254740992.0);
      const double sym = 2.0 * u - 1.0;
      float v;
      switch (s.kind) {
        case 'w': v = f16_bits_to_f32(f32_to_f16_bits((float)(sym / root))); break;
        case 'b': v = (float)(sym / root); break;
        case 'g': v = (float)(1.0 + 0.25 * sym); break;
        default: v = (float)(0.25 * sym); break;
      }
      out[pos + i] = v;
    }
    pos += n;
  }
  return out;
}

}  // namespace lbx
