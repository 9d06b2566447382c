// Host-side model description: parameter specs, deterministic generator, device weight layout.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace lbx {

struct FamilyInfo {
  int latent_channels;
  float scaling, shift;
  bool post_quant;
};
bool family_info(int family, FamilyInfo* out);

struct ParamSpec {
  std::string name;
  std::vector<int> shape;
  char kind;  // 'w' weight, 'b' bias, 'g' gamma, 'e' beta
  int fan_in;
  size_t count() const {
    size_t n = 1;
    for (int d : shape) n *= (size_t)d;
    return n;
  }
};

// Canonical order (diffusers AutoencoderKL decoder naming); identical to oracle/weights_ref.py.
std::vector<ParamSpec> param_specs(int latent_channels, bool post_quant);

// Generate all parameters (fp32, canonical order, concatenated).  Weights hold fp16-representable
// values (generated fp32, rounded to fp16), see DESIGN.md section 3.
std::vector<float> generate_params(int family, uint64_t seed);

// Host IEEE fp16 conversion helpers (round-to-nearest-even).
uint16_t f32_to_f16_bits(float f);
float f16_bits_to_f32(uint16_t h);

}  // namespace lbx
