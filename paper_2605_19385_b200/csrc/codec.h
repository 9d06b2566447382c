// Product-side LBLP v1 host code: the packer (write path) and blob validation before H2D.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace lbx {

// Encode one fp16 NCHW latent.  Returns false (and sets *why) on bad arguments.
bool lblp_pack(const uint16_t* latent, int mode, uint32_t c, uint32_t h, uint32_t w, std::vector<uint8_t>* out,
               std::string* why);

// Validate a blob's header, tables and row extents against (c, h, w).  Cheap (O(rows)).
bool lblp_validate(const uint8_t* blob, size_t nbytes, uint32_t c, uint32_t h, uint32_t w, std::string* why);

}  // namespace lbx
