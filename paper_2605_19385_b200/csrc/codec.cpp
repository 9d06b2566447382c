// LBLP v1 packer and validator (format: include/lbx/lblp.h).  The packer is the write path of
// SURVEY.md 8(f) item 2; decode happens on the GPU (unpack.cu).  Mode-1 rows are encoded in two
// passes over a row buffer (deltas -> per-mini-block widths -> bit packing).
#include "codec.h"

#include <cmath>
#include <cstring>

#include "lbx/lblp.h"
#include "model.h"

namespace lbx {

namespace {
inline void wr16(uint8_t* p, uint16_t v) { std::memcpy(p, &v, 2); }
inline void wr32(uint8_t* p, uint32_t v) { std::memcpy(p, &v, 4); }
inline uint16_t rd16(const uint8_t* p) { uint16_t v; std::memcpy(&v, p, 2); return v; }
inline uint32_t rd32(const uint8_t* p) { uint32_t v; std::memcpy(&v, p, 4); return v; }

inline uint16_t order_map(uint16_t u) { return (u & 0x8000u) ? (uint16_t)~u : (uint16_t)(u | 0x8000u); }
inline uint16_t zz16(uint16_t d) { return (uint16_t)((uint16_t)(d << 1) ^ (uint16_t)((int16_t)d >> 15)); }
inline int width_of(uint32_t x) { return x ? 32 - __builtin_clz(x) : 0; }

void put_header(uint8_t* p, int mode, uint32_t c, uint32_t h, uint32_t w, uint32_t total, uint32_t table,
                uint32_t payload) {
  std::memset(p, 0, LBLP_HEADER_BYTES);
  std::memcpy(p, LBLP_MAGIC, 4);
  p[4] = LBLP_VERSION;
  p[5] = LBLP_DTYPE_F16;
  p[6] = (uint8_t)mode;
  wr16(p + 8, (uint16_t)c);
  wr16(p + 10, (uint16_t)h);
  wr16(p + 12, (uint16_t)w);
  wr32(p + 16, total);
  wr32(p + 20, table);
  wr32(p + 24, payload);
}
}  // namespace

bool lblp_pack(const uint16_t* x, int mode, uint32_t c, uint32_t h, uint32_t w, std::vector<uint8_t>* out,
               std::string* why) {
  if (!x || !out || c == 0 || h == 0 || w == 0 || c > 65535 || h > 65535 || w > 65535) {
    if (why) *why = "lblp_pack: bad shape or null pointer";
    return false;
  }
  const size_t n = (size_t)c * h * w, rows = (size_t)c * h;
  if (mode == LBLP_RAW) {
    out->assign(LBLP_HEADER_BYTES + 2 * n, 0);
    put_header(out->data(), mode, c, h, w, (uint32_t)out->size(), 0, LBLP_HEADER_BYTES);
    std::memcpy(out->data() + LBLP_HEADER_BYTES, x, 2 * n);
    return true;
  }
  if (mode == LBLP_Q8) {
    const size_t plane = (size_t)h * w;
    const uint32_t payload = LBLP_HEADER_BYTES + 8u * c;
    out->assign(payload + n, 0);
    uint8_t* o = out->data();
    put_header(o, mode, c, h, w, (uint32_t)out->size(), LBLP_HEADER_BYTES, payload);
    for (uint32_t ch = 0; ch < c; ++ch) {
      const uint16_t* src = x + ch * plane;
      float lo = INFINITY, hi = -INFINITY;
      for (size_t i = 0; i < plane; ++i) {
        const float f = f16_bits_to_f32(src[i]);
        if (std::isfinite(f)) { lo = f < lo ? f : lo; hi = f > hi ? f : hi; }
      }
      if (!(lo <= hi)) lo = hi = 0.f;
      float scale = (hi - lo) / 255.0f;
      if (!(scale > 0.f)) scale = 1.0f;
      const int32_t zp = -128 - (int32_t)std::lrintf(lo / scale);
      std::memcpy(o + LBLP_HEADER_BYTES + 4 * ch, &scale, 4);
      wr32(o + LBLP_HEADER_BYTES + 4 * c + 4 * ch, (uint32_t)zp);
      int8_t* q = reinterpret_cast<int8_t*>(o + payload + ch * plane);
      for (size_t i = 0; i < plane; ++i) {
        const float f = f16_bits_to_f32(src[i]);
        long v = std::isfinite(f) ? std::lrintf(f / scale) + zp : (f > 0 ? 127 : -128);
        q[i] = (int8_t)(v < -128 ? -128 : (v > 127 ? 127 : v));
      }
    }
    return true;
  }
  if (mode != LBLP_LOSSLESS || (w % 32)) {
    if (why) *why = mode == LBLP_LOSSLESS ? "lblp_pack: mode 1 needs W % 32 == 0" : "lblp_pack: unknown mode";
    return false;
  }
  const uint32_t nmb = w / 32;
  const uint32_t head = (2u + nmb + 3u) & ~3u;
  const uint32_t payload = LBLP_HEADER_BYTES + 4u * (uint32_t)rows;
  // pass 1: zigzag deltas and widths for every row
  std::vector<uint16_t> z(n);
  std::vector<uint8_t> widths(rows * nmb);
  std::vector<uint32_t> row_off(rows);
  uint32_t off = 0;
  for (size_t r = 0; r < rows; ++r) {
    const uint16_t* s = x + r * w;
    uint16_t* zr = z.data() + r * w;
    uint16_t prev = order_map(s[0]);
    zr[0] = 0;
    for (uint32_t i = 1; i < w; ++i) {
      const uint16_t v = order_map(s[i]);
      zr[i] = zz16((uint16_t)(v - prev));
      prev = v;
    }
    uint32_t words = 0;
    for (uint32_t j = 0; j < nmb; ++j) {
      uint32_t m = 0;
      for (uint32_t k = 0; k < 32; ++k) m |= zr[32 * j + k];  // OR has the same bit length as max
      const int bw = width_of(m);
      widths[r * nmb + j] = (uint8_t)bw;
      words += (uint32_t)bw;
    }
    row_off[r] = off;
    off += head + 4u * words;
  }
  out->assign((size_t)payload + off, 0);
  uint8_t* o = out->data();
  put_header(o, mode, c, h, w, (uint32_t)out->size(), LBLP_HEADER_BYTES, payload);
  // pass 2: row table and bit packing
  for (size_t r = 0; r < rows; ++r) {
    wr32(o + LBLP_HEADER_BYTES + 4 * r, row_off[r]);
    uint8_t* row = o + payload + row_off[r];
    wr16(row, x[r * w]);
    std::memcpy(row + 2, widths.data() + r * nmb, nmb);
    uint32_t* words = reinterpret_cast<uint32_t*>(row + head);  // rows are 4-byte aligned
    const uint16_t* zr = z.data() + r * w;
    for (uint32_t j = 0; j < nmb; ++j) {
      const uint32_t bw = widths[r * nmb + j];
      if (bw) {
        uint64_t acc = 0;
        uint32_t fill = 0, wi = 0;
        for (uint32_t k = 0; k < 32; ++k) {
          acc |= (uint64_t)zr[32 * j + k] << fill;
          fill += bw;
          if (fill >= 32) {
            words[wi++] = (uint32_t)acc;
            acc >>= 32;
            fill -= 32;
          }
        }
        // 32*bw bits is a whole number of words: nothing left over
      }
      words += bw;
    }
  }
  return true;
}

bool lblp_validate(const uint8_t* b, size_t nbytes, uint32_t c, uint32_t h, uint32_t w, std::string* why) {
  auto fail = [&](const char* m) {
    if (why) *why = m;
    return false;
  };
  if (!b || nbytes < LBLP_HEADER_BYTES) return fail("blob shorter than the 32-byte LBLP header");
  if (std::memcmp(b, LBLP_MAGIC, 4)) return fail("bad magic (expected LBLP)");
  if (b[4] != LBLP_VERSION) return fail("unsupported LBLP version");
  if (b[5] != LBLP_DTYPE_F16) return fail("unsupported LBLP dtype");
  if (rd16(b + 8) != c || rd16(b + 10) != h || rd16(b + 12) != w) return fail("blob shape != decoder latent shape");
  if (rd32(b + 16) != nbytes) return fail("total_bytes != blob size");
  const uint32_t table = rd32(b + 20), payload = rd32(b + 24);
  const size_t n = (size_t)c * h * w, rows = (size_t)c * h;
  switch (b[6]) {
    case LBLP_RAW:
      if (payload != LBLP_HEADER_BYTES || nbytes < payload + 2 * n) return fail("raw blob truncated");
      return true;
    case LBLP_Q8:
      if (table != LBLP_HEADER_BYTES || payload != LBLP_HEADER_BYTES + 8 * c || nbytes < payload + n)
        return fail("q8 blob truncated or bad offsets");
      return true;
    case LBLP_LOSSLESS: {
      if (w % 32) return fail("lossless blob needs W % 32 == 0");
      if (table != LBLP_HEADER_BYTES || payload != LBLP_HEADER_BYTES + 4 * rows || payload > nbytes)
        return fail("lossless blob bad table offsets");
      const uint32_t nmb = w / 32, head = (2u + nmb + 3u) & ~3u;
      for (size_t r = 0; r < rows; ++r) {
        const uint32_t off = rd32(b + LBLP_HEADER_BYTES + 4 * r);
        if (off & 3u) return fail("lossless row offset not 4-byte aligned");
        size_t end = (size_t)payload + off + head;
        if (end > nbytes) return fail("lossless row header out of bounds");
        for (uint32_t j = 0; j < nmb; ++j) {
          const uint32_t bw = b[payload + off + 2 + j];
          if (bw > 16) return fail("lossless mini-block width > 16");
          end += 4u * bw;
        }
        if (end > nbytes) return fail("lossless row payload out of bounds");
      }
      return true;
    }
    default:
      return fail("unknown LBLP mode");
  }
}

}  // namespace lbx
