// LBLP v1 packer and validator (format: include/lbx/lblp.h).  The packer is the write path of
// SURVEY.md 8(f) item 2; decode happens on the GPU (unpack.cu).  Mode-1 rows are encoded in two
// passes over a row buffer (deltas -> per-mini-block widths -> bit packing).
#include "codec.h"

#include <algorithm>
#include <array>
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
// ---------------------------------------------------------------- mode 3 (binned rANS, lblp.h)
constexpr uint32_t kEntL = 12, kEntM = 1u << kEntL;
constexpr int kEntMaxBins = 256;

struct EntPlane {
  std::vector<uint8_t> bytes;
};

// One plane (h x w) under `delta` (0: values, 1: differences down each column) -> its bytes.
void ent_plane(const uint16_t* x, uint32_t h, uint32_t w, int delta, EntPlane* out) {
  const size_t n = (size_t)h * w;
  std::vector<uint16_t> sym(n);
  for (uint32_t y = 0; y < h; ++y)
    for (uint32_t c = 0; c < w; ++c) {
      const uint16_t v = order_map(x[(size_t)y * w + c]);
      const uint16_t up = (delta && y) ? order_map(x[(size_t)(y - 1) * w + c]) : 0;
      sym[(size_t)y * w + c] = delta ? zz16((uint16_t)(v - up)) : v;
    }
  // raw low bits: the smallest b whose bins (s >> b) number at most 256
  std::vector<uint32_t> hist(65536);
  uint32_t b = 0;
  for (;; ++b) {
    std::fill(hist.begin(), hist.end(), 0u);
    int used = 0;
    for (uint16_t v : sym) used += hist[v >> b]++ == 0;
    if (used <= kEntMaxBins || b == 16) break;
  }
  std::vector<uint16_t> hi;
  std::vector<uint32_t> cnt;
  std::vector<int> bin_of(65536, -1);
  for (uint32_t v = 0; v < 65536; ++v)
    if (hist[v]) {
      bin_of[v] = (int)hi.size();
      hi.push_back((uint16_t)v);
      cnt.push_back(hist[v]);
    }
  const int K = (int)hi.size();
  // frequencies summing to M: floor(cnt * M / n) (at least 1), then unit corrections cycling over
  // the bins by (count desc, hi asc)
  std::vector<uint32_t> f(K), cum(K);
  int64_t total = 0;
  for (int k = 0; k < K; ++k) {
    f[k] = std::max<uint32_t>(1u, (uint32_t)(((uint64_t)cnt[k] * kEntM) / n));
    total += f[k];
  }
  std::vector<int> order(K);
  for (int k = 0; k < K; ++k) order[k] = k;
  std::stable_sort(order.begin(), order.end(), [&](int a, int c) { return cnt[a] > cnt[c]; });
  for (int i = 0; total < (int64_t)kEntM; i = (i + 1) % K, ++total) ++f[order[i]];
  for (int i = 0; total > (int64_t)kEntM; i = (i + 1) % K)
    if (f[order[i]] > 1) { --f[order[i]]; --total; }
  for (int k = 0, acc = 0; k < K; ++k) { cum[k] = (uint32_t)acc; acc += (int)f[k]; }

  std::vector<uint8_t>& o = out->bytes;
  auto pad4 = [&] { o.resize((o.size() + 3) & ~size_t(3), 0); };
  o.assign(16, 0);
  o[0] = (uint8_t)delta;
  o[1] = (uint8_t)kEntL;
  o[2] = (uint8_t)b;
  wr16(o.data() + 4, (uint16_t)K);
  for (int k = 0; k < K; ++k) {
    const size_t p = o.size();
    o.resize(p + 4);
    wr16(o.data() + p, hi[k]);
    wr16(o.data() + p + 2, (uint16_t)f[k]);
  }
  pad4();
  const size_t st_pos = o.size(), woff_pos = st_pos + 4 * (size_t)w;
  o.resize(woff_pos + 4 * (size_t)(w / 32), 0);
  // rANS per column; the encoder walks (y, column) backwards, so each warp's renormalisation words,
  // reversed, come out in the decoder's (y, lane) order
  std::vector<uint32_t> state(w, 1u << 16);
  std::vector<uint16_t> emitted;
  emitted.reserve(n / 4);
  for (uint32_t g = 0; g < w / 32; ++g) {
    emitted.clear();
    for (int64_t y = (int64_t)h - 1; y >= 0; --y)
      for (int l = 31; l >= 0; --l) {
        const uint32_t col = 32 * g + (uint32_t)l;
        const int k = bin_of[sym[(size_t)y * w + col] >> b];
        uint32_t st = state[col];
        if (st >= (f[k] << (32 - kEntL))) {
          emitted.push_back((uint16_t)st);
          st >>= 16;
        }
        state[col] = ((st / f[k]) << kEntL) + st % f[k] + cum[k];
      }
    wr32(o.data() + woff_pos + 4 * g, (uint32_t)o.size());
    const size_t p = o.size();
    o.resize(p + 2 * emitted.size());
    for (size_t i = 0; i < emitted.size(); ++i) wr16(o.data() + p + 2 * i, emitted[emitted.size() - 1 - i]);
    pad4();
  }
  for (uint32_t col = 0; col < w; ++col) wr32(o.data() + st_pos + 4 * col, state[col]);
  // raw low bits, column-major
  const size_t nwo = ((size_t)h * b + 31) / 32, raw = o.size();
  wr32(o.data() + 8, (uint32_t)raw);
  o.resize(raw + 4 * nwo * w, 0);
  if (b) {
    const uint32_t mask = (1u << b) - 1u;
    for (uint32_t col = 0; col < w; ++col) {
      uint32_t* words = reinterpret_cast<uint32_t*>(o.data() + raw) + nwo * col;
      uint64_t acc = 0;
      uint32_t fill = 0, wi = 0;
      for (uint32_t y = 0; y < h; ++y) {
        acc |= (uint64_t)(sym[(size_t)y * w + col] & mask) << fill;
        fill += b;
        if (fill >= 32) {
          words[wi++] = (uint32_t)acc;
          acc >>= 32;
          fill -= 32;
        }
      }
      if (fill) words[wi] = (uint32_t)acc;
    }
  }
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
  if (mode == LBLP_ENTROPY) {
    if (w % 32 || w > 1024 || (size_t)h * w > 16384) {
      if (why) *why = "lblp_pack: mode 3 needs W % 32 == 0, W <= 1024 and H*W <= 16384 (one plane per CTA)";
      return false;
    }
    const uint32_t payload = LBLP_HEADER_BYTES + 4u * c;
    out->assign(payload, 0);
    const size_t plane = (size_t)h * w;
    for (uint32_t ch = 0; ch < c; ++ch) {
      EntPlane p0, p1;
      ent_plane(x + ch * plane, h, w, 0, &p0);
      ent_plane(x + ch * plane, h, w, 1, &p1);
      const EntPlane& best = p1.bytes.size() < p0.bytes.size() ? p1 : p0;
      wr32(out->data() + LBLP_HEADER_BYTES + 4 * ch, (uint32_t)(out->size() - payload));
      out->insert(out->end(), best.bytes.begin(), best.bytes.end());
    }
    put_header(out->data(), mode, c, h, w, (uint32_t)out->size(), LBLP_HEADER_BYTES, payload);
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
    case LBLP_ENTROPY: {
      if (w % 32 || w > 1024 || (size_t)h * w > 16384)
        return fail("entropy blob needs W % 32 == 0, W <= 1024 and H*W <= 16384");
      if (table != LBLP_HEADER_BYTES || payload != LBLP_HEADER_BYTES + 4 * c || payload > nbytes)
        return fail("entropy blob bad table offsets");
      const uint32_t nwo_per_b = h;  // raw words per column = ceil(h * b / 32)
      (void)nwo_per_b;
      for (uint32_t ch = 0; ch < c; ++ch) {
        const uint32_t po = rd32(b + LBLP_HEADER_BYTES + 4 * ch);
        const uint64_t pend = ch + 1 < c ? rd32(b + LBLP_HEADER_BYTES + 4 * (ch + 1)) : nbytes - payload;
        if ((po & 3u) || pend > nbytes - payload || (uint64_t)po + 16 > pend) return fail("entropy plane out of bounds");
        const uint8_t* pl = b + payload + po;
        const uint64_t plen = pend - po;
        const uint32_t bb = pl[2], K = rd16(pl + 4), raw = rd32(pl + 8);
        if (pl[0] > 1 || pl[1] != kEntL || bb > 16 || K < 1 || K > (uint32_t)kEntMaxBins)
          return fail("entropy plane header invalid");
        const uint64_t hdr = (16u + 4u * K + 3u) & ~3u, nwo = ((uint64_t)h * bb + 31) / 32;
        if (hdr + 4ull * w + 4ull * (w / 32) > raw || (raw & 3u) || raw + 4 * nwo * w > plen)
          return fail("entropy plane sections out of bounds");
        uint32_t sum = 0, prev = 0;
        for (uint32_t k = 0; k < K; ++k) {
          const uint32_t hv = rd16(pl + 16 + 4 * k), fv = rd16(pl + 18 + 4 * k);
          if (fv == 0 || (k && hv <= prev) || (hv >> (16 - bb))) return fail("entropy bin table invalid");
          sum += fv;
          prev = hv;
        }
        if (sum != kEntM) return fail("entropy bin frequencies do not sum to 2^L");
        uint64_t lo = hdr + 4ull * w + 4ull * (w / 32);
        for (uint32_t g = 0; g < w / 32; ++g) {
          const uint32_t ws = rd32(pl + hdr + 4ull * w + 4 * g);
          if ((ws & 3u) || ws < lo || ws > raw) return fail("entropy warp stream offsets invalid");
          lo = ws;
        }
      }
      return true;
    }
    default:
      return fail("unknown LBLP mode");
  }
}

}  // namespace lbx
