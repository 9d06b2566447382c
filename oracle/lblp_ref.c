/*
 * ORACLE (test infrastructure only) -- scalar C restatement of the LBLP v1 latent codec
 * (encoder + decoder).  Normative format: include/lbx/lblp.h.
 *
 * Only tests/ and __graft_entry__.smoke() load this (oracle/_build/liblblp_ref.so via ctypes);
 * the product codec is paper_2605_19385_b200/csrc/codec.cpp (host packer) and unpack.cu (GPU).
 *
 * The reference has no codec (pcodec is external; the simulator only knows
 * ObjectMeta::latent_bytes, proj/include/latentbox/trace.hpp:21-26): parity is pinned by this
 * restatement plus the committed known-answer vectors in tests/golden/lblp_kat.json.
 *
 * Every function returns the number of bytes written/required, or a negative error:
 *   -1 bad argument, -2 bad magic/version/dtype, -3 shape mismatch, -4 truncated / out of bounds,
 *   -5 unsupported mode.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static void put16(uint8_t* p, uint16_t v) { p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); }
static void put32(uint8_t* p, uint32_t v) {
  p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); p[2] = (uint8_t)(v >> 16); p[3] = (uint8_t)(v >> 24);
}
static uint16_t get16(const uint8_t* p) { return (uint16_t)(p[0] | (p[1] << 8)); }
static uint32_t get32(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

static uint16_t omap(uint16_t u) { return (u & 0x8000u) ? (uint16_t)(~u) : (uint16_t)(u | 0x8000u); }
static uint16_t omap_inv(uint16_t v) { return (v & 0x8000u) ? (uint16_t)(v & 0x7FFFu) : (uint16_t)(~v); }
static uint16_t zigzag(uint16_t d) {
  int16_t s = (int16_t)d;
  return (uint16_t)(((uint16_t)s << 1) ^ (uint16_t)(s >> 15));
}
static uint16_t unzigzag(uint16_t z) { return (uint16_t)((z >> 1) ^ (uint16_t)(-(int)(z & 1))); }
static int bitlen(uint32_t x) { int n = 0; while (x) { n++; x >>= 1; } return n; }

static void header(uint8_t* out, int mode, int c, int h, int w, uint32_t total, uint32_t table,
                   uint32_t payload) {
  memset(out, 0, 32);
  memcpy(out, "LBLP", 4);
  out[4] = 1; out[5] = 1; out[6] = (uint8_t)mode;
  put16(out + 8, (uint16_t)c); put16(out + 10, (uint16_t)h); put16(out + 12, (uint16_t)w);
  put32(out + 16, total); put32(out + 20, table); put32(out + 24, payload);
}

/* Size of one mode-1 row, in bytes, for the values src[0..w). */
static uint32_t row_bytes(const uint16_t* src, int w) {
  uint32_t head = 2u + (uint32_t)(w / 32);
  head = (head + 3u) & ~3u;
  uint32_t words = 0;
  uint16_t prev = 0;
  for (int j = 0; j < w / 32; j++) {
    uint32_t mx = 0;
    for (int k = 0; k < 32; k++) {
      int i = 32 * j + k;
      uint16_t v = omap(src[i]);
      uint16_t z = i == 0 ? 0 : zigzag((uint16_t)(v - prev));
      prev = v;
      if (z > mx) mx = z;
    }
    words += (uint32_t)bitlen(mx);
  }
  return head + 4u * words;
}

/* Bytes an encoding of fp16 NCHW `src` (c*h*w values) needs in `mode`. */
long lblp_ref_encoded_size(const uint16_t* src, int mode, int c, int h, int w) {
  if (c <= 0 || h <= 0 || w <= 0 || c > 65535 || h > 65535 || w > 65535) return -1;
  size_t n = (size_t)c * h * w;
  if (mode == 0) return (long)(32 + 2 * n);
  if (mode == 2) return (long)(32 + 8 * (size_t)c + n);
  if (mode != 1) return -5;
  if (w % 32) return -3;
  size_t total = 32 + 4 * (size_t)c * h;
  for (size_t r = 0; r < (size_t)c * h; r++) total += row_bytes(src + r * w, w);
  return (long)total;
}

long lblp_ref_encode(const uint16_t* src, int mode, int c, int h, int w, uint8_t* out, long cap) {
  long need = lblp_ref_encoded_size(src, mode, c, h, w);
  if (need < 0) return need;
  if (cap < need) return -4;
  size_t n = (size_t)c * h * w;
  memset(out, 0, (size_t)need);
  if (mode == 0) {
    header(out, 0, c, h, w, (uint32_t)need, 0, 32);
    for (size_t i = 0; i < n; i++) put16(out + 32 + 2 * i, src[i]);
    return need;
  }
  if (mode == 2) {
    uint32_t payload = 32u + 8u * (uint32_t)c;
    header(out, 2, c, h, w, (uint32_t)need, 32, payload);
    size_t plane = (size_t)h * w;
    for (int ch = 0; ch < c; ch++) {
      /* fp16 -> float via the exact bit formula (no host half type needed) */
      float mn = INFINITY, mx = -INFINITY;
      for (size_t i = 0; i < plane; i++) {
        uint16_t u = src[ch * plane + i];
        int e = (u >> 10) & 31, m = u & 1023;
        float f = e == 0 ? ldexpf((float)m, -24) : (e == 31 ? (m ? NAN : INFINITY) : ldexpf((float)(m | 1024), e - 25));
        if (u & 0x8000) f = -f;
        if (isfinite(f)) { if (f < mn) mn = f; if (f > mx) mx = f; }
      }
      if (!(mn <= mx)) { mn = 0.f; mx = 0.f; }
      float scale = (mx - mn) / 255.0f;
      if (!(scale > 0.f)) scale = 1.0f;
      int32_t zp = -128 - (int32_t)lrintf(mn / scale);
      memcpy(out + 32 + 4 * ch, &scale, 4);
      put32(out + 32 + 4 * (size_t)c + 4 * ch, (uint32_t)zp);
      for (size_t i = 0; i < plane; i++) {
        uint16_t u = src[ch * plane + i];
        int e = (u >> 10) & 31, m = u & 1023;
        float f = e == 0 ? ldexpf((float)m, -24) : (e == 31 ? (m ? NAN : INFINITY) : ldexpf((float)(m | 1024), e - 25));
        if (u & 0x8000) f = -f;
        long q = isfinite(f) ? lrintf(f / scale) + zp : (f > 0 ? 127 : -128);
        if (q < -128) q = -128;
        if (q > 127) q = 127;
        out[payload + ch * plane + i] = (uint8_t)(int8_t)q;
      }
    }
    return need;
  }
  /* mode 1 */
  uint32_t rows = (uint32_t)c * h;
  uint32_t payload = 32u + 4u * rows;
  header(out, 1, c, h, w, (uint32_t)need, 32, payload);
  uint32_t off = 0;
  for (uint32_t r = 0; r < rows; r++) {
    const uint16_t* s = src + (size_t)r * w;
    put32(out + 32 + 4 * r, off);
    uint8_t* row = out + payload + off;
    put16(row, s[0]);
    uint32_t head = (2u + (uint32_t)(w / 32) + 3u) & ~3u;
    uint32_t wpos = head;
    uint16_t prev = 0;
    for (int j = 0; j < w / 32; j++) {
      uint16_t z[32];
      uint32_t mx = 0;
      for (int k = 0; k < 32; k++) {
        int i = 32 * j + k;
        uint16_t v = omap(s[i]);
        z[k] = i == 0 ? 0 : zigzag((uint16_t)(v - prev));
        prev = v;
        if (z[k] > mx) mx = z[k];
      }
      int bw = bitlen(mx);
      row[2 + j] = (uint8_t)bw;
      uint32_t words[16] = {0};
      for (int k = 0; k < 32; k++) {
        uint32_t bit = (uint32_t)(k * bw);
        words[bit >> 5] |= (uint32_t)z[k] << (bit & 31);
        if ((bit & 31) + (uint32_t)bw > 32) words[(bit >> 5) + 1] |= (uint32_t)z[k] >> (32 - (bit & 31));
      }
      for (int q = 0; q < bw; q++) put32(row + wpos + 4 * q, words[q]);
      wpos += 4u * (uint32_t)bw;
    }
    off += wpos;
  }
  return need;
}

/* Decode one blob to fp16 NCHW `dst` (c*h*w values).  Shape must equal (c,h,w). */
long lblp_ref_decode(const uint8_t* blob, long nbytes, int c, int h, int w, uint16_t* dst) {
  if (!blob || nbytes < 32) return -4;
  if (memcmp(blob, "LBLP", 4) || blob[4] != 1 || blob[5] != 1) return -2;
  int mode = blob[6];
  if (get16(blob + 8) != c || get16(blob + 10) != h || get16(blob + 12) != w) return -3;
  uint32_t total = get32(blob + 16), table = get32(blob + 20), payload = get32(blob + 24);
  if ((long)total != nbytes) return -4;
  size_t n = (size_t)c * h * w;
  if (mode == 0) {
    if (payload != 32 || (size_t)total < 32 + 2 * n) return -4;
    for (size_t i = 0; i < n; i++) dst[i] = get16(blob + payload + 2 * i);
    return (long)n;
  }
  if (mode == 2) {
    if (table != 32 || payload != 32u + 8u * (uint32_t)c || (size_t)total < payload + n) return -4;
    size_t plane = (size_t)h * w;
    for (int ch = 0; ch < c; ch++) {
      float scale;
      memcpy(&scale, blob + 32 + 4 * ch, 4);
      int32_t zp = (int32_t)get32(blob + 32 + 4 * (size_t)c + 4 * ch);
      for (size_t i = 0; i < plane; i++) {
        int32_t q = (int8_t)blob[payload + ch * plane + i];
        volatile float f = (float)(q - zp) * scale; /* one fp32 rounding, no contraction */
        /* float -> fp16 round-to-nearest-even, done in integer arithmetic */
        uint32_t b; float ff = f; memcpy(&b, &ff, 4);
        uint32_t sign = (b >> 16) & 0x8000u, e = (b >> 23) & 255u, m = b & 0x7FFFFFu;
        uint16_t hbits;
        if (e == 255) hbits = (uint16_t)(sign | 0x7C00u | (m ? 0x200u : 0));
        else {
          int ee = (int)e - 127 + 15;
          if (ee >= 31) hbits = (uint16_t)(sign | 0x7C00u);
          else if (ee <= 0) {
            if (ee < -10) hbits = (uint16_t)sign;
            else {
              uint32_t mm = m | 0x800000u;
              int shift = 14 - ee;
              uint32_t v = mm >> shift, rem = mm & ((1u << shift) - 1), half = 1u << (shift - 1);
              if (rem > half || (rem == half && (v & 1))) v++;
              hbits = (uint16_t)(sign | v);
            }
          } else {
            uint32_t v = ((uint32_t)ee << 10) | (m >> 13), rem = m & 0x1FFFu;
            if (rem > 0x1000u || (rem == 0x1000u && (v & 1))) v++;
            hbits = (uint16_t)(sign | v);
          }
        }
        dst[ch * plane + i] = hbits;
      }
    }
    return (long)n;
  }
  if (mode != 1) return -5;
  if (w % 32) return -3;
  uint32_t rows = (uint32_t)c * h;
  if (table != 32 || payload != 32u + 4u * rows || payload > total) return -4;
  uint32_t head = (2u + (uint32_t)(w / 32) + 3u) & ~3u;
  for (uint32_t r = 0; r < rows; r++) {
    uint32_t off = get32(blob + 32 + 4 * r);
    if ((uint64_t)payload + off + head > total) return -4;
    const uint8_t* row = blob + payload + off;
    uint16_t v = omap(get16(row)); /* row header holds the raw fp16 bits of value 0 */
    uint32_t wpos = head;
    for (int j = 0; j < w / 32; j++) {
      int bw = row[2 + j];
      if (bw > 16) return -4;
      if ((uint64_t)payload + off + wpos + 4u * (uint32_t)bw > total) return -4;
      for (int k = 0; k < 32; k++) {
        uint32_t z = 0;
        if (bw) {
          uint32_t bit = (uint32_t)(k * bw);
          uint32_t lo = get32(row + wpos + 4 * (bit >> 5)) >> (bit & 31);
          if ((bit & 31) + (uint32_t)bw > 32) lo |= get32(row + wpos + 4 * ((bit >> 5) + 1)) << (32 - (bit & 31));
          z = lo & ((1u << bw) - 1u);
        }
        int i = 32 * j + k;
        if (i > 0) v = (uint16_t)(v + unzigzag((uint16_t)z));
        dst[(size_t)r * w + i] = omap_inv(v);
      }
      wpos += 4u * (uint32_t)bw;
    }
  }
  return (long)n;
}
