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

/* ---------------------------------------------------------------- mode 3 (binned rANS)
 * Restatement of include/lbx/lblp.h "mode 3".  Per channel plane: symbols are the order-mapped
 * values (delta 0) or the zigzagged vertical differences (delta 1); a symbol s is coded as its bin
 * hi = s >> b with a 12-bit rANS (one stream per column, 16-bit renormalisation) plus the low b bits
 * raw.  The encoder tries delta 0 and 1 and keeps the smaller plane (ties: delta 0). */
#define M3_L 12
#define M3_M (1u << M3_L)
#define M3_KMAX 256

typedef struct { uint8_t* p; size_t n, cap; } buf_t;
static int bput(buf_t* b, const void* src, size_t k) {
  if (b->n + k > b->cap) {
    size_t nc = b->cap ? b->cap * 2 : 65536;
    while (nc < b->n + k) nc *= 2;
    uint8_t* q = (uint8_t*)realloc(b->p, nc);
    if (!q) return -1;
    b->p = q; b->cap = nc;
  }
  if (src) memcpy(b->p + b->n, src, k); else memset(b->p + b->n, 0, k);
  b->n += k;
  return 0;
}
static void bpad4(buf_t* b) { while (b->n & 3) bput(b, NULL, 1); }
static void bput16(buf_t* b, uint16_t v) { uint8_t t[2]; put16(t, v); bput(b, t, 2); }


/* symbols of one plane under `delta` */
static void m3_symbols(const uint16_t* plane, int h, int w, int delta, uint16_t* sym) {
  for (int y = 0; y < h; y++)
    for (int x = 0; x < w; x++) {
      uint16_t u = omap(plane[(size_t)y * w + x]);
      if (!delta) { sym[(size_t)y * w + x] = u; continue; }
      uint16_t up = y ? omap(plane[(size_t)(y - 1) * w + x]) : 0;
      sym[(size_t)y * w + x] = zigzag((uint16_t)(u - up));
    }
}

/* encode one plane with a given delta into b (appended); returns 0 or -1 */
static int m3_plane(const uint16_t* plane, int h, int w, int delta, buf_t* b) {
  size_t n = (size_t)h * w;
  uint16_t* sym = (uint16_t*)malloc(n * 2);
  uint32_t* cnt = (uint32_t*)calloc(65536, 4);
  if (!sym || !cnt) { free(sym); free(cnt); return -1; }
  m3_symbols(plane, h, w, delta, sym);
  int bb = 0;
  for (; bb <= 16; bb++) { /* smallest b with <= 256 occupied bins */
    memset(cnt, 0, 65536 * 4);
    int k = 0;
    for (size_t i = 0; i < n; i++) if (cnt[sym[i] >> bb]++ == 0) k++;
    if (k <= M3_KMAX) break;
  }
  /* bins in ascending hi */
  uint16_t hi[M3_KMAX]; uint32_t nk[M3_KMAX], f[M3_KMAX], cum[M3_KMAX];
  int K = 0;
  for (uint32_t v = 0; v < 65536u; v++) if (cnt[v]) { hi[K] = (uint16_t)v; nk[K] = cnt[v]; K++; }
  /* frequencies: max(1, floor(n_k * M / N)), then fix the sum cycling through bins ordered by
   * (count desc, hi asc): +1 each while short, -1 (only where > 1) while over */
  int order[M3_KMAX];
  long sum = 0;
  for (int k = 0; k < K; k++) {
    f[k] = (uint32_t)(((uint64_t)nk[k] * M3_M) / n);
    if (f[k] == 0) f[k] = 1;
    sum += f[k];
    order[k] = k;
  }
  for (int a = 1; a < K; a++) { /* insertion sort: count desc, hi asc */
    int t = order[a], j = a - 1;
    while (j >= 0 && (nk[order[j]] < nk[t] || (nk[order[j]] == nk[t] && hi[order[j]] > hi[t]))) { order[j + 1] = order[j]; j--; }
    order[j + 1] = t;
  }
  for (int r = 0; sum < (long)M3_M; r = (r + 1) % K) { f[order[r]]++; sum++; }
  for (int r = 0; sum > (long)M3_M; r = (r + 1) % K) if (f[order[r]] > 1) { f[order[r]]--; sum--; }
  uint32_t c0 = 0;
  for (int k = 0; k < K; k++) { cum[k] = c0; c0 += f[k]; }
  int* kof = (int*)malloc(65536 * sizeof(int));
  uint32_t* st = (uint32_t*)malloc((size_t)w * 4);
  uint16_t* words = (uint16_t*)malloc(n * 2 + 2);
  if (!kof || !st || !words) { free(kof); free(st); free(words); free(sym); free(cnt); return -1; }
  for (int k = 0; k < K; k++) kof[hi[k]] = k;
  /* rANS per column, encoded in reverse (y, x) order; the renormalisation words of warp g's 32
   * columns are emitted into one sequence and stored reversed (= the decoder's read order) */
  for (int x = 0; x < w; x++) st[x] = 1u << 16;
  size_t pstart = b->n;
  uint8_t hd[16] = {(uint8_t)delta, (uint8_t)M3_L, (uint8_t)bb, 0};
  put16(hd + 4, (uint16_t)K);
  bput(b, hd, 16);
  for (int k = 0; k < K; k++) { bput16(b, hi[k]); bput16(b, (uint16_t)f[k]); }
  bpad4(b);
  size_t stpos = b->n;
  bput(b, NULL, 4 * (size_t)w + 4 * (size_t)(w / 32));
  for (int g = 0; g < w / 32; g++) {
    size_t nw = 0;
    for (int y = h - 1; y >= 0; y--)
      for (int x = 32 * g + 31; x >= 32 * g; x--) {
        int k = kof[sym[(size_t)y * w + x] >> bb];
        uint32_t xmax = f[k] << (32 - M3_L); /* ((2^16 >> L) << 16) * f */
        uint32_t v = st[x];
        if (v >= xmax) { words[nw++] = (uint16_t)(v & 0xFFFFu); v >>= 16; }
        st[x] = ((v / f[k]) << M3_L) + (v % f[k]) + cum[k];
      }
    put32(b->p + stpos + 4 * (size_t)w + 4 * (size_t)g, (uint32_t)(b->n - pstart));
    for (size_t q = 0; q < nw; q++) bput16(b, words[nw - 1 - q]);
    bpad4(b);
  }
  for (int x = 0; x < w; x++) put32(b->p + stpos + 4 * (size_t)x, st[x]);
  /* raw low bits: column-major, column x's ceil(H*b/32) words, value y at bit y*b, LSB-first */
  size_t nwo = ((size_t)h * bb + 31) / 32;
  put32(b->p + pstart + 8, (uint32_t)(b->n - pstart));
  size_t ow0 = b->n;
  bput(b, NULL, 4 * nwo * (size_t)w);
  if (bb)
    for (int x = 0; x < w; x++) {
      uint8_t* ow = b->p + ow0 + 4 * nwo * (size_t)x;
      uint32_t msk = (1u << bb) - 1u;
      for (int y = 0; y < h; y++) {
        uint32_t o = sym[(size_t)y * w + x] & msk, bit = (uint32_t)y * bb;
        uint8_t* wp = ow + 4 * (bit >> 5);
        put32(wp, get32(wp) | (o << (bit & 31)));
        if ((bit & 31) + bb > 32) put32(wp + 4, get32(wp + 4) | (o >> (32 - (bit & 31))));
      }
    }
  free(words); free(st); free(kof); free(sym); free(cnt);
  return 0;
}

/* whole mode-3 blob into a malloc'd buffer; returns its size or a negative error */
static long m3_encode(const uint16_t* src, int c, int h, int w, uint8_t** outp) {
  if (w % 32 || w > 1024) return -3;
  buf_t b = {0, 0, 0};
  bput(&b, NULL, 32 + 4 * (size_t)c);
  size_t plane = (size_t)h * w;
  for (int ch = 0; ch < c; ch++) {
    buf_t t[2] = {{0, 0, 0}, {0, 0, 0}};
    for (int d = 0; d < 2; d++)
      if (m3_plane(src + ch * plane, h, w, d, &t[d])) { free(t[0].p); free(t[1].p); free(b.p); return -1; }
    int best = t[1].n < t[0].n ? 1 : 0;
    put32(b.p + 32 + 4 * ch, (uint32_t)(b.n - (32 + 4 * (size_t)c)));
    bput(&b, t[best].p, t[best].n);
    free(t[0].p); free(t[1].p);
  }
  header(b.p, 3, c, h, w, (uint32_t)b.n, 32, 32u + 4u * (uint32_t)c);
  *outp = b.p;
  return (long)b.n;
}

/* decode one mode-3 blob (already checked: magic, shape, total) */
static long m3_decode(const uint8_t* blob, uint32_t total, uint32_t table, uint32_t payload, int c, int h, int w,
                      uint16_t* dst) {
  if (w % 32 || w > 1024 || table != 32 || payload != 32u + 4u * (uint32_t)c || payload > total) return -4;
  for (int ch = 0; ch < c; ch++) {
    uint32_t po = get32(blob + 32 + 4 * ch);
    uint32_t pend = ch + 1 < c ? get32(blob + 32 + 4 * (ch + 1)) : total - payload;
    if ((po & 3) || pend > total - payload || (uint64_t)po + 16 > pend) return -4;
    const uint8_t* pl = blob + payload + po;
    uint32_t plen = pend - po;
    int delta = pl[0], L = pl[1], bb = pl[2], K = get16(pl + 4);
    uint32_t opos = get32(pl + 8);
    if (delta > 1 || L != M3_L || bb > 16 || K < 1 || K > M3_KMAX) return -4;
    uint32_t hdr = (16u + 4u * (uint32_t)K + 3u) & ~3u;
    uint32_t nwo = (uint32_t)(((size_t)h * bb + 31) / 32);
    if ((uint64_t)hdr + 4ull * w + 4ull * (w / 32) > opos || (opos & 3) || (uint64_t)opos + 4ull * nwo * w > plen)
      return -4;
    uint16_t hi[M3_KMAX]; uint32_t f[M3_KMAX], cum[M3_KMAX];
    uint8_t slot2k[M3_M];
    uint32_t c0 = 0;
    for (int k = 0; k < K; k++) {
      hi[k] = get16(pl + 16 + 4 * k);
      f[k] = get16(pl + 18 + 4 * k);
      if (f[k] == 0 || (k && hi[k] <= hi[k - 1]) || (hi[k] >> (16 - bb))) return -4;
      cum[k] = c0; c0 += f[k];
      if (c0 > M3_M) return -4;
      for (uint32_t sl = cum[k]; sl < c0; sl++) slot2k[sl] = (uint8_t)k;
    }
    if (c0 != M3_M) return -4;
    for (int g = 0; g < w / 32; g++) {
      uint32_t ws = get32(pl + hdr + 4 * w + 4 * g);
      uint32_t we = g + 1 < w / 32 ? get32(pl + hdr + 4 * w + 4 * (g + 1)) : opos;
      if ((ws & 3) || ws < hdr + 4u * w + 4u * (w / 32) || we > opos || ws > we) return -4;
      uint32_t nw = (we - ws) / 2, wi = 0;
      uint32_t st[32];
      uint16_t prev[32];
      for (int l = 0; l < 32; l++) { st[l] = get32(pl + hdr + 4 * (32 * g + l)); prev[l] = 0; }
      for (int y = 0; y < h; y++)
        for (int l = 0; l < 32; l++) { /* lane order within the warp = word order */
          int x = 32 * g + l;
          uint32_t sl = st[l] & (M3_M - 1);
          int k = slot2k[sl];
          st[l] = f[k] * (st[l] >> M3_L) + sl - cum[k];
          if (st[l] < (1u << 16)) {
            if (wi >= nw) return -4;
            st[l] = (st[l] << 16) | get16(pl + ws + 2 * wi);
            wi++;
          }
          uint32_t o = 0;
          if (bb) {
            const uint8_t* ow = pl + opos + 4 * (size_t)nwo * x;
            uint32_t bit = (uint32_t)y * bb;
            uint32_t lo = get32(ow + 4 * (bit >> 5)) >> (bit & 31);
            if ((bit & 31) + bb > 32) lo |= get32(ow + 4 * ((bit >> 5) + 1)) << (32 - (bit & 31));
            o = lo & ((1u << bb) - 1u);
          }
          uint16_t symv = (uint16_t)((bb == 16 ? 0u : ((uint32_t)hi[k] << bb)) | o);
          uint16_t u = delta ? (uint16_t)(prev[l] + unzigzag(symv)) : symv;
          prev[l] = u;
          dst[(size_t)ch * h * w + (size_t)y * w + x] = omap_inv(u);
        }
    }
  }
  return (long)c * h * w;
}

/* Bytes an encoding of fp16 NCHW `src` (c*h*w values) needs in `mode`. */
long lblp_ref_encoded_size(const uint16_t* src, int mode, int c, int h, int w) {
  if (c <= 0 || h <= 0 || w <= 0 || c > 65535 || h > 65535 || w > 65535) return -1;
  size_t n = (size_t)c * h * w;
  if (mode == 0) return (long)(32 + 2 * n);
  if (mode == 2) return (long)(32 + 8 * (size_t)c + n);
  if (mode == 3) {
    uint8_t* p = NULL;
    long r = m3_encode(src, c, h, w, &p);
    free(p);
    return r;
  }
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
  if (mode == 3) {
    uint8_t* p = NULL;
    long r = m3_encode(src, c, h, w, &p);
    if (r > 0) memcpy(out, p, (size_t)r);
    free(p);
    return r;
  }
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
  if (mode == 3) return m3_decode(blob, total, table, payload, c, h, w, dst);
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
