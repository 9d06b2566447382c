// PNG encode of decoded RGB on the GPU -- SURVEY.md 8(f) item 3: the paper encodes the returned
// image as PNG in a CPU compute pool (~10 ms network for the PNG); here
// the uint8 RGB the decoder leaves in HBM is encoded where it lies and only the PNG crosses PCIe.
//
// Format (PNG 1.2 / RFC 1950 zlib / RFC 1951 DEFLATE): signature, IHDR (8-bit RGB, no interlace),
// one IDAT chunk per strip of R rows, IEND.  The zlib stream is the concatenation of the strips'
// DEFLATE data: every strip is one block (dynamic Huffman, or stored when that is smaller); a
// non-final strip ends with an empty stored block (a "sync flush") so the next strip starts on a
// byte boundary, and its matches may reach back into the previous strip's last row (the inflater
// keeps a 32 KB window across blocks).
//
//   K-a png_strip_kernel   one CTA per strip: per-row filter choice, one warp per row (the minimum
//                          sum of |signed residual| over the five PNG filters, the libpng
//                          heuristic); LZ77 parse in 255 independent segments (greedy, distances
//                          {1, 3, 6, row}); Huffman codes length-limited to 15 / 7, built in
//                          phases (bitonic symbol sort, one-thread merge per alphabet, parallel
//                          depths / lengths / canonical codes); the block header as a parallel
//                          run-length coding; bit packing through per-thread offsets from block
//                          scans; Adler-32 partials of the strip.
//   K-b png_image_kernel   one CTA per image: Adler-32 combine, chunk offsets (scan), total size.
//   K-b2 png_frame_kernel  image bases (strided, or packed back to back), signature, IHDR, IEND.
//   K-c png_chunk_kernel   one CTA per strip: copy the strip's data to its chunk and CRC-32 it
//                          (per-thread segments combined by multiplication by x^(8n) mod P).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gemm_tc.cuh"
#include "kernels.cuh"

namespace lbx {

namespace {

constexpr int kT = 256;                 // threads per CTA
constexpr int kMaxStripBytes = 32768;   // filtered bytes per strip
constexpr uint32_t kAdler = 65521u;
constexpr uint32_t kCrcPoly = 0xEDB88320u;

struct StripMeta {
  uint32_t bytes;  // zlib bytes of the strip (incl. the 4 Adler-32 bytes of the last strip)
  uint32_t a, b;   // Adler-32 partials of the strip's filtered bytes (mod 65521)
  uint32_t rsv;
};

struct PngGeom {
  int n, H, W;
  int RS;       // filtered row bytes, 3W + 1
  int R;        // rows per strip
  int nstrips;  // strips per image
  int cap;      // scratch bytes per strip
  int G;        // parse segment bytes per thread
  int MC;       // LZ77 matches kept per parse segment
  unsigned long long* tl;  // diagnostics (LBX_PNG_TIMING): per-strip phase timestamps, or null
  // dynamic smem layout (bytes): raw rows, then Huffman work arrays, then the output words share
  // offset 0 (each dead before the next); filtered rows, match lists and tables follow
  int off_filt, off_ml, off_tab, smem;
};

__host__ __device__ inline int strip_rows(const PngGeom& g, int s) {
  const int r = g.H - s * g.R;
  return r < g.R ? r : g.R;
}

// --------------------------------------------------------------------------- DEFLATE symbol maps
__device__ __forceinline__ void len_sym(int len, int& code, int& nb, int& ev) {  // RFC 1951 3.2.5
  if (len <= 10) { code = 254 + len; nb = 0; ev = 0; return; }
  if (len == 258) { code = 285; nb = 0; ev = 0; return; }
  const int l = len - 3;
  nb = 29 - __clz(l);  // floor(log2 l) - 2
  code = 257 + 4 * (nb + 1) + ((l >> nb) & 3);
  ev = l & ((1 << nb) - 1);
}
__device__ __forceinline__ void dist_sym(int d, int& code, int& nb, int& ev) {
  const int v = d - 1;
  if (v < 4) { code = v; nb = 0; ev = 0; return; }
  nb = 30 - __clz(v);  // floor(log2 v) - 1
  code = 2 * (nb + 1) + ((v >> nb) & 1);
  ev = v & ((1 << nb) - 1);
}

__device__ __forceinline__ uint32_t rev_bits(uint32_t c, int n) { return __brev(c) >> (32 - n); }

// --------------------------------------------------------------------------- Huffman construction
// The literal/length (286 symbols) and distance (30) codes are built in phases spread over the CTA,
// so that only the inherently sequential part -- the two-queue merge of the rank-sorted leaves and
// the depths of the m-1 internal nodes -- runs on a single thread (a different warp per alphabet):
//   rank sort (all threads) -> merge (1 thread per alphabet) -> leaf depths and per-length counts
//   (all) -> Kraft repair of the counts to <= 15 bits (1 thread) -> lengths by frequency rank and
//   canonical codes (all).
// Fewer than two used symbols get a dummy second code so every code is complete (zlib's inflate
// rejects incomplete codes other than a single distance code).
template <int N>
struct Alpha {
  uint32_t wl[N];  // leaf weights in rank order
  uint32_t wi[N];  // internal node weights
  uint16_t pl[N];  // parent (internal index) of each leaf
  uint16_t pi[N];  // parent of each internal node
  uint8_t di[N];   // internal node depth (saturating)
};
struct HuffWork {
  Alpha<286> lit;
  Alpha<30> dst;
  uint32_t keys[512];       // bitonic sort keys: (freq << 9 | sym) literal/length, (1 << 31 | freq << 5 | sym) distance
  uint32_t ccnt[10][32];    // canonical codes: per 32-symbol chunk, count per (alphabet, length)
};

// code-length run-length coding (RFC 1951 3.2.7) of one maximal run of `run` copies of `v`:
// returns the token count; writes the tokens (sym | extra << 5) when out != null
__device__ __forceinline__ int rle_run(int v, int run, uint16_t* out) {
  int n = 0;
  if (v == 0) {
    int r = run;
    while (r >= 11) { const int k = r < 138 ? r : 138; if (out) out[n] = (uint16_t)(18 | ((k - 11) << 5)); ++n; r -= k; }
    if (r >= 3) { if (out) out[n] = (uint16_t)(17 | ((r - 3) << 5)); ++n; r = 0; }
    for (; r > 0; --r) { if (out) out[n] = 0; ++n; }
  } else {
    if (out) out[n] = (uint16_t)v;
    ++n;
    int r = run - 1;
    while (r >= 3) { const int k = r < 6 ? r : 6; if (out) out[n] = (uint16_t)(16 | ((k - 3) << 5)); ++n; r -= k; }
    for (; r > 0; --r) { if (out) out[n] = (uint16_t)v; ++n; }
  }
  return n;
}

__device__ void huff_merge(const uint32_t* wl, uint32_t* wi, uint16_t* pl, uint16_t* pi, uint8_t* di, int m) {
  int li = 0, ii = 0, ni = 0;
  uint32_t hl = wl[0], hl1 = m > 1 ? wl[1] : 0u, hi = 0;  // queue heads (next leaf prefetched)
  for (int k = 0; k < m - 1; ++k) {
    uint32_t w2 = 0;
#pragma unroll
    for (int pick = 0; pick < 2; ++pick) {
      if (li < m && (ii >= ni || hl <= hi)) {
        w2 += hl;
        pl[li++] = (uint16_t)ni;
        hl = hl1;
        hl1 = li + 1 < m ? wl[li + 1] : 0u;
      } else {
        w2 += hi;
        pi[ii++] = (uint16_t)ni;
        hi = ii < ni ? wi[ii] : 0u;
      }
    }
    wi[ni++] = w2;
    if (ii == ni - 1) hi = w2;
  }
  di[ni - 1] = 0;  // root; parents have larger indices
  for (int j = ni - 2; j >= 0; --j) {
    const int d = di[pi[j]] + 1;
    di[j] = (uint8_t)(d > 255 ? 255 : d);
  }
}

// Kraft repair of per-length counts (cnt[1..L], overlong codes already counted at L), then the
// canonical first code of every length (RFC 1951 3.2.2)
__device__ void huff_repair(uint32_t* cnt, uint32_t* next, int L) {
  uint32_t total = 0;
  for (int i = 1; i <= L; ++i) total += cnt[i] << (L - i);
  while (total > (1u << L)) {
    --cnt[L];
    for (int i = L - 1; i > 0; --i)
      if (cnt[i]) { --cnt[i]; cnt[i + 1] += 2; break; }
    --total;
  }
  uint32_t code = 0;
  next[0] = 0;
  for (int b = 1; b <= L; ++b) {
    code = (code + (b > 1 ? cnt[b - 1] : 0u)) << 1;
    next[b] = code;
  }
}

// small alphabets (the 19 code-length symbols): all on one thread
__device__ void huff_small(const uint32_t* freq, int n, const uint16_t* order, int m, int L, uint8_t* lens,
                           uint16_t* codes) {
  uint32_t w[20], wi[20];
  uint16_t pl[20], pi[20];
  uint8_t di[20];
  for (int i = 0; i < n; ++i) lens[i] = 0;
  uint32_t cnt[16] = {0}, next[16];
  if (m < 2) {
    const int a = m == 1 ? order[0] : 0;
    lens[a] = 1;
    lens[a == 0 ? 1 : 0] = 1;
    cnt[1] = 2;
  } else {
    for (int i = 0; i < m; ++i) w[i] = freq[order[i]];
    huff_merge(w, wi, pl, pi, di, m);
    for (int i = 0; i < m; ++i) {
      const int d = di[pl[i]] + 1;
      ++cnt[d > L ? L : d];
    }
  }
  huff_repair(cnt, next, L);
  if (m >= 2) {
    int r = 0;
    for (int len = L; len >= 1; --len)
      for (uint32_t c = 0; c < cnt[len]; ++c) lens[order[r++]] = (uint8_t)len;
  }
  for (int i = 0; i < n; ++i) codes[i] = lens[i] ? (uint16_t)rev_bits(next[lens[i]]++, lens[i]) : (uint16_t)0;
}

// LSB-first bit writer into a zeroed word buffer (words shared with neighbours: atomicOr)
struct BitW {
  uint32_t* w;
  uint32_t pos;  // word index
  uint64_t acc;
  int nacc;
  __device__ BitW(uint32_t* words, uint32_t bit) : w(words), pos(bit >> 5), acc(0), nacc((int)(bit & 31)) {}
  __device__ __forceinline__ void put(uint32_t v, int n) {
    acc |= (uint64_t)v << nacc;
    nacc += n;
    if (nacc >= 32) {
      atomicOr(&w[pos++], (uint32_t)acc);
      acc >>= 32;
      nacc -= 32;
    }
  }
  __device__ __forceinline__ void flush() {
    if (nacc > 0) atomicOr(&w[pos], (uint32_t)acc);
  }
};

__device__ __forceinline__ int paeth(int a, int b, int c) {
  const int p = a + b - c, pa = abs(p - a), pb = abs(p - b), pc = abs(p - c);
  return (pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c);
}

__device__ __forceinline__ uint8_t filt_byte(int type, int x, int a, int b, int c) {
  switch (type) {
    case 0: return (uint8_t)x;
    case 1: return (uint8_t)(x - a);
    case 2: return (uint8_t)(x - b);
    case 3: return (uint8_t)(x - ((a + b) >> 1));
    default: return (uint8_t)(x - paeth(a, b, c));
  }
}

__device__ __forceinline__ uint32_t block_sum_u32(uint32_t v, uint32_t* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  uint32_t s = 0;
  for (int i = 0; i < kT / 32; ++i) s += red[i];
  return s;
}

// exclusive block scan of per-thread values; returns this thread's prefix, *total the sum
__device__ __forceinline__ uint32_t block_scan_u32(uint32_t v, uint32_t* red, uint32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  __syncthreads();
  if (lane == 31) red[wid] = inc;
  __syncthreads();
  uint32_t before = 0, all = 0;
  for (int i = 0; i < kT / 32; ++i) {
    if (i < wid) before += red[i];
    all += red[i];
  }
  *total = all;
  return before + inc - v;
}

struct StripTables {
  uint32_t lfreq[286 + 30];  // literal/length then distance frequencies
  uint32_t cfreq[19];
  uint32_t cnt[2][16];       // code lengths per length (literal/length, distance)
  uint32_t next[2][16];      // canonical first code per length
  uint16_t order[320];       // used symbols by (freq, symbol): literal/length at 0, distance at 286
  uint16_t corder[19];
  uint8_t llen[286 + 30];
  uint8_t clen[19];
  uint16_t lcode[286 + 30];
  uint16_t ccode[19];
  uint16_t rle[320];   // code-length RLE symbols (sym | extra << 5)
  uint16_t rle_off[320];  // their bit offsets within the header's RLE part
  uint32_t red[kT / 32];
  uint32_t scal[8];    // 0 nrle, 1 hlit, 2 hdist, 3 hclen, 4 header bits, 5 m_lit, 6 m_dist
  uint8_t nmatch[kT];
  unsigned long long ab[2][kT / 32];
  uint32_t fsum[5][kT / 32];
};

// short match distances (1, 3, 6 bytes back); the fourth candidate is the row above (RS)
__device__ __forceinline__ int short_dist(int di) { return di == 0 ? 1 : di == 1 ? 3 : 6; }

__device__ __forceinline__ void png_mark(const PngGeom& g, int i) {
  if (g.tl && threadIdx.x == 0) {
    unsigned long long ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    g.tl[blockIdx.x * 16 + i] = ns;
  }
}

__global__ void __launch_bounds__(kT) png_strip_kernel(const uint8_t* __restrict__ rgb, PngGeom g,
                                                       uint8_t* __restrict__ scratch, StripMeta* __restrict__ meta) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int t = threadIdx.x;
  const int img = blockIdx.x / g.nstrips, s = blockIdx.x - img * g.nstrips;
  const int y0 = s * g.R, rows = strip_rows(g, s);
  const int rb = 3 * g.W, RS = g.RS;
  const int S = rows * RS;
  const bool first = s == 0, last = s == g.nstrips - 1;
  uint8_t* raw = sm;                        // rows y0-2 .. y0+rows-1 (3W bytes each), until filtered
  HuffWork& hw = *reinterpret_cast<HuffWork*>(sm);   // then the Huffman work arrays
  uint32_t* ow = reinterpret_cast<uint32_t*>(sm);    // then the strip's zlib bytes
  uint8_t* filt = sm + g.off_filt;          // row y0-1 then the strip's rows (RS bytes each)
  uint32_t* mlist = reinterpret_cast<uint32_t*>(sm + g.off_ml);  // per-thread LZ77 matches
  StripTables& T = *reinterpret_cast<StripTables*>(sm + g.off_tab);
  png_mark(g, 0);

  // ---- 1. raw rows into smem (rows before the image are zero)
  const uint8_t* src = rgb + (size_t)img * g.H * rb;
  const int nraw = rows + 2;
  if ((rb & 15) == 0) {
    const int per = rb / 16;
    for (int i = t; i < nraw * per; i += kT) {
      const int r = i / per, c = i - r * per, y = y0 - 2 + r;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (y >= 0) v = __ldg(reinterpret_cast<const uint4*>(src + (size_t)y * rb) + c);
      reinterpret_cast<uint4*>(raw + r * rb)[c] = v;
    }
  } else {
    for (int i = t; i < nraw * rb; i += kT) {
      const int r = i / rb, c = i - r * rb, y = y0 - 2 + r;
      raw[i] = y >= 0 ? src[(size_t)y * rb + c] : (uint8_t)0;
    }
  }
  for (int i = t; i < 286 + 30; i += kT) T.lfreq[i] = 0;
  if (t < 19) T.cfreq[t] = 0;
  if (t < 32) { T.cnt[t >> 4][t & 15] = 0; }
  __syncthreads();

  // ---- 2. filter rows y0-1 (history, when it exists) .. y0+rows-1
  png_mark(g, 1);
  if ((rb & 3) == 0) {
    // one warp per row, no block barriers: 32-bit shared loads, lane l takes words l, l+32, ...;
    // the word before (for the left / up-left neighbours, 3 bytes back) comes from lane l-1
    const int lane = t & 31, nwords = rb >> 2;
    for (int fr = (y0 > 0 ? 0 : 1) + (t >> 5); fr <= rows; fr += kT / 32) {
      const uint32_t* c32 = reinterpret_cast<const uint32_t*>(raw + (fr + 1) * rb);
      const uint32_t* u32 = reinterpret_cast<const uint32_t*>(raw + fr * rb);
      auto pass = [&](int mode, uint8_t* out) -> void {  // mode < 0: sums; else write filter `mode`
        uint32_t cc = 0, uc = 0;  // lane 31's words of the previous round
        uint32_t sum[5] = {0, 0, 0, 0, 0};
        for (int base = 0; base < nwords; base += 32) {
          const int w = base + lane;
          const uint32_t cw = w < nwords ? c32[w] : 0u, uw = w < nwords ? u32[w] : 0u;
          uint32_t cp = __shfl_up_sync(0xffffffffu, cw, 1), upw = __shfl_up_sync(0xffffffffu, uw, 1);
          if (lane == 0) { cp = cc; upw = uc; }
          cc = __shfl_sync(0xffffffffu, cw, 31);
          uc = __shfl_sync(0xffffffffu, uw, 31);
          if (w < nwords) {
            const uint64_t cwin = (uint64_t)cw << 32 | cp, uwin = (uint64_t)uw << 32 | upw;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int x = (int)((cw >> (8 * j)) & 255u), a = (int)((cwin >> (8 * j + 8)) & 255u);
              const int b = (int)((uw >> (8 * j)) & 255u), c = (int)((uwin >> (8 * j + 8)) & 255u);
              if (mode < 0) {
#pragma unroll
                for (int k = 0; k < 5; ++k) sum[k] += (uint32_t)abs((int)(int8_t)filt_byte(k, x, a, b, c));
              } else {
                out[1 + 4 * w + j] = filt_byte(mode, x, a, b, c);
              }
            }
          }
        }
        if (mode < 0) {
          int best = 0;
          uint32_t bsum = 0xffffffffu;
#pragma unroll
          for (int k = 0; k < 5; ++k) {
            uint32_t v = sum[k];
#pragma unroll
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (v < bsum) { bsum = v; best = k; }  // ties: the lower filter type
          }
          out[0] = (uint8_t)best;  // every lane holds the same choice
        }
      };
      uint8_t* out = filt + fr * RS;
      uint8_t choice[1];
      pass(-1, choice);
      if (lane == 0) out[0] = choice[0];
      pass(choice[0], out);
    }
  } else
  for (int fr = (y0 > 0 ? 0 : 1); fr <= rows; ++fr) {
    const uint8_t* cur = raw + (fr + 1) * rb;  // image row y0-1+fr
    const uint8_t* up = raw + fr * rb;         // zeros above row 0
    uint32_t sum[5] = {0, 0, 0, 0, 0};
    for (int i = t; i < rb; i += kT) {
      const int x = cur[i], a = i >= 3 ? cur[i - 3] : 0, b = up[i], c = i >= 3 ? up[i - 3] : 0;
#pragma unroll
      for (int k = 0; k < 5; ++k) sum[k] += (uint32_t)abs((int)(int8_t)filt_byte(k, x, a, b, c));
    }
    const int lane = t & 31, wid = t >> 5;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
#pragma unroll
      for (int o = 16; o; o >>= 1) sum[k] += __shfl_xor_sync(0xffffffffu, sum[k], o);
    }
    __syncthreads();
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < 5; ++k) T.fsum[k][wid] = sum[k];
    }
    __syncthreads();
    int best = 0;
    uint32_t bsum = 0xffffffffu;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      uint32_t tot = 0;
      for (int w = 0; w < kT / 32; ++w) tot += T.fsum[k][w];
      if (tot < bsum) { bsum = tot; best = k; }  // ties: the lower filter type
    }
    uint8_t* out = filt + fr * RS;
    if (t == 0) out[0] = (uint8_t)best;
    for (int i = t; i < rb; i += kT) {
      const int x = cur[i], a = i >= 3 ? cur[i - 3] : 0, b = up[i], c = i >= 3 ? up[i - 3] : 0;
      out[1 + i] = filt_byte(best, x, a, b, c);
    }
  }
  __syncthreads();
  const uint8_t* f = filt + RS;  // the strip's bytes; f[-RS..-1] is the previous row when y0 > 0

  // ---- 3. Adler-32 partials: a = sum x_j, b = sum (S - j) x_j
  png_mark(g, 2);
  {
    unsigned long long a = 0, b = 0;
    for (int j = t; j < S; j += kT) {
      a += f[j];
      b += (unsigned long long)(S - j) * f[j];
    }
    const int lane = t & 31, wid = t >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if (lane == 0) { T.ab[0][wid] = a; T.ab[1][wid] = b; }
  }

  // ---- 4. LZ77 parse: thread t > 0 owns [(t-1)*G, t*G) of the strip, greedy, matches end inside it and
  // at most MC per segment.  The bytes 1..6 before p sit in a register window, so a literal costs
  // two shared loads (f[p], f[p - RS]); only a first-byte hit runs the extension loop.
  const int lo = y0 > 0 ? -RS : 0;
  // (thread 0 has no segment: it builds the block header while the others count their bits)
  const int p0 = t ? min((t - 1) * g.G, S) : S, p1 = t ? min(p0 + g.G, S) : S;
  uint32_t* ml = mlist + t * g.MC;
  {
    auto window = [&](int p) -> uint64_t {
      uint64_t w = 0;
#pragma unroll
      for (int k = 1; k <= 6; ++k)
        if (p - k >= lo) w |= (uint64_t)f[p - k] << (8 * (k - 1));
      return w;
    };
    int nm = 0;
    uint64_t back = window(p0);
    // f[p] and f[p - RS] of the next position are loaded one step ahead (the common step is a
    // literal), so the shared-memory latency overlaps the current step's work
    auto up_at = [&](int p) -> int { return p - RS >= lo ? (int)f[p - RS] : -1; };
    int x = p0 < p1 ? (int)f[p0] : 0, u = p0 < p1 ? up_at(p0) : -1;
    for (int p = p0; p < p1;) {
      const int xn = p + 1 < p1 ? (int)f[p + 1] : 0, un = p + 1 < p1 ? up_at(p + 1) : -1;
      const int maxl = min(258, p1 - p);
      int bl = 0, bd = 0;
      if (maxl >= 3 && nm < g.MC) {
#pragma unroll
        for (int di = 0; di < 4; ++di) {
          const int d = di < 3 ? short_dist(di) : RS;
          if (p - d < lo) continue;
          const int y = di < 3 ? (int)((back >> (8 * (d - 1))) & 255u) : u;
          if (y != x) continue;
          int l = 1;
          while (l < maxl && f[p + l] == f[p + l - d]) ++l;
          if (l > bl) { bl = l; bd = di; }
        }
      }
      if (bl >= 3) {
        ml[nm++] = (uint32_t)(p - p0) << 16 | (uint32_t)bd << 8 | (uint32_t)(bl - 3);
        int c, nb, ev;
        len_sym(bl, c, nb, ev);
        atomicAdd(&T.lfreq[c], 1u);
        dist_sym(bd < 3 ? short_dist(bd) : RS, c, nb, ev);
        atomicAdd(&T.lfreq[286 + c], 1u);
        p += bl;
        back = window(p);
        if (p < p1) { x = f[p]; u = up_at(p); }
      } else {
        atomicAdd(&T.lfreq[x], 1u);
        back = ((back << 8) | (uint64_t)x) & 0xFFFFFFFFFFFFull;
        ++p;
        x = xn;
        u = un;
      }
    }
    T.nmatch[t] = (uint8_t)nm;
  }
  __syncthreads();
  if (t == 0) T.lfreq[256] = 1;  // end of block
  __syncthreads();

  // ---- 5. sort the used symbols by (freq, symbol): one bitonic sort of 512 keys, literal/length
  // keys first, then distance keys, unused last
  png_mark(g, 3);
  uint32_t ml_cnt = 0, md_cnt = 0;
  for (int i = t; i < 512; i += kT) {
    uint32_t key = 0xFFFFFFFFu;
    if (i < 316) {
      T.llen[i] = 0;
      const uint32_t fs = T.lfreq[i];
      if (fs) {
        key = i < 286 ? (fs << 9 | (uint32_t)i) : (1u << 31 | fs << 5 | (uint32_t)(i - 286));
        if (i < 286) ++ml_cnt; else ++md_cnt;
      }
    }
    hw.keys[i] = key;
  }
  if (t < 2) { T.scal[1 + t] = t ? 1u : 257u; }  // hlit / hdist minima (raised by atomicMax below)
  const int m_l = (int)block_sum_u32(ml_cnt, T.red);
  const int m_d = (int)block_sum_u32(md_cnt, T.red);
  for (int k = 2; k <= 512; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1)), ixj = i | j;
      const uint32_t x = hw.keys[i], y = hw.keys[ixj];
      if ((x > y) == ((i & k) == 0)) { hw.keys[i] = y; hw.keys[ixj] = x; }
      __syncthreads();
    }
  }
  for (int r = t; r < m_l + m_d; r += kT) {
    const uint32_t key = hw.keys[r];
    if (r < m_l) {
      T.order[r] = (uint16_t)(key & 511u);
      hw.lit.wl[r] = key >> 9;
    } else {
      T.order[286 + r - m_l] = (uint16_t)(key & 31u);
      hw.dst.wl[r - m_l] = (key >> 5) & 0x3FFFFFFu;
    }
  }
  __syncthreads();

  // ---- 6. code lengths and codes
  png_mark(g, 4);
  if (t == 0 && m_l >= 2) huff_merge(hw.lit.wl, hw.lit.wi, hw.lit.pl, hw.lit.pi, hw.lit.di, m_l);
  if (t == 32 && m_d >= 2) huff_merge(hw.dst.wl, hw.dst.wi, hw.dst.pl, hw.dst.pi, hw.dst.di, m_d);
  __syncthreads();
  for (int r = t; r < m_l; r += kT) {
    const int d = hw.lit.di[hw.lit.pl[r]] + 1;
    atomicAdd(&T.cnt[0][d > 15 ? 15 : d], 1u);
  }
  if (t < m_d && m_d >= 2) {
    const int d = hw.dst.di[hw.dst.pl[t]] + 1;
    atomicAdd(&T.cnt[1][d > 15 ? 15 : d], 1u);
  }
  for (int i = t; i < 320; i += kT) hw.ccnt[i >> 5][i & 31] = 0;
  __syncthreads();
  if (t == 0 || t == 32) {
    const int k = t ? 1 : 0, m = k ? m_d : m_l;
    if (m < 2) {  // dummy second code (only the distance alphabet can get here)
      const int a = m == 1 ? T.order[286 * k] : 0;
      T.llen[286 * k + a] = 1;
      T.llen[286 * k + (a == 0 ? 1 : 0)] = 1;
      T.cnt[k][1] = 2;
    }
    huff_repair(T.cnt[k], T.next[k], 15);
  }
  __syncthreads();
  // lengths by rank: the least frequent symbols take the longest lengths
  for (int i = t; i < 316; i += kT) {
    const int k = i < 286 ? 0 : 1, r = i - 286 * k, m = k ? m_d : m_l;
    if (m < 2 || r >= m) continue;
    uint32_t acc = 0;
    for (int len = 15; len >= 1; --len) {
      acc += T.cnt[k][len];
      if ((uint32_t)r < acc) { T.llen[286 * k + T.order[286 * k + r]] = (uint8_t)len; break; }
    }
  }
  __syncthreads();
  // canonical codes: next[len] + the number of lower symbols of the same alphabet and length,
  // counted per 32-symbol chunk (shared counters, then a prefix over chunks) and within the chunk
  // by a warp match
  for (int i = t; i < 316; i += kT) {
    const int len = T.llen[i];
    if (len) atomicAdd(&hw.ccnt[i >> 5][(i >= 286) * 16 + len], 1u);
  }
  __syncthreads();
  if (t < 32) {
    uint32_t acc = 0;
    for (int c = 0; c < 10; ++c) { const uint32_t v = hw.ccnt[c][t]; hw.ccnt[c][t] = acc; acc += v; }
  }
  // hlit / hdist: one past the last used symbol of each alphabet
  for (int i = t; i < 316; i += kT)
    if (T.llen[i]) atomicMax(&T.scal[i < 286 ? 1 : 2], (uint32_t)(i < 286 ? i + 1 : i - 285));
  __syncthreads();
  {
    const int lane = t & 31;
    for (int i0 = t & ~31; i0 < 316; i0 += kT) {  // warp-uniform
      const int i = i0 + lane;
      const int len = i < 316 ? T.llen[i] : 0, k = i >= 286;
      const int key = len ? k * 16 + len : 255;
      const unsigned grp = __match_any_sync(0xffffffffu, key);
      if (i < 316) {
        uint16_t code = 0;
        if (len)
          code = (uint16_t)rev_bits(T.next[k][len] + hw.ccnt[i >> 5][key] + __popc(grp & ((1u << lane) - 1u)), len);
        T.lcode[i] = code;
      }
    }
  }
  __syncthreads();

  // ---- 7. token bits; the block header: parallel run-length coding of the code lengths, their
  // code (thread 0), bit offsets by block scans; dynamic vs stored
  int dcs[4], dns[4], dvs[4];
#pragma unroll
  for (int di = 0; di < 4; ++di) dist_sym(di < 3 ? short_dist(di) : RS, dcs[di], dns[di], dvs[di]);
  const int nm = T.nmatch[t];
  uint32_t mybits = 0;
  png_mark(g, 5);
  {
    int mi = 0, mp = nm ? (int)(ml[0] >> 16) + p0 : p1;
    for (int p = p0; p < p1;) {
      if (p == mp) {
        const uint32_t v = ml[mi];
        const int len = (int)(v & 255) + 3, di = (int)(v >> 8) & 3;
        int c, nb, ev;
        len_sym(len, c, nb, ev);
        mybits += T.llen[c] + nb + T.llen[286 + dcs[di]] + dns[di];
        p += len;
        ++mi;
        mp = mi < nm ? (int)(ml[mi] >> 16) + p0 : p1;
      } else {
        mybits += T.llen[f[p]];
        ++p;
      }
    }
  }
  const int hlit = (int)T.scal[1], hdist = (int)T.scal[2], nl = hlit + hdist;
  auto seq = [&](int i) -> int { return i < hlit ? T.llen[i] : T.llen[286 + i - hlit]; };
  int rv[2] = {0, 0}, rn[2] = {0, 0}, rc[2] = {0, 0};
#pragma unroll
  for (int q = 0; q < 2; ++q) {  // runs starting at 2t, 2t+1 (index order, for the scan)
    const int i = 2 * t + q;
    if (i < nl) {
      const int v = seq(i);
      if (i == 0 || seq(i - 1) != v) {
        int run = 1;
        while (i + run < nl && seq(i + run) == v) ++run;
        rv[q] = v; rn[q] = run; rc[q] = rle_run(v, run, nullptr);
      }
    }
  }
  uint32_t nr_tot;
  const uint32_t roff = block_scan_u32((uint32_t)(rc[0] + rc[1]), T.red, &nr_tot);
#pragma unroll
  for (int q = 0; q < 2; ++q)
    if (rc[q]) {
      uint16_t* o = T.rle + roff + (q ? rc[0] : 0);
      rle_run(rv[q], rn[q], o);
      for (int k = 0; k < rc[q]; ++k) atomicAdd(&T.cfreq[o[k] & 31], 1u);
    }
  __syncthreads();
  if (t == 0) {  // the code-length code: 19 symbols, one thread
    int mc = 0;
    for (int sym = 0; sym < 19; ++sym)  // insertion sort of the used code-length symbols
      if (T.cfreq[sym]) {
        int j = mc++;
        while (j > 0 && (T.cfreq[T.corder[j - 1]] > T.cfreq[sym])) { T.corder[j] = T.corder[j - 1]; --j; }
        T.corder[j] = (uint16_t)sym;
      }
    huff_small(T.cfreq, 19, T.corder, mc, 7, T.clen, T.ccode);
    const uint8_t kOrd[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};
    int hclen = 19;
    while (hclen > 4 && !T.clen[kOrd[hclen - 1]]) --hclen;
    T.scal[3] = (uint32_t)hclen;
    T.scal[0] = nr_tot;
  }
  __syncthreads();
  uint32_t rb2[2] = {0, 0};
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int i = 2 * t + q;
    if (i < (int)nr_tot) {
      const int sym = T.rle[i] & 31;
      rb2[q] = T.clen[sym] + (sym == 16 ? 2 : sym == 17 ? 3 : sym == 18 ? 7 : 0);
    }
  }
  uint32_t rle_bits;
  const uint32_t rboff = block_scan_u32(rb2[0] + rb2[1], T.red, &rle_bits);
  if (2 * t < (int)nr_tot) T.rle_off[2 * t] = (uint16_t)rboff;
  if (2 * t + 1 < (int)nr_tot) T.rle_off[2 * t + 1] = (uint16_t)(rboff + rb2[0]);
  const uint32_t hfix = 3 + 5 + 5 + 4 + 3 * T.scal[3];  // BFINAL, BTYPE, HLIT, HDIST, HCLEN, lengths
  uint32_t tbits;
  const uint32_t myoff = block_scan_u32(mybits, T.red, &tbits);
  png_mark(g, 6);
  const uint32_t pre = first ? 16u : 0u;  // zlib header
  const uint32_t hdr_bits = hfix + rle_bits;
  const uint32_t dyn_end = pre + hdr_bits + tbits + T.llen[256];  // bit after the end-of-block code
  const uint32_t dyn_bytes = (last ? (dyn_end + 7) / 8 : (dyn_end + 3 + 7) / 8 + 4) + (last ? 4 : 0);
  const uint32_t sto_bytes = pre / 8 + 5 + (uint32_t)S + (last ? 4 : 0);
  const bool dyn = dyn_bytes < sto_bytes;
  const uint32_t bytes = dyn ? dyn_bytes : sto_bytes;
  const int nw = (int)(bytes + 3) / 4 + 1;
  for (int i = t; i < nw; i += kT) ow[i] = 0;  // the Huffman work arrays are dead
  __syncthreads();

  // ---- 8. write
  if (dyn) {
    if (t == 0) {  // fixed part of the header
      BitW w(ow, 0);
      if (first) { w.put(0x78, 8); w.put(0x5E, 8); }
      w.put(last ? 1u : 0u, 1);
      w.put(2, 2);
      w.put((uint32_t)hlit - 257, 5);
      w.put((uint32_t)hdist - 1, 5);
      w.put(T.scal[3] - 4, 4);
      const uint8_t kOrd[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};
      for (int i = 0; i < (int)T.scal[3]; ++i) w.put(T.clen[kOrd[i]], 3);
      w.flush();
    }
    for (int i = t; i < (int)nr_tot; i += kT) {  // run-length coded code lengths, one token each
      BitW w(ow, pre + hfix + T.rle_off[i]);
      const int sym = T.rle[i] & 31, ex = T.rle[i] >> 5;
      w.put(T.ccode[sym], T.clen[sym]);
      if (sym == 16) w.put(ex, 2);
      else if (sym == 17) w.put(ex, 3);
      else if (sym == 18) w.put(ex, 7);
      w.flush();
    }
    {
      BitW w(ow, pre + hdr_bits + myoff);
      int mi = 0, mp = nm ? (int)(ml[0] >> 16) + p0 : p1;
      for (int p = p0; p < p1;) {
        if (p == mp) {
          const uint32_t v = ml[mi];
          const int len = (int)(v & 255) + 3, di = (int)(v >> 8) & 3;
          int c, nb, ev;
          len_sym(len, c, nb, ev);
          w.put(T.lcode[c], T.llen[c]);
          if (nb) w.put((uint32_t)ev, nb);
          w.put(T.lcode[286 + dcs[di]], T.llen[286 + dcs[di]]);
          if (dns[di]) w.put((uint32_t)dvs[di], dns[di]);
          p += len;
          ++mi;
          mp = mi < nm ? (int)(ml[mi] >> 16) + p0 : p1;
        } else {
          const int x = f[p];
          w.put(T.lcode[x], T.llen[x]);
          ++p;
        }
      }
      w.flush();
    }
    __syncthreads();
    if (t == 0) {
      BitW w(ow, dyn_end - T.llen[256]);
      w.put(T.lcode[256], T.llen[256]);
      if (!last) w.put(0, 3);  // empty stored block: BFINAL 0, BTYPE 00, then pad + 00 00 FF FF
      w.flush();
      if (!last) {
        uint8_t* ob = reinterpret_cast<uint8_t*>(ow);
        const uint32_t e = (dyn_end + 3 + 7) / 8;
        ob[e] = 0; ob[e + 1] = 0; ob[e + 2] = 0xFF; ob[e + 3] = 0xFF;
      }
    }
  } else {
    uint8_t* ob = reinterpret_cast<uint8_t*>(ow);
    const int h = (int)pre / 8;
    if (t == 0) {
      if (first) { ob[0] = 0x78; ob[1] = 0x5E; }
      ob[h] = last ? 1 : 0;  // BFINAL, BTYPE 00, padding
      ob[h + 1] = (uint8_t)(S & 255); ob[h + 2] = (uint8_t)(S >> 8);
      ob[h + 3] = (uint8_t)(~S & 255); ob[h + 4] = (uint8_t)((~S >> 8) & 255);
    }
    __syncthreads();
    for (int j = t; j < S; j += kT) ob[h + 5 + j] = f[j];
  }
  __syncthreads();

  // ---- 9. out to the strip's scratch slot; meta
  png_mark(g, 7);
  uint8_t* dst = scratch + (size_t)blockIdx.x * g.cap;
  const int nvec = ((int)bytes + 15) / 16;
  for (int i = t; i < nvec; i += kT) reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(ow)[i];
  if (t == 0) {
    unsigned long long a = 0, b = 0;
    for (int w = 0; w < kT / 32; ++w) { a += T.ab[0][w]; b += T.ab[1][w]; }
    StripMeta m;
    m.bytes = bytes;
    m.a = (uint32_t)(a % kAdler);
    m.b = (uint32_t)(b % kAdler);
    m.rsv = dyn ? 1u : 0u;
    meta[blockIdx.x] = m;
  }
  png_mark(g, 8);
}

// --------------------------------------------------------------------------- CRC-32
__device__ __forceinline__ uint32_t crc_mulmod(uint32_t a, uint32_t b) {  // a*b mod P, reflected
  if (!a) return 0;
  uint32_t m = 1u << 31, p = 0;
  for (;;) {
    if (a & m) {
      p ^= b;
      if (!(a & (m - 1))) break;
    }
    m >>= 1;
    b = (b & 1) ? (b >> 1) ^ kCrcPoly : b >> 1;
  }
  return p;
}
__device__ uint32_t crc_x8n(unsigned long long n) {  // x^(8n) mod P
  uint32_t r = 1u << 31, base = 1u << 23;             // x^0, x^8
  while (n) {
    if (n & 1) r = crc_mulmod(base, r);
    base = crc_mulmod(base, base);
    n >>= 1;
  }
  return r;
}
__device__ __forceinline__ void crc_table(uint32_t* tab) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t c = (uint32_t)i;
    for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ kCrcPoly : c >> 1;
    tab[i] = c;
  }
}
__device__ __forceinline__ uint32_t crc_raw(const uint32_t* tab, uint32_t c, const uint8_t* p, int n) {
  for (int i = 0; i < n; ++i) c = (c >> 8) ^ tab[(c ^ p[i]) & 255];
  return c;
}

__device__ __forceinline__ void put_be32(uint8_t* p, uint32_t v) {
  p[0] = (uint8_t)(v >> 24); p[1] = (uint8_t)(v >> 16); p[2] = (uint8_t)(v >> 8); p[3] = (uint8_t)v;
}

// --------------------------------------------------------------------------- K-b: per image
__global__ void __launch_bounds__(kT) png_image_kernel(PngGeom g, uint8_t* __restrict__ scratch,
                                                       const StripMeta* __restrict__ meta, uint32_t* __restrict__ offs,
                                                       uint32_t* __restrict__ sizes) {
  __shared__ uint32_t red[kT / 32];
  __shared__ unsigned long long ared[2][kT / 32];
  const int img = blockIdx.x, t = threadIdx.x, ns = g.nstrips;
  const StripMeta* mi = meta + (size_t)img * ns;
  const unsigned long long N = (unsigned long long)g.H * g.RS;
  // Adler-32 of the whole filtered stream: A = 1 + sum a_s, B = N + sum (b_s + (N - o_s - S_s) a_s)
  unsigned long long A = 0, B = 0;
  const int per = (ns + kT - 1) / kT, s0 = t * per;
  uint32_t mine = 0;
  for (int s = s0; s < s0 + per && s < ns; ++s) {
    const unsigned long long o = (unsigned long long)s * g.R * g.RS, Ss = (unsigned long long)strip_rows(g, s) * g.RS;
    A += mi[s].a;
    B += mi[s].b + ((N - o - Ss) % kAdler) * mi[s].a % kAdler;
    mine += 12u + mi[s].bytes;
  }
  {
    const int lane = t & 31, wid = t >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      A += __shfl_xor_sync(0xffffffffu, A, o);
      B += __shfl_xor_sync(0xffffffffu, B, o);
    }
    if (lane == 0) { ared[0][wid] = A; ared[1][wid] = B; }
  }
  uint32_t total;
  uint32_t off = 33u + block_scan_u32(mine, red, &total);  // after signature + IHDR
  for (int s = s0; s < s0 + per && s < ns; ++s) {
    offs[(size_t)img * ns + s] = off;
    off += 12u + mi[s].bytes;
  }
  if (t == 0) {
    unsigned long long a = 1, b = N % kAdler;
    for (int w = 0; w < kT / 32; ++w) { a += ared[0][w]; b += ared[1][w]; }
    const uint32_t adler = (uint32_t)((b % kAdler) << 16 | (a % kAdler));
    put_be32(scratch + ((size_t)img * ns + ns - 1) * g.cap + mi[ns - 1].bytes - 4, adler);
    sizes[img] = 33u + total + 12u;
  }
}

// --------------------------------------------------------------------------- K-b2: image bases, frames
// base[i] = i * stride, or (contiguous) the exclusive scan of the sizes; then the signature, IHDR
// and IEND of every image
__global__ void __launch_bounds__(kT) png_frame_kernel(PngGeom g, const uint32_t* __restrict__ sizes,
                                                       unsigned long long* __restrict__ bases, uint8_t* __restrict__ out,
                                                       long long stride, int contiguous) {
  __shared__ uint32_t tab[256];
  __shared__ unsigned long long part[kT];
  crc_table(tab);
  const int t = threadIdx.x, n = g.n;
  const int per = (n + kT - 1) / kT, i0 = t * per;
  unsigned long long sum = 0;
  for (int i = i0; i < i0 + per && i < n; ++i) sum += sizes[i];
  part[t] = sum;
  __syncthreads();
  if (t == 0) {  // n / kT partial sums: a serial scan is plenty
    unsigned long long acc = 0;
    for (int k = 0; k < kT; ++k) { const unsigned long long v = part[k]; part[k] = acc; acc += v; }
  }
  __syncthreads();
  unsigned long long base = part[t];
  for (int i = i0; i < i0 + per && i < n; ++i) {
    const unsigned long long b = contiguous ? base : (unsigned long long)i * (unsigned long long)stride;
    base += sizes[i];
    bases[i] = b;
    uint8_t* o = out + b;
    const uint8_t sig[8] = {0x89, 'P', 'N', 'G', 0x0D, 0x0A, 0x1A, 0x0A};
    for (int k = 0; k < 8; ++k) o[k] = sig[k];
    uint8_t ih[17] = {'I', 'H', 'D', 'R'};
    put_be32(ih + 4, (uint32_t)g.W);
    put_be32(ih + 8, (uint32_t)g.H);
    ih[12] = 8; ih[13] = 2; ih[14] = 0; ih[15] = 0; ih[16] = 0;  // 8-bit RGB, deflate, adaptive, no interlace
    put_be32(o + 8, 13);
    for (int k = 0; k < 17; ++k) o[12 + k] = ih[k];
    put_be32(o + 29, ~crc_raw(tab, 0xFFFFFFFFu, ih, 17));
    const uint8_t iend[12] = {0, 0, 0, 0, 'I', 'E', 'N', 'D', 0xAE, 0x42, 0x60, 0x82};
    uint8_t* e = o + sizes[i] - 12;
    for (int k = 0; k < 12; ++k) e[k] = iend[k];
  }
}

// --------------------------------------------------------------------------- K-c: per strip
__global__ void __launch_bounds__(kT) png_chunk_kernel(PngGeom g, const uint8_t* __restrict__ scratch,
                                                       const StripMeta* __restrict__ meta,
                                                       const uint32_t* __restrict__ offs,
                                                       const unsigned long long* __restrict__ bases,
                                                       uint8_t* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ uint32_t tab[256];
  __shared__ uint32_t xr[kT / 32];
  crc_table(tab);
  const int t = threadIdx.x, img = blockIdx.x / g.nstrips;
  const uint32_t d = meta[blockIdx.x].bytes, L = d + 4;  // CRC covers "IDAT" + data
  uint8_t* buf = sm;                                      // "IDAT" at 12..15, data from 16
  const uint8_t* src = scratch + (size_t)blockIdx.x * g.cap;
  for (int i = t; i < (int)(d + 15) / 16; i += kT)
    reinterpret_cast<uint4*>(buf + 16)[i] = reinterpret_cast<const uint4*>(src)[i];
  if (t == 0) { buf[12] = 'I'; buf[13] = 'D'; buf[14] = 'A'; buf[15] = 'T'; }
  __syncthreads();
  const uint8_t* c0 = buf + 12;
  const uint32_t seg = (L + kT - 1) / kT, b0 = min(L, t * seg), b1 = min(L, b0 + seg);
  uint32_t c = crc_raw(tab, 0u, c0 + b0, (int)(b1 - b0));
  c = crc_mulmod(crc_x8n(L - b1), c);  // shift past the bytes after this segment
  if (t == 0) c ^= crc_mulmod(crc_x8n(L), 0xFFFFFFFFu);
#pragma unroll
  for (int o = 16; o; o >>= 1) c ^= __shfl_xor_sync(0xffffffffu, c, o);
  if ((t & 31) == 0) xr[t >> 5] = c;
  __syncthreads();
  uint8_t* o = out + bases[img] + offs[blockIdx.x];
  for (uint32_t i = t; i < L; i += kT) o[4 + i] = c0[i];
  if (t == 0) {
    uint32_t x = 0;
    for (int w = 0; w < kT / 32; ++w) x ^= xr[w];
    put_be32(o, d);
    put_be32(o + 8 + d, ~x);
  }
}

PngGeom png_geom(int n, int H, int W) {
  PngGeom g{};
  g.n = n; g.H = H; g.W = W;
  g.RS = 3 * W + 1;
  g.MC = 16;
  // rows per strip: at most 8, at most 32 KB of filtered bytes, and shared memory for three CTAs
  // per SM where the width allows
  int R = kMaxStripBytes / g.RS;
  if (R > 8) R = 8;
  if (R < 1) R = 1;
  for (;; --R) {
    const int S = R * g.RS;
    g.R = R;
    g.G = (S + kT - 2) / (kT - 1);
    const int raw = ((R + 2) * 3 * W + 15) & ~15, ow = ((S + 48) & ~15) + 16;
    int r0 = raw > ow ? raw : ow;
    if (r0 < (int)sizeof(HuffWork)) r0 = ((int)sizeof(HuffWork) + 15) & ~15;
    g.off_filt = r0;
    g.off_ml = g.off_filt + (((R + 1) * g.RS + 15) & ~15);
    g.off_tab = g.off_ml + kT * g.MC * 4;
    g.smem = g.off_tab + (int)((sizeof(StripTables) + 15) & ~size_t(15));
    if (R == 1 || g.smem <= 74 * 1024) break;
  }
  g.nstrips = (H + g.R - 1) / g.R;
  g.cap = ((g.R * g.RS + 16 + 15) & ~15) + 16;
  return g;
}

}  // namespace

size_t png_bound(int H, int W) {
  if (H <= 0 || W <= 0) return 0;
  const PngGeom g = png_geom(1, H, W);
  return 45 + (size_t)g.nstrips * (12 + (size_t)g.cap);
}

size_t png_workspace(int n, int H, int W) {
  const PngGeom g = png_geom(n, H, W);
  const size_t ns = (size_t)n * g.nstrips;
  return ns * g.cap + ns * sizeof(StripMeta) + ns * 4 + 8 * (size_t)n + 256;
}

cudaError_t launch_png_encode(const uint8_t* rgb, int n, int H, int W, uint8_t* out, long long stride,
                              uint32_t* sizes, uint8_t* work, cudaStream_t s, bool contiguous) {
  if (n <= 0 || H <= 0 || W <= 0 || W > 8192 || H > 65535 || (!contiguous && (size_t)stride < png_bound(H, W)))
    return cudaErrorInvalidValue;
  const PngGeom g = png_geom(n, H, W);
  if (!ensure_smem_attr(reinterpret_cast<const void*>(png_strip_kernel), g.smem) ||
      !ensure_smem_attr(reinterpret_cast<const void*>(png_chunk_kernel), g.cap + 32))
    return cudaErrorNotSupported;
  const size_t ns = (size_t)n * g.nstrips;
  uint8_t* scratch = work;
  StripMeta* meta = reinterpret_cast<StripMeta*>(work + ns * g.cap);
  uint32_t* offs = reinterpret_cast<uint32_t*>(meta + ns);
  unsigned long long* bases =
      reinterpret_cast<unsigned long long*>((reinterpret_cast<uintptr_t>(offs + ns) + 7) & ~uintptr_t(7));
  static const bool timing = getenv("LBX_PNG_TIMING") != nullptr;
  PngGeom gt = g;
  if (timing) cudaMallocAsync(reinterpret_cast<void**>(&gt.tl), ns * 16 * 8, s);
  png_strip_kernel<<<(unsigned)ns, kT, g.smem, s>>>(rgb, gt, scratch, meta);
  if (timing) {  // per-phase mean durations over the strips, and the kernel's span
    std::vector<unsigned long long> h(ns * 16);
    cudaMemcpyAsync(h.data(), gt.tl, h.size() * 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    cudaFreeAsync(gt.tl, s);
    double ph[8] = {0};
    unsigned long long lo = ~0ull, hi = 0;
    for (size_t b = 0; b < ns; ++b) {
      for (int i = 0; i < 8; ++i) ph[i] += (double)(h[b * 16 + i + 1] - h[b * 16 + i]);
      lo = std::min(lo, h[b * 16]);
      hi = std::max(hi, h[b * 16 + 8]);
    }
    const char* names[8] = {"load", "filter", "adler+parse", "rank sort", "huffman", "header||bits+scan", "write", "copy out"};
    fprintf(stderr, "png_strip timing: %zu strips, span %.3f ms; mean per strip (us):", ns, (hi - lo) * 1e-6);
    for (int i = 0; i < 8; ++i) fprintf(stderr, " %s %.1f", names[i], ph[i] / ns * 1e-3);
    fprintf(stderr, "\n");
  }
  png_image_kernel<<<n, kT, 0, s>>>(g, scratch, meta, offs, sizes);
  png_frame_kernel<<<1, kT, 0, s>>>(g, sizes, bases, out, stride, contiguous ? 1 : 0);
  png_chunk_kernel<<<(unsigned)ns, kT, g.cap + 32, s>>>(g, scratch, meta, offs, bases, out);
  return cudaGetLastError();
}

}  // namespace lbx
