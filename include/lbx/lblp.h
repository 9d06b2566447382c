/*
 * LBLP v1 -- LatentBox latent pack format (normative definition).
 *
 * The reference has no latent codec: the paper stores latents with pcodec, a Rust crate that is
 * not vendored and has no pinned version and decompresses them on CPU
 * (PAPER.md:669); the simulator only carries a byte count, ObjectMeta::latent_bytes
 * (proj/include/latentbox/trace.hpp:21-26).  LBLP is therefore self-defined
 * and laid out for one-warp-per-row GPU decode.  Bit-exactness is pinned by two independent
 * implementations (oracle/lblp_ref.c and paper_2605_19385_b200/csrc/codec.cpp + unpack.cu) and the
 * known-answer vectors in tests/golden/.
 *
 * All integers little-endian.  A blob is:
 *
 *   offset size  field
 *   0      4     magic "LBLP"
 *   4      1     version            = 1
 *   5      1     dtype              = 1 (IEEE fp16 latent values)
 *   6      1     mode               0 raw | 1 lossless | 2 q8 | 3 entropy (lossless)
 *   7      1     flags              = 0
 *   8      2     C
 *   10     2     H
 *   12     2     W
 *   14     2     reserved           = 0
 *   16     4     total_bytes        size of the whole blob
 *   20     4     table_offset       mode 1: row table; mode 2: channel params; mode 3: plane table;
 *                                      mode 0: 0
 *   24     4     payload_offset
 *   28     4     reserved           = 0
 *
 * mode 0 (raw):       payload = C*H*W fp16 bit patterns, NCHW.  payload_offset = 32.
 *
 * mode 1 (lossless):  rows r = c*H + y, each W values (W % 32 == 0).
 *   table_offset = 32: uint32 row_off[C*H], byte offset of row r relative to payload_offset,
 *   multiple of 4.  payload_offset = 32 + 4*C*H.
 *   Per value: v = omap(bits) with omap(u) = (u & 0x8000) ? (~u & 0xFFFF) : (u | 0x8000)
 *   (order-preserving), d[0] = 0, d[i] = (v[i] - v[i-1]) mod 2^16 read as int16,
 *   z = zigzag16(d) = ((d << 1) ^ (d >> 15)) & 0xFFFF.
 *   Row layout: uint16 bits0 (raw fp16 bits of value 0); uint8 width[W/32]; zero padding to a
 *   multiple of 4 bytes from the row start; then for each 32-value mini-block j, width[j]
 *   uint32 words holding the 32 values z[32j+k] at bit offset k*width[j], LSB-first across the
 *   word sequence.  width[j] = bit length of max_k z[32j+k] (0..16).
 *
 * mode 2 (q8):        lossy per-channel affine int8.
 *   table_offset = 32: float32 scale[C], then int32 zero_point[C].  payload_offset = 32 + 8*C.
 *   payload = int8 q[C*H*W] NCHW.  Decode (fixed operation order, no FMA contraction):
 *     x = fp16_rn( fp32_rn( (float)(q - zero_point[c]) * scale[c] ) )
 *
 * mode 3 (entropy, lossless): the algorithm class of pcodec -- values mapped to
 * order-preserving integers, optional delta, binned and entropy-coded, low bits raw -- laid out
 * for one-thread-per-column GPU decode.  NOT the pcodec wire format (no pco implementation or
 * spec exists in this build environment to pin one against).  W % 32 == 0, W <= 1024.
 *   table_offset = 32: uint32 plane_off[C], byte offset of plane c relative to payload_offset,
 *   multiple of 4.  payload_offset = 32 + 4*C.
 *   Plane (H rows x W columns of channel c), all offsets below relative to the plane start:
 *     0   uint8  delta   0: s = omap(bits); 1: s = zigzag16(omap(bits[y][x]) - omap(bits[y-1][x]))
 *                        (mod 2^16, row -1 reads as 0) -- differences down each column
 *     1   uint8  L       = 12 (rANS table size M = 2^L)
 *     2   uint8  b       raw low bits per value, 0..16
 *     3   uint8  0
 *     4   uint16 K       bins, 1..256
 *     6   uint16 0
 *     8   uint32 raw_pos start of the raw low bits (multiple of 4)
 *     12  uint32 0
 *     16  K x {uint16 hi, uint16 freq}: bin k holds the symbols [hi << b, (hi+1) << b); hi strictly
 *         increasing, hi < 2^(16-b); freq >= 1, sum = M; cum[k] = freq[0] + ... + freq[k-1].
 *     then (padded to 4) uint32 state[W]: each column's initial rANS decoder state, in [2^16, 2^32)
 *     then uint32 warp_off[W/32]: start of warp g's (columns 32g..32g+31) renormalisation words,
 *         multiple of 4; the words run to the next warp's start (the last: to raw_pos)
 *     then the word sequences (uint16), each padded to 4 bytes
 *     raw_pos: W x ceil(H*b/32) uint32, column x's words at x*ceil(H*b/32)*4: value y's low b bits at
 *         bit y*b, LSB-first across the words.
 *   Decode: for y = 0..H-1, for each warp g, for lanes l = 0..31 in order (column x = 32g + l):
 *     slot = st & (M-1); k = the bin with cum[k] <= slot < cum[k] + freq[k];
 *     st = freq[k] * (st >> L) + slot - cum[k];  if st < 2^16: st = (st << 16) | next word of warp g;
 *     s = (hi[k] << b) | low_bits(x, y);  v = delta ? v_prev(x) + unzigzag16(s) : s;  bits = omap^-1(v)
 *   The encoder (rANS over the column, symbols in reverse) tries delta 0 and 1 and keeps the shorter
 *   plane (ties: 0); b is the smallest value that leaves <= 256 occupied bins; freq = max(1,
 *   floor(count * M / (H*W))), then +1 (while the sum is short) or -1 (where > 1, while over) cycling
 *   through the bins in (count desc, hi asc) order.
 */
#ifndef LBX_LBLP_H
#define LBX_LBLP_H

#include <stdint.h>

#define LBLP_MAGIC "LBLP"
#define LBLP_VERSION 1
#define LBLP_DTYPE_F16 1
#define LBLP_HEADER_BYTES 32

enum lblp_mode { LBLP_RAW = 0, LBLP_LOSSLESS = 1, LBLP_Q8 = 2, LBLP_ENTROPY = 3 };

typedef struct lblp_header {
  char magic[4];
  uint8_t version;
  uint8_t dtype;
  uint8_t mode;
  uint8_t flags;
  uint16_t c, h, w;
  uint16_t reserved0;
  uint32_t total_bytes;
  uint32_t table_offset;
  uint32_t payload_offset;
  uint32_t reserved1;
} lblp_header;

#endif /* LBX_LBLP_H */
