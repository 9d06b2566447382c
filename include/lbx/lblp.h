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
 *   6      1     mode               0 raw | 1 lossless | 2 q8
 *   7      1     flags              = 0
 *   8      2     C
 *   10     2     H
 *   12     2     W
 *   14     2     reserved           = 0
 *   16     4     total_bytes        size of the whole blob
 *   20     4     table_offset       mode 1: row table; mode 2: channel params; mode 0: 0
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
 */
#ifndef LBX_LBLP_H
#define LBX_LBLP_H

#include <stdint.h>

#define LBLP_MAGIC "LBLP"
#define LBLP_VERSION 1
#define LBLP_DTYPE_F16 1
#define LBLP_HEADER_BYTES 32

enum lblp_mode { LBLP_RAW = 0, LBLP_LOSSLESS = 1, LBLP_Q8 = 2 };

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
