// BLAKE2b (RFC 7693), unkeyed, for the canonical graph hash.
//
// The reference hashes with Python's hashlib.blake2b (graph.py:510-549):
// 16-byte node keys, 16-byte weight digests and an 8-byte graph digest.  This
// is the same function restated for the device so that every 64-bit hash the
// GPU search produces is bit-identical to the reference's.  The message is
// streamed into a 128-byte block held as 16 little-endian words; a block is
// compressed only when more input arrives (or at finalisation), which is what
// makes the last block carry the finalisation flag.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define EF_HD __host__ __device__ __forceinline__
#else
#define EF_HD inline
#endif

namespace ef {

#ifdef __CUDACC__
__constant__ uint64_t kB2bIV[8] = {
#else
static const uint64_t kB2bIV[8] = {
#endif
    0x6a09e667f3bcc908ULL, 0xbb67ae8584caa73bULL, 0x3c6ef372fe94f82bULL, 0xa54ff53a5f1d36f1ULL,
    0x510e527fade682d1ULL, 0x9b05688c2b3e6c1fULL, 0x1f83d9abfb41bd6bULL, 0x5be0cd19137e2179ULL};

EF_HD uint64_t b2b_iv(int i) {
  // literal copy usable from host and device without touching __constant__ on host
  switch (i) {
    case 0: return 0x6a09e667f3bcc908ULL;
    case 1: return 0xbb67ae8584caa73bULL;
    case 2: return 0x3c6ef372fe94f82bULL;
    case 3: return 0xa54ff53a5f1d36f1ULL;
    case 4: return 0x510e527fade682d1ULL;
    case 5: return 0x9b05688c2b3e6c1fULL;
    case 6: return 0x1f83d9abfb41bd6bULL;
    default: return 0x5be0cd19137e2179ULL;
  }
}

EF_HD uint64_t rotr64(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

// The four rotations of G on the device, spelled on the 32-bit halves: 32 is a register swap,
// 24 and 16 one PRMT per half, 63 one funnel shift per half.  The generic shift-or form costs
// ~4 more ALU-pipe instructions per G (2,254 vs 1,966 ALU instructions per compression) and
// measures 8.0 vs 9.4 G compressions/s on a B200 (the ALU pipe is the bound).
#ifdef __CUDA_ARCH__
__device__ __forceinline__ void b2b_split(uint64_t x, uint32_t& lo, uint32_t& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(x));
}
__device__ __forceinline__ uint64_t b2b_join(uint32_t lo, uint32_t hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}
__device__ __forceinline__ uint64_t b2b_rot32(uint64_t x) {
  uint32_t lo, hi;
  b2b_split(x, lo, hi);
  return b2b_join(hi, lo);
}
__device__ __forceinline__ uint64_t b2b_rot24(uint64_t x) {
  uint32_t lo, hi;
  b2b_split(x, lo, hi);
  return b2b_join(__byte_perm(lo, hi, 0x6543), __byte_perm(lo, hi, 0x2107));
}
__device__ __forceinline__ uint64_t b2b_rot16(uint64_t x) {
  uint32_t lo, hi;
  b2b_split(x, lo, hi);
  return b2b_join(__byte_perm(lo, hi, 0x5432), __byte_perm(lo, hi, 0x1076));
}
__device__ __forceinline__ uint64_t b2b_rot63(uint64_t x) {
  uint32_t lo, hi;
  b2b_split(x, lo, hi);
  return b2b_join(__funnelshift_l(hi, lo, 1), __funnelshift_l(lo, hi, 1));
}
#else
inline uint64_t b2b_rot32(uint64_t x) { return rotr64(x, 32); }
inline uint64_t b2b_rot24(uint64_t x) { return rotr64(x, 24); }
inline uint64_t b2b_rot16(uint64_t x) { return rotr64(x, 16); }
inline uint64_t b2b_rot63(uint64_t x) { return rotr64(x, 63); }
#endif

#define EF_B2B_G(a, b, c, d, x, y)  \
  do {                              \
    a = a + b + (x);                \
    d = ef::b2b_rot32(d ^ a);       \
    c = c + d;                      \
    b = ef::b2b_rot24(b ^ c);       \
    a = a + b + (y);                \
    d = ef::b2b_rot16(d ^ a);       \
    c = c + d;                      \
    b = ef::b2b_rot63(b ^ c);       \
  } while (0)

// one round with the message schedule spelled out (sigma row r), fully unrolled
#define EF_B2B_ROUND(m, s0, s1, s2, s3, s4, s5, s6, s7, s8, s9, s10, s11, s12, s13, s14, s15) \
  do {                                                                                         \
    EF_B2B_G(v0, v4, v8, v12, m[s0], m[s1]);                                                   \
    EF_B2B_G(v1, v5, v9, v13, m[s2], m[s3]);                                                   \
    EF_B2B_G(v2, v6, v10, v14, m[s4], m[s5]);                                                  \
    EF_B2B_G(v3, v7, v11, v15, m[s6], m[s7]);                                                  \
    EF_B2B_G(v0, v5, v10, v15, m[s8], m[s9]);                                                  \
    EF_B2B_G(v1, v6, v11, v12, m[s10], m[s11]);                                                \
    EF_B2B_G(v2, v7, v8, v13, m[s12], m[s13]);                                                 \
    EF_B2B_G(v3, v4, v9, v14, m[s14], m[s15]);                                                 \
  } while (0)

// compress one 128-byte block m[16] into h[8]; t = byte count including this block
EF_HD void b2b_compress(uint64_t* h, const uint64_t* m, uint64_t t, bool last) {
  uint64_t v0 = h[0], v1 = h[1], v2 = h[2], v3 = h[3], v4 = h[4], v5 = h[5], v6 = h[6], v7 = h[7];
  uint64_t v8 = b2b_iv(0), v9 = b2b_iv(1), v10 = b2b_iv(2), v11 = b2b_iv(3);
  uint64_t v12 = b2b_iv(4) ^ t, v13 = b2b_iv(5), v14 = b2b_iv(6), v15 = b2b_iv(7);
  if (last) v14 = ~v14;
  EF_B2B_ROUND(m, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15);
  EF_B2B_ROUND(m, 14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3);
  EF_B2B_ROUND(m, 11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4);
  EF_B2B_ROUND(m, 7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8);
  EF_B2B_ROUND(m, 9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13);
  EF_B2B_ROUND(m, 2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9);
  EF_B2B_ROUND(m, 12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11);
  EF_B2B_ROUND(m, 13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10);
  EF_B2B_ROUND(m, 6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5);
  EF_B2B_ROUND(m, 10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0);
  EF_B2B_ROUND(m, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15);
  EF_B2B_ROUND(m, 14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3);
  h[0] ^= v0 ^ v8;
  h[1] ^= v1 ^ v9;
  h[2] ^= v2 ^ v10;
  h[3] ^= v3 ^ v11;
  h[4] ^= v4 ^ v12;
  h[5] ^= v5 ^ v13;
  h[6] ^= v6 ^ v14;
  h[7] ^= v7 ^ v15;
}

// Streaming state.  `m` holds the pending block (zero-filled past `fill`).
struct B2b {
  uint64_t h[8];
  uint64_t m[16];
  uint64_t t;
  uint32_t fill;

  EF_HD void init(int outlen) {
#pragma unroll
    for (int i = 0; i < 8; ++i) h[i] = b2b_iv(i);
    h[0] ^= 0x01010000ULL ^ (uint64_t)outlen;
#pragma unroll
    for (int i = 0; i < 16; ++i) m[i] = 0;
    t = 0;
    fill = 0;
  }
  EF_HD void flush_if_full() {
    if (fill == 128) {
      t += 128;
      b2b_compress(h, m, t, false);
#pragma unroll
      for (int i = 0; i < 16; ++i) m[i] = 0;
      fill = 0;
    }
  }
  EF_HD void byte(uint8_t b) {
    flush_if_full();
    m[fill >> 3] |= (uint64_t)b << (8 * (fill & 7));
    ++fill;
  }
  EF_HD void bytes(const uint8_t* p, uint32_t n) {
    for (uint32_t i = 0; i < n; ++i) byte(p[i]);
  }
  // 8 message bytes given as a little-endian word (i.e. the bytes of a double)
  EF_HD void word_le(uint64_t w) {
    flush_if_full();
    uint32_t sh = 8 * (fill & 7);
    uint32_t k = fill >> 3;
    if (sh == 0) {
      m[k] = w;
      fill += 8;
    } else {
      m[k] |= w << sh;
      uint32_t room = 128 - fill;  // bytes left in this block (1..7 here would split)
      if (room >= 8) {
        m[k + 1] = w >> (64 - sh);
        fill += 8;
      } else {
        // the word straddles the block boundary: finish this block, carry the rest
        fill = 128;
        flush_if_full();
        m[0] = w >> (64 - sh);
        fill = 8 - room;
      }
    }
  }
  // 16 raw bytes given as two big-endian words (a node key stored as hi, lo)
  EF_HD void key_be(uint64_t hi, uint64_t lo) {
    word_le(bswap64(hi));
    word_le(bswap64(lo));
  }
  EF_HD void u16_be(uint32_t v) {
    byte((uint8_t)(v >> 8));
    byte((uint8_t)v);
  }
  EF_HD static uint64_t bswap64(uint64_t x) {
#ifdef __CUDA_ARCH__
    uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
    return ((uint64_t)__byte_perm(lo, 0, 0x0123) << 32) | __byte_perm(hi, 0, 0x0123);
#else
    return __builtin_bswap64(x);
#endif
  }
  // finalise; h[0..] little-endian bytes are the digest
  EF_HD void final() {
    t += fill;
    b2b_compress(h, m, t, true);
  }
};

}  // namespace ef

#ifdef __CUDACC__
namespace ef {

__constant__ uint8_t kB2bSigma[10][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0}};

// Compression with the 12 rounds rolled into a loop (~3 KB of SASS instead of ~35 KB), the
// message read from a per-thread shared-memory column (word k at col[k * BT]) in each round's
// schedule order: keeps the hot loop of the hash kernels inside the instruction cache.
template <int BT>
__device__ __forceinline__ void b2b_compress_col(uint64_t* h, const uint64_t* col, uint64_t t, bool last) {
  uint64_t v0 = h[0], v1 = h[1], v2 = h[2], v3 = h[3], v4 = h[4], v5 = h[5], v6 = h[6], v7 = h[7];
  uint64_t v8 = b2b_iv(0), v9 = b2b_iv(1), v10 = b2b_iv(2), v11 = b2b_iv(3);
  uint64_t v12 = b2b_iv(4) ^ t, v13 = b2b_iv(5), v14 = b2b_iv(6), v15 = b2b_iv(7);
  if (last) v14 = ~v14;
#pragma unroll 1
  for (int r = 0; r < 12; ++r) {
    const uint8_t* s = kB2bSigma[r < 10 ? r : r - 10];
    uint64_t m[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) m[i] = col[s[i] * BT];
    EF_B2B_G(v0, v4, v8, v12, m[0], m[1]);
    EF_B2B_G(v1, v5, v9, v13, m[2], m[3]);
    EF_B2B_G(v2, v6, v10, v14, m[4], m[5]);
    EF_B2B_G(v3, v7, v11, v15, m[6], m[7]);
    EF_B2B_G(v0, v5, v10, v15, m[8], m[9]);
    EF_B2B_G(v1, v6, v11, v12, m[10], m[11]);
    EF_B2B_G(v2, v7, v8, v13, m[12], m[13]);
    EF_B2B_G(v3, v4, v9, v14, m[14], m[15]);
  }
  h[0] ^= v0 ^ v8;
  h[1] ^= v1 ^ v9;
  h[2] ^= v2 ^ v10;
  h[3] ^= v3 ^ v11;
  h[4] ^= v4 ^ v12;
  h[5] ^= v5 ^ v13;
  h[6] ^= v6 ^ v14;
  h[7] ^= v7 ^ v15;
}

// The same compression for kernels with few resident warps (large graphs): the rounds are
// rolled in pairs with two message register sets, and the next round's schedule-ordered words
// are read from the column while the current round runs, so the shared-memory latency does not
// sit in front of every round's G chain.
template <int BT>
__device__ __forceinline__ void b2b_col_load(uint64_t* m, const uint64_t* col, int r) {
  const uint8_t* s = kB2bSigma[r < 10 ? r : r - 10];
#pragma unroll
  for (int i = 0; i < 16; ++i) m[i] = col[s[i] * BT];
}

template <int BT>
__device__ __forceinline__ void b2b_compress_col_pf(uint64_t* h, const uint64_t* col, uint64_t t, bool last) {
  uint64_t v0 = h[0], v1 = h[1], v2 = h[2], v3 = h[3], v4 = h[4], v5 = h[5], v6 = h[6], v7 = h[7];
  uint64_t v8 = b2b_iv(0), v9 = b2b_iv(1), v10 = b2b_iv(2), v11 = b2b_iv(3);
  uint64_t v12 = b2b_iv(4) ^ t, v13 = b2b_iv(5), v14 = b2b_iv(6), v15 = b2b_iv(7);
  if (last) v14 = ~v14;
  uint64_t ma[16], mb[16];
  b2b_col_load<BT>(ma, col, 0);
#define EF_B2B_ROUND_COL(m)                          \
  EF_B2B_G(v0, v4, v8, v12, m[0], m[1]);         \
  EF_B2B_G(v1, v5, v9, v13, m[2], m[3]);         \
  EF_B2B_G(v2, v6, v10, v14, m[4], m[5]);        \
  EF_B2B_G(v3, v7, v11, v15, m[6], m[7]);        \
  EF_B2B_G(v0, v5, v10, v15, m[8], m[9]);        \
  EF_B2B_G(v1, v6, v11, v12, m[10], m[11]);      \
  EF_B2B_G(v2, v7, v8, v13, m[12], m[13]);       \
  EF_B2B_G(v3, v4, v9, v14, m[14], m[15]);
#pragma unroll 1
  for (int r = 0; r < 12; r += 2) {
    b2b_col_load<BT>(mb, col, r + 1);
    EF_B2B_ROUND_COL(ma)
    if (r + 2 < 12) b2b_col_load<BT>(ma, col, r + 2);
    EF_B2B_ROUND_COL(mb)
  }
#undef EF_B2B_ROUND_COL
  h[0] ^= v0 ^ v8;
  h[1] ^= v1 ^ v9;
  h[2] ^= v2 ^ v10;
  h[3] ^= v3 ^ v11;
  h[4] ^= v4 ^ v12;
  h[5] ^= v5 ^ v13;
  h[6] ^= v6 ^ v14;
  h[7] ^= v7 ^ v15;
}

}  // namespace ef
#endif
