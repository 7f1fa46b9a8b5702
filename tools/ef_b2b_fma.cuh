// BLAKE2b compression (RFC 7693; same function as ef_blake2b.cuh) on 32-bit word pairs,
// arranged for the sm_100 issue pipes.  XOR and rotations go to the ALU pipe (LOP3 / PRMT /
// SHF); the high halves of the 64-bit additions go to the FMA pipe as IMAD with a run-time
// multiplier `one` (== 1, which ptxas cannot fold back into IADD3).  Measured on the SASS of
// one compression: 1938 ALU-pipe + 1212 FMA-pipe instructions versus 2230 + 325 for the plain
// 64-bit formulation -- yet tools/b2b_peak measures 6.1e9 compressions/s for this variant
// against 8.0e9 for the plain one on a B200, so the kernels use the plain one; this variant is
// kept for the microbenchmark.
#pragma once
#include <stdint.h>
namespace ef {
struct W2 { uint32_t lo, hi; };
__device__ __forceinline__ W2 w2(uint64_t x) { W2 r; asm("mov.b64 {%0, %1}, %2;" : "=r"(r.lo), "=r"(r.hi) : "l"(x)); return r; }
__device__ __forceinline__ uint64_t u64(W2 x) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(x.lo), "r"(x.hi)); return r; }
// a + b
__device__ __forceinline__ W2 fadd2(W2 a, W2 b, uint32_t one) {
  uint64_t t;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(t) : "r"(a.lo), "r"(one), "l"(u64(b)));
  W2 r = w2(t);
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r.hi) : "r"(a.hi), "r"(one), "r"(r.hi));
  return r;
}
// a + b + c
__device__ __forceinline__ W2 fadd3(W2 a, W2 b, W2 c, uint32_t one) {
  uint64_t t;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(t) : "r"(a.lo), "r"(one), "l"(u64(b)));
  asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(t) : "r"(c.lo), "r"(one));
  W2 r = w2(t);
  asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(r.hi) : "r"(a.hi), "r"(one));
  asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(r.hi) : "r"(c.hi), "r"(one));
  return r;
}
__device__ __forceinline__ W2 xr(W2 a, W2 b) { return W2{a.lo ^ b.lo, a.hi ^ b.hi}; }
__device__ __forceinline__ W2 rot32(W2 x) { return W2{x.hi, x.lo}; }
__device__ __forceinline__ W2 rot24(W2 x) { return W2{__byte_perm(x.lo, x.hi, 0x6543), __byte_perm(x.lo, x.hi, 0x2107)}; }
__device__ __forceinline__ W2 rot16(W2 x) { return W2{__byte_perm(x.lo, x.hi, 0x5432), __byte_perm(x.lo, x.hi, 0x1076)}; }
__device__ __forceinline__ W2 rot63(W2 x) { return W2{__funnelshift_l(x.hi, x.lo, 1), __funnelshift_l(x.lo, x.hi, 1)}; }

#define EF_G2(a, b, c, d, x, y)          \
  do {                                   \
    a = fadd3(a, b, x, one);             \
    d = rot32(xr(d, a));                 \
    c = fadd2(c, d, one);                \
    b = rot24(xr(b, c));                 \
    a = fadd3(a, b, y, one);             \
    d = rot16(xr(d, a));                 \
    c = fadd2(c, d, one);                \
    b = rot63(xr(b, c));                 \
  } while (0)

#define EF_R2(s0, s1, s2, s3, s4, s5, s6, s7, s8, s9, s10, s11, s12, s13, s14, s15) \
  do {                                                                             \
    EF_G2(v[0], v[4], v[8], v[12], M[s0], M[s1]);                                  \
    EF_G2(v[1], v[5], v[9], v[13], M[s2], M[s3]);                                  \
    EF_G2(v[2], v[6], v[10], v[14], M[s4], M[s5]);                                 \
    EF_G2(v[3], v[7], v[11], v[15], M[s6], M[s7]);                                 \
    EF_G2(v[0], v[5], v[10], v[15], M[s8], M[s9]);                                 \
    EF_G2(v[1], v[6], v[11], v[12], M[s10], M[s11]);                               \
    EF_G2(v[2], v[7], v[8], v[13], M[s12], M[s13]);                                \
    EF_G2(v[3], v[4], v[9], v[14], M[s14], M[s15]);                                \
  } while (0)

__device__ __forceinline__ void b2b_compress_fma(uint64_t* h, const uint64_t* m, uint64_t t, bool last, uint32_t one) {
  W2 v[16], M[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) M[i] = w2(m[i]);
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = w2(h[i]);
  v[8] = w2(0x6a09e667f3bcc908ULL); v[9] = w2(0xbb67ae8584caa73bULL);
  v[10] = w2(0x3c6ef372fe94f82bULL); v[11] = w2(0xa54ff53a5f1d36f1ULL);
  v[12] = w2(0x510e527fade682d1ULL ^ t); v[13] = w2(0x9b05688c2b3e6c1fULL);
  v[14] = w2(last ? ~0x1f83d9abfb41bd6bULL : 0x1f83d9abfb41bd6bULL); v[15] = w2(0x5be0cd19137e2179ULL);
  EF_R2(0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15);
  EF_R2(14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3);
  EF_R2(11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4);
  EF_R2(7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8);
  EF_R2(9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13);
  EF_R2(2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9);
  EF_R2(12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11);
  EF_R2(13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10);
  EF_R2(6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5);
  EF_R2(10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0);
  EF_R2(0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15);
  EF_R2(14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3);
#pragma unroll
  for (int i = 0; i < 8; ++i) h[i] ^= u64(v[i]) ^ u64(v[i + 8]);
}
}  // namespace ef
