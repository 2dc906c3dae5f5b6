// Philox4x32-10 counter-based generator (Salmon, Moraes, Dror, Shaw, SC'11),
// shared by the host topology generator and the device one so the two agree
// bit for bit.  The draw layout is reading C-4: the paper's
// `choice(world_size, roulette, seed=rseed)` (Alg.2 l.7) becomes
// one 32-bit word of Philox(ctr = [i>>2, attempt | tag<<16, segment, step],
// key = [seed lo32, seed hi32]), word index i & 3.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define CS_HD __host__ __device__ __forceinline__
#else
#define CS_HD inline
#endif

namespace cs {

struct U32x4 { uint32_t v[4]; };

CS_HD void mulhilo32(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
#if defined(__CUDA_ARCH__)
  lo = a * b;
  hi = __umulhi(a, b);
#else
  uint64_t p = (uint64_t)a * (uint64_t)b;
  hi = (uint32_t)(p >> 32);
  lo = (uint32_t)p;
#endif
}

CS_HD U32x4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                          uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += W0; k1 += W1; }
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo32(M0, c0, hi0, lo0);
    mulhilo32(M1, c2, hi1, lo1);
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  U32x4 out;
  out.v[0] = c0; out.v[1] = c1; out.v[2] = c2; out.v[3] = c3;
  return out;
}

// Roulette pick over |cand| uniform candidates (reading C-7): floor(u/2^32 * |cand|).
CS_HD uint32_t roulette_index(uint32_t u, uint32_t ncand) {
  return (uint32_t)(((uint64_t)u * (uint64_t)ncand) >> 32);
}

}  // namespace cs
