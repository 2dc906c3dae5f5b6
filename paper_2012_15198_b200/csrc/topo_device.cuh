// Device-side Alg. 2 for small topologies, shared by the fused kernels.
#pragma once
#include "common.cuh"
#include "philox.cuh"

namespace cs {

// Alg. 2 for one segment by one warp, n <= 64 (readings C-5..C-7):
// lanes draw the Philox words of an attempt in parallel, lane 0 runs the
// sequential roulette over a 64-bit availability mask, the warp restarts on a
// dead end.  Same definition as host_alg2 / the oracle; different code.
// u: >= 64 words of per-warp scratch; src: n outputs (shared or global).
__device__ inline void warp_alg2_small(uint64_t seed, uint32_t step, int s, int n, int tag, uint32_t* u,
                                       int32_t* src, int* err) {
  const int lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  const int nb = (n + 3) >> 2;
  for (int attempt = 0; attempt < kMaxAttempts; ++attempt) {
    if (lane < nb) {
      U32x4 r = philox4x32_10((uint32_t)lane, (uint32_t)attempt | ((uint32_t)tag << 16), (uint32_t)s, step, k0,
                              k1);
      u[4 * lane] = r.v[0];
      u[4 * lane + 1] = r.v[1];
      u[4 * lane + 2] = r.v[2];
      u[4 * lane + 3] = r.v[3];
    }
    __syncwarp();
    int ok = 1;
    if (lane == 0) {
      uint64_t avail = (n == 64) ? ~0ull : ((1ull << n) - 1ull);
      for (int i = 0; i < n; ++i) {
        const uint64_t cand = avail & ~(1ull << i);        // zero diagonal + picked ranks
        const uint32_t cnt = (uint32_t)__popcll(cand);
        if (cnt == 0) { ok = 0; break; }                   // dead end -> restart (C-6)
        const uint32_t c = roulette_index(u[i], cnt);      // C-7
        const uint32_t lo = (uint32_t)cand, hi = (uint32_t)(cand >> 32);
        const uint32_t plo = (uint32_t)__popc(lo);
        const int bit = c < plo ? (int)__fns(lo, 0, (int)c + 1) : 32 + (int)__fns(hi, 0, (int)(c - plo) + 1);
        src[i] = bit;
        avail &= ~(1ull << bit);
      }
    }
    ok = __shfl_sync(FULL, ok, 0);
    __syncwarp();
    if (ok) return;
  }
  if (lane == 0) {
    atomicOr(err + kErrTopology, 1);
    for (int i = 0; i < n; ++i) src[i] = (i + 1) % n;
  }
  __syncwarp();
}

}  // namespace cs
