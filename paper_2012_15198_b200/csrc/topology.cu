// Load-balanced random topology (§3.2, Algorithm 2), host and device.
//
// For every rank i = 0..n-1 in order, Alg. 2 zeroes the roulette entries of the
// ranks already in dest_list (l.2-4) — and, reading C-5/C-7, of i itself (zero
// diagonal) — renormalises the row (l.5-6) and draws (l.7).  With
// uniform initial roulettes the renormalised row is uniform over the remaining
// candidates, so the draw is "the c-th remaining candidate in ascending rank
// order", c = (u32 * |cand|) >> 32 (reading C-7).  A dead end (only i itself
// left) restarts the whole draw with attempt + 1 (reading C-6).  The result
// src[i] is the rank i receives from (reading C-1).
//
// Device form: one warp per segment; the set of not-yet-picked ranks is a
// 1024-bit mask, one 32-bit word per lane; the c-th candidate is found with a
// warp prefix sum of popcounts.  After the draw the same warp derives the
// inverse permutation (send_to, Alg.1 l.6), the cycle order used by the
// single-GPU column-owner kernel, and the push-sum weight mix
// w' = (w + w_src) * 0.5 (reading C-11).
#include <vector>

#include "common.cuh"
#include "philox.cuh"

namespace cs {

// ---------------------------------------------------------------- host ------
int host_alg2(uint64_t seed, uint32_t step, uint32_t seg, int n, int tag, int32_t* src) {
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  std::vector<uint32_t> u(n);
  std::vector<int32_t> avail;
  avail.reserve(n);
  for (int attempt = 0; attempt < kMaxAttempts; ++attempt) {
    for (int q = 0; q < (n + 3) / 4; ++q) {
      U32x4 r = philox4x32_10((uint32_t)q, (uint32_t)attempt | ((uint32_t)tag << 16), seg, step, k0, k1);
      for (int e = 0; e < 4 && 4 * q + e < n; ++e) u[4 * q + e] = r.v[e];
    }
    avail.clear();
    for (int r = 0; r < n; ++r) avail.push_back(r);
    bool ok = true;
    for (int i = 0; i < n; ++i) {
      // candidates = avail without i, ascending
      int has_self = 0;
      for (int32_t r : avail) has_self |= (r == i);
      uint32_t ncand = (uint32_t)avail.size() - (uint32_t)has_self;
      if (ncand == 0) { ok = false; break; }
      uint32_t c = roulette_index(u[i], ncand);
      size_t pos = 0;
      for (; pos < avail.size(); ++pos) {
        if (avail[pos] == i) continue;
        if (c == 0) break;
        --c;
      }
      src[i] = avail[pos];
      avail.erase(avail.begin() + (long)pos);
    }
    if (ok) return attempt + 1;
  }
  return -1;
}

// -------------------------------------------------------------- device ------
__global__ void __launch_bounds__(32) k_topology(TopoArgs a) {
  const int s = blockIdx.x;
  const int lane = threadIdx.x;
  const int n = a.n;
  const unsigned FULL = 0xffffffffu;
  __shared__ uint32_t u[kMaxWorld];
  __shared__ int32_t src[kMaxWorld];
  __shared__ float wsnap[kMaxWorld];

  if (a.given != nullptr) {
    for (int i = lane; i < n; i += 32) src[i] = a.given[(int64_t)s * n + i];
  } else if (n == 1) {
    if (lane == 0) src[0] = 0;   // a single leader (G = 1): no exchange partner, no mixing
  } else {
    const uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);
    bool done = false;
    for (int attempt = 0; attempt < kMaxAttempts && !done; ++attempt) {
      for (int q = lane; q < (n + 3) / 4; q += 32) {
        U32x4 r = philox4x32_10((uint32_t)q, (uint32_t)attempt | ((uint32_t)a.tag << 16),
                                (uint32_t)s, a.step, k0, k1);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (4 * q + e < n) u[4 * q + e] = r.v[e];
      }
      __syncwarp();
      // availability word of ranks [32*lane, 32*lane + 32)
      int lo = 32 * lane;
      uint32_t avail = lo >= n ? 0u : (n - lo >= 32 ? FULL : ((1u << (n - lo)) - 1u));
      bool ok = true;
      for (int i = 0; i < n; ++i) {
        uint32_t own = avail;
        if (lane == (i >> 5)) own &= ~(1u << (i & 31));      // zero diagonal
        uint32_t cnt = __popc(own);
        uint32_t incl = cnt;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          uint32_t t = __shfl_up_sync(FULL, incl, off);
          if (lane >= off) incl += t;
        }
        uint32_t total = __shfl_sync(FULL, incl, 31);
        if (total == 0) { ok = false; break; }               // dead end -> restart
        uint32_t c = roulette_index(u[i], total);
        uint32_t excl = incl - cnt;
        if (c >= excl && c < incl) {
          uint32_t mm = own;
          for (uint32_t t = 0; t < c - excl; ++t) mm &= mm - 1u;
          int bit = __ffs(mm) - 1;
          src[i] = lo + bit;
          avail &= ~(1u << bit);
        }
      }
      done = ok;
      __syncwarp();
    }
    if (!done) {
      if (lane == 0) atomicOr(a.err + kErrTopology, 1);
      for (int i = lane; i < n; i += 32) src[i] = (i + 1) % n;   // keep tables a valid permutation
    }
  }
  __syncwarp();

  for (int i = lane; i < n; i += 32) {
    a.src[(int64_t)s * n + i] = src[i];
    a.dst[(int64_t)s * n + src[i]] = i;
  }

  // push-sum weights: snapshot, then w'_{i,s} = (w_{i,s} + w_{src(i),s}) * 0.5 on every
  // row of rank i's group (group_size rows; 1 for the flat step).
  if (a.psw != nullptr) {
    const int gs = a.group_size;
    for (int i = lane; i < n; i += 32) wsnap[i] = a.psw[(int64_t)i * gs * a.k + s];
    __syncwarp();
    double wsum = 0.0;
    for (int i = lane; i < n; i += 32) {
      float nw = (n >= 2) ? __fmul_rn(__fadd_rn(wsnap[i], wsnap[src[i]]), 0.5f) : wsnap[i];
      for (int r = 0; r < gs; ++r) a.psw[((int64_t)i * gs + r) * a.k + s] = nw;
      if (a.rw != nullptr) a.rw[(int64_t)s * n + i] = 1.0 / (double)nw;
      wsum += (double)nw * (double)gs;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) wsum += __shfl_xor_sync(FULL, wsum, off);
    if (lane == 0 && a.inv_wsum != nullptr) a.inv_wsum[s] = 1.0 / wsum;
  }

  // cycle order (single-GPU column-owner kernel)
  if (lane == 0 && a.ord != nullptr) {
    uint32_t* seen = u;  // reuse: draws are no longer needed
    for (int i = 0; i < n; ++i) seen[i] = 0;
    int pos = 0;
    for (int i0 = 0; i0 < n; ++i0) {
      if (seen[i0]) continue;
      int p = i0;
      uint32_t flag = kOrdStart;
      do {
        seen[p] = 1;
        int nx = src[p];
        uint32_t e = (uint32_t)p | flag | (nx == i0 ? kOrdEnd : 0u);
        a.ord[(int64_t)s * n + pos++] = e;
        flag = 0;
        p = nx;
      } while (p != i0);
    }
  }
}

cudaError_t launch_topology(const TopoArgs& a, cudaStream_t st) {
  k_topology<<<a.k, 32, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace cs
