// Device-side pieces shared by the multi-GPU kernels (peer.cu, peer_merge.cu).
#pragma once
#include "common.cuh"
#include "peer.cuh"
#include "ptx.cuh"

namespace cs {

// The CTAs of one launch, split among the ranks it runs for.  A real multi-GPU launch
// runs for one rank (vranks == 1: every CTA is rank s.rank's).  The single-GPU emulation of
// the multi-GPU protocol (PeerState::vranks = V > 1) runs ONE cooperative launch over all
// V ranks' data: CTAs [v*G, (v+1)*G) act as rank v, so CTAs that wait for another rank's
// CTAs are co-resident by construction (B200_PROFILING.md: ranks that wait on one another
// must not be separate launches on one GPU).
struct RankCta {
  int rank;   // the rank this CTA works for
  int b;      // CTA index within that rank's grid
  int G;      // CTAs per rank
};

__device__ __forceinline__ RankCta rank_cta(int vranks, int rank) {
  RankCta r;
  if (vranks <= 1) {
    r.rank = rank;
    r.b = blockIdx.x;
    r.G = gridDim.x;
  } else {
    r.G = gridDim.x / vranks;
    r.rank = blockIdx.x / r.G;
    r.b = blockIdx.x - r.rank * r.G;
  }
  return r;
}

// Rank `rank`'s view of step arguments given for rank 0 of an emulated launch: its local
// workers are rows [rank*n_loc, (rank+1)*n_loc) of the caller's whole-world buffers.
// g_off != 0: the gradient lives in the rank's exchange region (the hierarchical group mean).
__device__ __forceinline__ void rank_view(PeerStepArgs& s, char* const* peers, int vranks, int rank) {
  if (vranks > 1) {
    const int64_t rows = (int64_t)rank * s.n_loc;
    s.rank = rank;
    s.first = rank * s.n_loc;
    s.x += rows * s.ld;
    s.m += rows * s.ld;
    if (s.g_off == 0) s.g += rows * s.ld;
    s.psw += rows * s.k;
    if (s.lrs) s.lrs += rows * s.n_layers;
  }
  if (s.g_off != 0) s.g = reinterpret_cast<const float*>(peers[s.rank] + s.g_off);
}

// Bulk-load the gradient columns [c0, c0 + n4) (n4 a multiple of 4) of a one-worker-per-GPU
// step into smem: from s.g, or -- pulled group mean -- from the gbar row of each owning member
// (one copy per owner crossed; chunk bounds are multiples of 4 elements, so every piece is a
// whole number of 16-byte units).
__device__ __forceinline__ void bulk_load_g(const PeerStepArgs& s, char* const* peers, float* dst, int64_t off,
                                            int64_t c0, int64_t n4, uint64_t* bar) {
  if (s.gpull_chunk <= 0) {
    ptx::bulk_g2s(dst, s.g + off, (uint32_t)(n4 * 4), bar);
    return;
  }
  const int gbase = (s.rank / s.gs) * s.gs;
  for (int64_t c = c0; c < c0 + n4;) {
    const int own = (int)(c / s.gpull_chunk);
    const int64_t e = (own + 1) * s.gpull_chunk < c0 + n4 ? (own + 1) * s.gpull_chunk : c0 + n4;
    ptx::bulk_g2s(dst + (c - c0), reinterpret_cast<const float*>(peers[gbase + own] + s.g_off) + c,
                  (uint32_t)((e - c) * 4), bar);
    c = e;
  }
}

// Global worker that receives segment s of local worker r (send_to, Alg.1 l.6):
// flat: dst_s(first + r); hierarchical: the member of the same index in group
// dstL_s(my group) (replicated leader).
__device__ __forceinline__ int receiver_worker(const PeerStepArgs& s, int seg, int r) {
  if (s.gs == 0) return s.dst[(int64_t)seg * s.world + s.first + r];
  const int grp = s.rank / s.gs, member = s.rank - grp * s.gs;
  return s.dst[(int64_t)seg * s.groups + grp] * s.gs + member;
}

}  // namespace cs
