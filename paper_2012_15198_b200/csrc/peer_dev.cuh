// Device-side pieces shared by the multi-GPU kernels (peer.cu, peer_merge.cu).
#pragma once
#include "common.cuh"
#include "peer.cuh"

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

// Global worker that receives segment s of local worker r (send_to, Alg.1 l.6):
// flat: dst_s(first + r); hierarchical: the member of the same index in group
// dstL_s(my group) (replicated leader).
__device__ __forceinline__ int receiver_worker(const PeerStepArgs& s, int seg, int r) {
  if (s.gs == 0) return s.dst[(int64_t)seg * s.world + s.first + r];
  const int grp = s.rank / s.gs, member = s.rank - grp * s.gs;
  return s.dst[(int64_t)seg * s.groups + grp] * s.gs + member;
}

}  // namespace cs
