// Multi-GPU steps over NVLink peer memory (configs 3, 4 and 5).
//
// Workers are partitioned contiguously: worker w lives on GPU w / n_loc.  The
// segments a worker receives (Alg.1 l.4-8) come from workers on
// other GPUs, so each step is a streaming push followed by a streaming mix:
//
//   k_peer_push  (one CTA per unit = (tile q, local worker r), tiles of kPeerTile
//                columns inside one segment)  a bulk-TMA load warp stages the x, m,
//                g row-tiles; 8 compute warps form m', y (a3) and store m' and
//                y -> x into HBM and y into a shared-memory ring; a store warp
//                ships each 8 KB y tile with ONE bulk copy
//                (cp.async.bulk.global.shared::cta) into the inbox of the worker
//                that receives it, on that worker's GPU (Alg.1 l.7 isend to
//                send_to = dst_s(i)).  w_{i,s} goes to the receiver's wbox.  When
//                every CTA's bulk stores have landed, the last CTA publishes
//                push_done[rank] = epoch on every GPU (the irecv completion,
//                Alg.1 l.14).
//   k_peer_mix   waits until every GPU published push_done (Alg.1 l.12-14 "wait
//                send and recv"), then x = (y + inbox) * 0.5 and
//                w = (w + wbox) * 0.5 (a5, Alg.1 l.17); the last CTA publishes
//                done[rank] = epoch.
//
// Deferred merge (default, CS_PEER_FUSE): the mix of step e is not launched.  Step
// e+1's push applies it tile by tile: its load warp waits for push_done(e) from every
// GPU and bulk-loads the inbox tile next to x, m, g, and its compute warps form
// x = (y + inbox)/2 before the update.  Its last CTA stores the merged weights and
// publishes push_done(e+1) and done(e).  k_peer_mix runs only in peer_flush (cs_flush,
// cs_sync, diagnostics, LARS, reconfiguration).  The hybrid walk for several workers
// per GPU (k_hyb_walk, below) defers its chain-tail merge the same way.
//
// The inbox and wbox ping-pong on the epoch parity; a push at epoch e first waits
// until every GPU finished consuming epoch e-2's inbox (done >= e-2), the last reader
// of that parity.  Epochs are monotone, so no flag is ever reset.  Every wait is
// bounded (~20 s of %globaltimer) and reports CS_ETIMEOUT instead of hanging the GPU.
//
// The bulk-TMA push was chosen by measurement: on 2 B200s it moves
// the NVLink segment traffic at ~595 GB/s per direction against ~555 GB/s for
// 128-bit register stores, and fused single-kernel schedules with per-tile or
// per-wave flags lost more to synchronisation than they won in overlap.
//
// Hierarchical step (§3.3), one worker per GPU, groups of gs
// consecutive GPUs:
//   k_hier_scatter  each member sends chunk c of its gradient to member c's gbox
//                   (reduce-scatter, NVLink, destinations rotated);
//   k_hier_reduce   member c sums the chunk over the members in ascending order and
//                   scales by fp32(1/|G|) (reading C-12 — the oracle's exact order,
//                   so the result is bit-identical), then all-gathers the mean chunk
//                   into every member's gbar (optionally, CS_HIER_PIECES, the vector is
//                   cut into column pieces whose update overlaps the next piece's h1;
//                   measured slower, off by default);
//   k_peer_push/mix with g = gbar over the leader topology (tag HIER): every
//                   member exchanges with the member of the same index in the
//                   source group.  All members hold the leader's state bit for bit
//                   ("replicated leader"), so step h3 (propagation to the members)
//                   needs no transfer.  One group: no exchange, x = y.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/crossover_sgd.h"
#include "arith.cuh"
#include "common.cuh"
#include "peer.cuh"
#include "peer_dev.cuh"
#include "ptx.cuh"
#include "topo_device.cuh"

namespace cs {

long g_peer_launches = 0;

namespace {

std::string g_peer_err;

int perr(int code, const char* what, cudaError_t e) {
  char buf[256];
  snprintf(buf, sizeof(buf), "%s: %s", what, e == cudaSuccess ? "" : cudaGetErrorString(e));
  g_peer_err = buf;
  return code;
}

constexpr int kCompute = 256;                       // compute warps
constexpr int kPushThreads = kCompute + 64;         // + load warp + store warp
constexpr int kPer = kPeerTile / 4 / kCompute;      // float4 per compute thread per array
constexpr int kStagesA = 3, kSlotsY = 3;            // x, m, g ring depth; y ring depth (units)
constexpr size_t kTileBytes = sizeof(float) * kPeerTile;
constexpr size_t kRingBytes = kTileBytes * (3 * kStagesA + kSlotsY);
constexpr int kMaxRecvSmem = 2048;                  // receivers table in smem when k*n_loc <= this
constexpr int kMixThreads = 256;
constexpr int kHierThreads = 256;

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

size_t push_smem_bytes(int k, int n_loc) {
  size_t b = kRingBytes + sizeof(int64_t) * (k + 1) + sizeof(int32_t) * (k + 1);
  if ((int64_t)k * n_loc <= kMaxRecvSmem) b += sizeof(int32_t) * (size_t)k * n_loc;
  b += sizeof(uint32_t) * 128 * (kPushThreads / 32);  // per-warp Alg. 2 scratch
  return align_up(b, 16);
}

bool fused_topo_ok(int ntop, int k, int n_loc) { return ntop <= 64 && (int64_t)k * n_loc <= kMaxRecvSmem; }

__device__ __forceinline__ bool wait_acquire(const uint32_t* p, uint32_t target) {
  return ptx::wait_geq_sys(p, target);
}

// Grid-wide completion: every CTA adds 1 to the arrival counter at `count_off`;
// the CTA that brings it to `target` (the host's running total of CTAs launched
// against that counter, so launches of any grid size may interleave) publishes
// `epoch` at word [rank] of `flag_off` on the GPUs [first, first + count).
// (`copies` flag arrays `stride` bytes apart are published: every piece of a step
// that had nothing to exchange.)
__device__ void publish_when_last(char* const* peers, char* mine, size_t count_off, size_t flag_off, int rank,
                                  int first, int count, uint32_t epoch, uint32_t target, int copies = 1,
                                  size_t stride = 0) {
  __threadfence();
  uint32_t* cnt = reinterpret_cast<uint32_t*>(mine + count_off);
  const uint32_t prev = atomicAdd(cnt, 1u);
  if (prev + 1 == target) {
    __threadfence_system();
    for (int c = 0; c < copies; ++c)
      for (int p = first; p < first + count; ++p)
        ptx::st_release_sys(reinterpret_cast<uint32_t*>(peers[p] + flag_off + c * stride) + rank, epoch);
  }
}

struct PeerKernelArgs {
  PeerStepArgs s;
  char* const* peers;       // [nprocs] region bases
  const int64_t* bounds;    // [k+1] segment bounds
  const int32_t* seg_t0;    // [k+1] first tile of each segment (seg_t0[k] = n_tiles)
  const TileDesc* tiles;    // explicit tile table (layer table set) or nullptr
  int n_tiles;
  int tile_lo, tile_hi;     // this launch's piece of the step: tiles [tile_lo, tile_hi)
  int pieces;               // pieces per step and the stride of their flag arrays
  size_t flag_stride;
  int64_t col_lo, col_hi;   // ... = columns [col_lo, col_hi)
  uint32_t epoch;           // this step's epoch (>= 1)
  uint32_t done_target;     // arrival targets (see publish_when_last)
  uint32_t pdone_target;
  int final_only;           // hierarchical with one group: x = y, no exchange
  int fuse_mix;             // x holds y of epoch-1 and the inbox its received half: apply that
                            // step's merge x = (y + inbox)/2 (and psw) before this update
  int fused_topo;           // draw the topology in the push prologue (<= 64 ranks)
  int vranks;               // > 1: one cooperative launch over all emulated ranks (peer_dev.cuh)
  size_t off_inbox, off_wbox, off_done, off_count, off_pdone, off_pcount, off_d2;
};

// streaming store (evict-first): data not read again this step
__device__ __forceinline__ void st4_cs(float* p, float4 v, int valid) {
  if (valid == 4) {
    __stcs(reinterpret_cast<float4*>(p), v);
  } else {
    if (valid > 0) p[0] = v.x;
    if (valid > 1) p[1] = v.y;
    if (valid > 2) p[2] = v.z;
  }
}
// default-policy store: y (read back by the mix), remote buffers
__device__ __forceinline__ void st4(float* p, float4 v, int valid) {
  if (valid == 4) {
    *reinterpret_cast<float4*>(p) = v;
  } else {
    if (valid > 0) p[0] = v.x;
    if (valid > 1) p[1] = v.y;
    if (valid > 2) p[2] = v.z;
  }
}
__device__ __forceinline__ float4 ld4_valid(const float* p, int valid) {
  if (valid >= 4) return __ldcg(reinterpret_cast<const float4*>(p));
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (valid > 0) v.x = __ldcg(p);
  if (valid > 1) v.y = __ldcg(p + 1);
  if (valid > 2) v.z = __ldcg(p + 2);
  return v;
}
// Shared-memory unit metadata.
struct Meta {
  const int64_t* bnd;   // [k+1]
  const int32_t* t0;    // [k+1]
  const int32_t* recv;  // [k][n_loc] global worker receiving local worker r's segment s
  bool recv_global;     // table too large for smem: compute from the global dst table
};

struct Unit {
  int tile, r, seg, len, layer;
  int64_t c0;
  bool first_tile;
};

__device__ __forceinline__ Unit unit_at(const PeerKernelArgs& a, const Meta& M, int u, int& cursor) {
  Unit x;
  x.tile = u / a.s.n_loc;
  x.r = u - x.tile * a.s.n_loc;
  while (M.t0[cursor + 1] <= x.tile) ++cursor;
  x.seg = cursor;
  x.first_tile = x.tile == M.t0[cursor];
  if (a.tiles != nullptr) {  // layer table: explicit tiles
    const TileDesc td = a.tiles[x.tile];
    x.c0 = td.c0;
    x.len = td.len;
    x.layer = td.layer;
    return x;
  }
  const int64_t c0 = M.bnd[cursor] + (int64_t)(x.tile - M.t0[cursor]) * kPeerTile;
  const int64_t c1 = c0 + kPeerTile < M.bnd[cursor + 1] ? c0 + kPeerTile : M.bnd[cursor + 1];
  x.c0 = c0;
  x.len = (int)(c1 - c0);
  x.layer = 0;
  return x;
}

__device__ __forceinline__ void receiver_of(const PeerKernelArgs& a, const Meta& M, int seg, int r, int& rp,
                                            int& rl) {
  const int recv = M.recv_global ? receiver_worker(a.s, seg, r) : M.recv[seg * a.s.n_loc + r];
  rp = recv / a.s.n_loc;
  rl = recv - rp * a.s.n_loc;
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kPushThreads, 2) k_peer_push(const PeerKernelArgs a0) {
  PeerKernelArgs a = a0;
  const RankCta rc = rank_cta(a0.vranks, a0.s.rank);
  rank_view(a.s, a.peers, a0.vranks, rc.rank);
  const int BX = rc.b, GX = rc.G;
  extern __shared__ __align__(128) float smem_f[];
  float* ringA = smem_f;                                     // [kStagesA][3][kPeerTile]
  float* ringY = ringA + (size_t)kStagesA * 3 * kPeerTile;   // [kSlotsY][kPeerTile]
  // fused merge: the ring holds x, m, g and the previous step's inbox tile, 2 stages deep
  // (the same 9-tile region; 2 x 4 = 8 tiles)
  const int NS = a.fuse_mix ? 2 : kStagesA, NA = a.fuse_mix ? 4 : 3;
  __shared__ uint64_t a_full[kStagesA], a_empty[kStagesA], y_full[kSlotsY], y_empty[kSlotsY];
  __shared__ int s_timeout;
  const PeerStepArgs& s = a.s;
  const uint32_t e = a.epoch;
  const int par = (int)(e & 1u);
  char* mine = a.peers[s.rank];
  const int u_lo = a.tile_lo * s.n_loc;
  const int n_units = (a.tile_hi - a.tile_lo) * s.n_loc;
  const int G = GX;
  const int n_my = BX < n_units ? (n_units - BX + G - 1) / G : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  volatile int* timeout = &s_timeout;

  int64_t* bnd = reinterpret_cast<int64_t*>(ringY + (size_t)kSlotsY * kPeerTile);
  int32_t* t0 = reinterpret_cast<int32_t*>(bnd + s.k + 1);
  int32_t* recv = t0 + s.k + 1;
  Meta M;
  M.bnd = bnd;
  M.t0 = t0;
  M.recv = recv;
  M.recv_global = (int64_t)s.k * s.n_loc > kMaxRecvSmem;
  for (int i = threadIdx.x; i <= s.k; i += blockDim.x) {
    bnd[i] = a.bounds[i];
    t0[i] = a.seg_t0[i];
  }
  if (threadIdx.x == 0) {
    s_timeout = 0;
    for (int i = 0; i < kStagesA; ++i) {
      ptx::mbar_init(&a_full[i], 1);
      ptx::mbar_init(&a_empty[i], kCompute / 32);
    }
    for (int i = 0; i < kSlotsY; ++i) {
      ptx::mbar_init(&y_full[i], kCompute / 32);
      ptx::mbar_init(&y_empty[i], 1);
    }
    ptx::mbar_fence_init();
  }
  __syncthreads();
  constexpr int kLoadWarp = kCompute / 32;
  if (warp == kLoadWarp) {
    // the load warp starts streaming at once; hierarchical: it is the only reader of the
    // group mean (gbar), so it alone waits for it to be complete on this GPU
    if (s.gs > 0 && !s.gbar_local && lane < s.gs) {
      const uint32_t* d2 = reinterpret_cast<const uint32_t*>(mine + a.off_d2);
      const int gbase = (s.rank / s.gs) * s.gs;
      if (!wait_acquire(d2 + gbase + lane, e)) atomicOr(&s_timeout, 1);
    }
    if (a.fuse_mix && lane < s.nprocs) {  // every GPU's pushes of epoch e-1 have landed here
      const uint32_t* pd = reinterpret_cast<const uint32_t*>(mine + a.off_pdone);
      if (!wait_acquire(pd + lane, e - 1)) atomicOr(&s_timeout, 1);
    }
    __syncwarp();
  } else {
    // meanwhile the other warps draw the receivers table ...
    const int gw = warp < kLoadWarp ? warp : warp - 1, nw = (kPushThreads >> 5) - 1;
    if (!M.recv_global && !a.final_only) {
      if (a.fused_topo) {
        // this step's topologies (Alg. 2): one warp per segment, then
        // keep only where this GPU's workers send (send_to, Alg.1 l.6)
        const int ntop = s.gs > 0 ? s.groups : s.world;
        uint32_t* u = reinterpret_cast<uint32_t*>(recv + s.k * s.n_loc) + gw * 128;
        int32_t* srow = reinterpret_cast<int32_t*>(u + 64);
        for (int sg = gw; sg < s.k; sg += nw) {
          if (s.given != nullptr) {
            for (int i = lane; i < ntop; i += 32) srow[i] = s.given[(int64_t)sg * ntop + i];
            __syncwarp();
          } else {
            warp_alg2_small(s.seed, s.step, sg, ntop, s.gs > 0 ? CS_TAG_HIER : CS_TAG_FLAT, u, srow, s.err);
          }
          for (int r = lane; r < s.n_loc; r += 32) {
            const int grp = s.gs > 0 ? s.rank / s.gs : 0;
            const int target = s.gs > 0 ? grp : s.first + r;
            int to = 0;
            for (int jj = 0; jj < ntop; ++jj)
              if (srow[jj] == target) to = jj;
            recv[sg * s.n_loc + r] = s.gs > 0 ? to * s.gs + (s.rank - grp * s.gs) : to;
          }
          __syncwarp();
        }
      } else {
        for (int i = gw * 32 + lane; i < s.k * s.n_loc; i += nw * 32) {
          const int sg = i / s.n_loc, r = i - sg * s.n_loc;
          recv[i] = receiver_worker(s, sg, r);
        }
      }
    }
    // ... and make sure every GPU finished its mix of epoch e-2 (the last reader of the
    // inbox parity this step writes) before anything is pushed
    if (threadIdx.x < s.nprocs && e >= 3 && !a.final_only) {  // final_only writes no inbox
      const uint32_t* done = reinterpret_cast<const uint32_t*>(mine + a.off_done);
      if (!wait_acquire(done + threadIdx.x, e - 2)) atomicOr(&s_timeout, 1);
    }
  }
  // every warp, the load warp included, sees a timeout of the waits above before its loop:
  // on timeout all roles skip their loops together, so none waits on an mbarrier phase the
  // others never complete (these are the kernel's only cross-GPU waits)
  __syncthreads();

  if (warp < kCompute / 32) {
    // ---------------- compute warps: m', y; y -> x and the y ring --------------------
    bool bad = false;
    const int tid = threadIdx.x;
    int cur = 0;
    for (int i = 0; i < n_my && !*timeout; ++i) {
      const Unit U = unit_at(a, M, u_lo + BX + i * G, cur);
      const int st = i % NS, sy = i % kSlotsY;
      ptx::mbar_wait(&a_full[st], (uint32_t)((i / NS) & 1));
      if (!a.final_only) ptx::mbar_wait(&y_empty[sy], (uint32_t)(((i / kSlotsY) & 1) ^ 1));
      const float* bx = ringA + (size_t)st * NA * kPeerTile;
      float4* yt = reinterpret_cast<float4*>(ringY + (size_t)sy * kPeerTile);
      const int64_t rowoff = (int64_t)U.r * s.ld;
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int v = tid + q * kCompute;
        const int valid = U.len - 4 * v;
        if (valid > 0) {
          const int vv = valid < 4 ? valid : 4;
          float4 cx = reinterpret_cast<const float4*>(bx)[v];
          const float4 cm = reinterpret_cast<const float4*>(bx + kPeerTile)[v];
          float4 cg = reinterpret_cast<const float4*>(bx + 2 * kPeerTile)[v];
          if (s.g_scale != 1.f) cg = scale4(cg, s.g_scale);  // NCCL h1: the group sum -> mean
          if (a.fuse_mix)  // the previous step's a5: x = (y + received y) / 2 (Alg.1 l.17)
            cx = mean4(cx, s.wire ? unpack_bf16x4(reinterpret_cast<const uint2*>(bx + 3 * kPeerTile)[v])
                                  : reinterpret_cast<const float4*>(bx + 3 * kPeerTile)[v]);
          bad |= nonfinite4(cg);
          // LARS (C-18): m' = mu*m + (g + wd*x), y = x - lrs[r][layer]*m'
          const float4 mn = mom4(cm, s.lrs ? decay4(cg, cx, s.wd) : cg, s.mu);
          const float4 y = sgd4(cx, mn, s.lrs ? __ldg(s.lrs + (int64_t)U.r * s.n_layers + U.layer) : s.lr);
          const int64_t j = U.c0 + 4 * (int64_t)v;
          st4_cs(s.m + rowoff + j, mn, vv);
          if (a.final_only) {
            st4_cs(s.x + rowoff + j, y, vv);
          } else {
            st4(s.x + rowoff + j, y, vv);
            if (s.wire) reinterpret_cast<uint2*>(yt)[v] = pack_bf16x4(y);  // bf16 wire (C-20)
            else yt[v] = y;
          }
        }
      }
      if (!a.final_only) {
        if (U.first_tile && tid == 0) {
          int rp, rl;
          receiver_of(a, M, U.seg, U.r, rp, rl);
          float* wbox = reinterpret_cast<float*>(a.peers[rp] + a.off_wbox) + ((int64_t)par * s.n_loc + rl) * s.k;
          const float wv = s.psw[(int64_t)U.r * s.k + U.seg];
          // fused merge: the weight this worker holds after the previous step's merge
          wbox[U.seg] = a.fuse_mix ? pair_mean1(wv, __ldcg(reinterpret_cast<const float*>(mine + a.off_wbox) +
                                                           ((int64_t)(par ^ 1) * s.n_loc + U.r) * s.k + U.seg))
                                   : wv;
        }
        ptx::fence_proxy_async_shared();  // y tile -> the TMA engine's reads
      }
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive(&a_empty[st]);
        if (!a.final_only) ptx::mbar_arrive(&y_full[sy]);
      }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(s.err + kErrDiverged, 1);
  } else if (warp == kCompute / 32) {
    // ---------------- load warp: x, m, g tiles of the next units ---------------------
    if (lane == 0) {
      ptx::fence_proxy_async_global();  // acquired gbar (hierarchical) -> bulk-copy reads
      int cur = 0;
      for (int i = 0; i < n_my && !*timeout; ++i) {
        const Unit U = unit_at(a, M, u_lo + BX + i * G, cur);
        const int st = i % NS;
        ptx::mbar_wait(&a_empty[st], (uint32_t)(((i / NS) & 1) ^ 1));
        const uint32_t bytes = (uint32_t)(((U.len + 3) & ~3) * 4);
        const int64_t off = (int64_t)U.r * s.ld + U.c0;
        float* buf = ringA + (size_t)st * NA * kPeerTile;
        ptx::mbar_arrive_expect_tx(&a_full[st], 3 * bytes + (a.fuse_mix ? (s.wire ? (uint32_t)(((U.len + 7) & ~7) * 2) : bytes) : 0u));
        ptx::bulk_g2s(buf, s.x + off, bytes, &a_full[st]);
        ptx::bulk_g2s(buf + kPeerTile, s.m + off, bytes, &a_full[st]);
        bulk_load_g(s, a.peers, buf + 2 * kPeerTile, off, U.c0, bytes / 4, &a_full[st]);
        if (a.fuse_mix) {  // the previous step's received tile (inbox parity of epoch e-1)
          if (s.wire)  // bf16 rows, stride (ld + 7) & ~7, 16-byte units
            ptx::bulk_g2s(buf + 3 * kPeerTile,
                          reinterpret_cast<const uint16_t*>(mine + a.off_inbox) +
                              ((int64_t)(par ^ 1) * s.n_loc + U.r) * ((s.ld + 7) & ~7) + U.c0,
                          (uint32_t)(((U.len + 7) & ~7) * 2), &a_full[st]);
          else
            ptx::bulk_g2s(buf + 3 * kPeerTile,
                          reinterpret_cast<const float*>(mine + a.off_inbox) + (int64_t)(par ^ 1) * s.n_loc * s.ld + off,
                          bytes, &a_full[st]);
        }
      }
    }
    __syncwarp();
  } else if (!a.final_only) {
    // ---------------- store warp: y tiles -> receivers' inboxes over NVLink -----------
    if (lane == 0) {
      int cur = 0;
      for (int i = 0; i < n_my && !*timeout; ++i) {
        const Unit U = unit_at(a, M, u_lo + BX + i * G, cur);
        const int sy = i % kSlotsY;
        ptx::mbar_wait(&y_full[sy], (uint32_t)((i / kSlotsY) & 1));
        int rp, rl;
        receiver_of(a, M, U.seg, U.r, rp, rl);
        if (s.wire) {  // half the bytes: a bf16 row, rounded up to whole 16-byte units
          const int64_t ldw = (s.ld + 7) & ~7;
          uint16_t* inbox = reinterpret_cast<uint16_t*>(a.peers[rp] + a.off_inbox) +
                            ((int64_t)par * s.n_loc + rl) * ldw;
          ptx::bulk_s2g(inbox + U.c0, ringY + (size_t)sy * kPeerTile, (uint32_t)(((U.len + 7) & ~7) * 2));
        } else {
          float* inbox = reinterpret_cast<float*>(a.peers[rp] + a.off_inbox) + ((int64_t)par * s.n_loc + rl) * s.ld;
          ptx::bulk_s2g(inbox + U.c0, ringY + (size_t)sy * kPeerTile, (uint32_t)(((U.len + 3) & ~3) * 4));
        }
        ptx::bulk_commit();
        ptx::bulk_wait_read<1>();  // groups of units < i have read their tiles
        if (i >= 1) ptx::mbar_arrive(&y_empty[(i - 1) % kSlotsY]);
      }
      ptx::bulk_wait_all();  // every y tile has landed in its receiver's inbox
      ptx::fence_proxy_async_global();
      if (n_my >= 1) ptx::mbar_arrive(&y_empty[(n_my - 1) % kSlotsY]);
    }
    __syncwarp();
  }
  __syncthreads();
  if (a.fuse_mix) {
    // the last CTA: every CTA has read psw and the previous inbox.  Store the previous step's
    // merged weights, then publish this step's pushes (pdone = e) and the consumption of the
    // previous inbox (done = e - 1, the flag the senders' ping-pong wait reads)
    __shared__ int s_last;
    if (threadIdx.x == 0) {
      if (s_timeout) atomicOr(s.err + kErrTimeout, 1);
      __threadfence();
      const uint32_t prev = atomicAdd(reinterpret_cast<uint32_t*>(mine + a.off_pcount), 1u);
      s_last = prev + 1 == a.pdone_target;
    }
    __syncthreads();
    if (s_last) {
      const float* wprev = reinterpret_cast<const float*>(mine + a.off_wbox) + (int64_t)(par ^ 1) * s.n_loc * s.k;
      for (int i = threadIdx.x; i < s.n_loc * s.k; i += blockDim.x)
        s.psw[i] = pair_mean1(s.psw[i], __ldcg(wprev + i));
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence_system();
        for (int q = 0; q < s.nprocs; ++q) {
          ptx::st_release_sys(reinterpret_cast<uint32_t*>(a.peers[q] + a.off_pdone) + s.rank, e);
          ptx::st_release_sys(reinterpret_cast<uint32_t*>(a.peers[q] + a.off_done) + s.rank, e - 1);
        }
      }
    }
    return;
  }
  if (threadIdx.x == 0) {
    if (s_timeout) atomicOr(s.err + kErrTimeout, 1);
    if (a.final_only)  // nothing to exchange: this step is complete, for every piece
      publish_when_last(a.peers, mine, a.off_count, a.off_done, s.rank, 0, s.nprocs, e, a.done_target,
                        a.pieces, a.flag_stride);
    else  // every CTA's pushes have landed: publish them
      publish_when_last(a.peers, mine, a.off_pcount, a.off_pdone, s.rank, 0, s.nprocs, e, a.pdone_target);
  }
}

__global__ void __launch_bounds__(kMixThreads) k_peer_mix(const PeerKernelArgs a0) {
  PeerKernelArgs a = a0;
  const RankCta rc = rank_cta(a0.vranks, a0.s.rank);
  rank_view(a.s, a.peers, a0.vranks, rc.rank);
  const int BX = rc.b, GX = rc.G;
  const PeerStepArgs& s = a.s;
  const uint32_t e = a.epoch;
  const int par = (int)(e & 1u);
  char* mine = a.peers[s.rank];
  __shared__ int s_timeout;
  if (threadIdx.x == 0) s_timeout = 0;
  __syncthreads();
  if (threadIdx.x < s.nprocs) {
    const uint32_t* pd = reinterpret_cast<const uint32_t*>(mine + a.off_pdone);
    if (!wait_acquire(pd + threadIdx.x, e)) atomicOr(&s_timeout, 1);
  }
  __syncthreads();
  if (!s_timeout) {
    const int64_t nv = (a.col_hi - a.col_lo + 3) >> 2;
    const int64_t total = nv * s.n_loc;
    const float* inbox0 = reinterpret_cast<const float*>(mine + a.off_inbox) + (int64_t)par * s.n_loc * s.ld;
    const int64_t ldw = (s.ld + 7) & ~7;
    const uint16_t* inbox0w = reinterpret_cast<const uint16_t*>(mine + a.off_inbox) + (int64_t)par * s.n_loc * ldw;
    const int64_t stride = (int64_t)GX * blockDim.x;
    constexpr int U = 4;  // float4 pairs in flight per thread
    for (int64_t base = (int64_t)BX * blockDim.x + threadIdx.x; base < total; base += U * stride) {
      float4 yo[U], yi[U];
      int64_t off[U];
      int valid[U];
#pragma unroll
      for (int h = 0; h < U; ++h) {
        const int64_t idx = base + h * stride;
        valid[h] = 0;
        if (idx < total) {
          const int64_t r = idx / nv, v = idx - r * nv;
          const int64_t j = a.col_lo + 4 * v;
          valid[h] = (int)imin64(4, a.col_hi - j);
          off[h] = r * s.ld + j;
          yo[h] = __ldcs(reinterpret_cast<const float4*>(s.x + off[h]));
          if (s.wire)
            yi[h] = unpack_bf16x4(__ldcs(reinterpret_cast<const uint2*>(
                reinterpret_cast<const uint16_t*>(inbox0w) + r * ldw + j)));
          else
            yi[h] = __ldcs(reinterpret_cast<const float4*>(inbox0 + off[h]));
        }
      }
#pragma unroll
      for (int h = 0; h < U; ++h)
        if (valid[h] > 0) st4_cs(s.x + off[h], mean4(yo[h], yi[h]), valid[h]);
    }
    if (BX == 0) {  // weights of the segments whose first tile is in this piece
      for (int i = threadIdx.x; i < s.n_loc * s.k; i += blockDim.x) {
        const int r = i / s.k, sg = i - r * s.k;
        if (a.seg_t0[sg] < a.tile_lo || a.seg_t0[sg] >= a.tile_hi) continue;
        const float* wbox = reinterpret_cast<const float*>(mine + a.off_wbox) + ((int64_t)par * s.n_loc + r) * s.k;
        float* wp = s.psw + (int64_t)r * s.k + sg;
        *wp = __fmul_rn(__fadd_rn(*wp, __ldcg(wbox + sg)), 0.5f);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_timeout) atomicOr(s.err + kErrTimeout, 1);
    publish_when_last(a.peers, mine, a.off_count, a.off_done, s.rank, 0, s.nprocs, e, a.done_target);
  }
}

// ---------------------------------------------------------------------------
// Hierarchical h1: reduce-scatter of the gradient inside the group, then the
// fixed-order sum and all-gather of the mean.

struct HierArgs {
  const float* g;            // this GPU's worker gradient [d]
  char* const* peers;
  int64_t d, chunk;          // chunk: columns per member in this piece (multiple of 4)
  int64_t col_lo, col_hi;    // this piece's columns
  int64_t gstride;           // gbox slot stride (elements)
  int rank, gs;
  float inv_gs;
  uint32_t epoch;
  uint32_t c1_target, c2_target;  // arrival targets (see publish_when_last)
  int pull;                  // 1: the mean chunk stays in this member's gbar (the update pulls it)
  int vranks;                // > 1: emulated ranks (g is row `rank` of [vranks][ld])
  int64_t ld;
  size_t off_gbox, off_gbar, off_d1, off_c1, off_d2, off_c2;
  int* err;
};

// h1 over the columns [col_lo, col_hi) of one piece, split into gs member chunks of
// `chunk` columns (multiple of 4).  gbox slots are full rows (stride gstride), indexed by
// absolute column, so pieces need no layout of their own.
//   k_hier_scatter  member m sends chunk c of its gradient to member c's gbox slot m
//                   (reduce-scatter over NVLink).  Destinations rotate every 32 float4
//                   (512 contiguous bytes per warp), starting at this member's offset:
//                   the group's GPUs spread their stores over every peer at once instead
//                   of all writing member 0's chunk first (incast on one GPU's links).
//                   The own chunk stays in g.
//   k_hier_reduce   member c: gbar = fl(sum over members, ascending) * fp32(1/|G|) of its
//                   chunk (reading C-12), all-gathered into every member's gbar.
__global__ void __launch_bounds__(kHierThreads) k_hier_scatter(const HierArgs h0) {
  HierArgs h = h0;
  const RankCta rc = rank_cta(h0.vranks, h0.rank);
  h.rank = rc.rank;
  if (h0.vranks > 1) h.g += (int64_t)rc.rank * h0.ld;
  const int BX = rc.b, GX = rc.G;
  const int grp = h.rank / h.gs, member = h.rank - grp * h.gs, gbase = grp * h.gs;
  const int64_t cv = h.chunk / 4;
  const int64_t nblk = (cv + 31) / 32;
  const int64_t total = nblk * 32 * h.gs;
  for (int64_t idx = (int64_t)BX * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)GX * blockDim.x) {
    const int64_t b = idx >> 5;
    const int c = (int)((b + member) % h.gs);
    const int64_t v = (b / h.gs) * 32 + (idx & 31);
    if (c == member || v >= cv) continue;
    const int64_t j = h.col_lo + c * h.chunk + 4 * v;
    const int valid = (int)imin64(4, imin64(h.col_hi, h.col_lo + (c + 1) * h.chunk) - j);
    if (valid <= 0) continue;
    float* slot = reinterpret_cast<float*>(h.peers[gbase + c] + h.off_gbox) + (int64_t)member * h.gstride;
    st4(slot + j, ld4_valid(h.g + j, valid), valid);
  }
  __syncthreads();
  if (threadIdx.x == 0)
    publish_when_last(h.peers, h.peers[h.rank], h.off_c1, h.off_d1, h.rank, gbase, h.gs, h.epoch, h.c1_target);
}

__global__ void __launch_bounds__(kHierThreads) k_hier_reduce(const HierArgs h0) {
  HierArgs h = h0;
  const RankCta rc = rank_cta(h0.vranks, h0.rank);
  h.rank = rc.rank;
  if (h0.vranks > 1) h.g += (int64_t)rc.rank * h0.ld;
  const int BX = rc.b, GX = rc.G;
  const int grp = h.rank / h.gs, member = h.rank - grp * h.gs, gbase = grp * h.gs;
  char* mine = h.peers[h.rank];
  __shared__ int s_timeout;
  if (threadIdx.x == 0) s_timeout = 0;
  __syncthreads();
  if (threadIdx.x < h.gs && threadIdx.x != member) {  // the other members' chunks have arrived
    const uint32_t* d1 = reinterpret_cast<const uint32_t*>(mine + h.off_d1);
    if (!wait_acquire(d1 + gbase + threadIdx.x, h.epoch)) atomicOr(&s_timeout, 1);
  }
  __syncthreads();
  if (!s_timeout) {
    const float* gbox = reinterpret_cast<const float*>(mine + h.off_gbox);
    const int64_t c0 = h.col_lo + member * h.chunk;
    const int64_t c1 = imin64(h.col_hi, c0 + h.chunk);
    const int64_t cv = (c1 - c0 + 3) / 4;
    for (int64_t v = (int64_t)BX * blockDim.x + threadIdx.x; v < cv; v += (int64_t)GX * blockDim.x) {
      const int64_t j = c0 + 4 * v;
      const int valid = (int)imin64(4, c1 - j);
      // reading C-12: gbar = fl(...fl(g_0 + g_1)... + g_{gs-1}) * fp32(1/|G|), ascending members
      float4 acc = member == 0 ? ld4_valid(h.g + j, valid) : __ldcg(reinterpret_cast<const float4*>(gbox + j));
      for (int mm = 1; mm < h.gs; ++mm)
        acc = add4(acc, mm == member ? ld4_valid(h.g + j, valid)
                                     : __ldcg(reinterpret_cast<const float4*>(gbox + (int64_t)mm * h.gstride + j)));
      const float4 mean = scale4(acc, h.inv_gs);
      if (h.pull) {  // the members' updates read it from here
        st4(reinterpret_cast<float*>(mine + h.off_gbar) + j, mean, valid);
        continue;
      }
      for (int q = 0; q < h.gs; ++q) {  // rotated start: spread the all-gather over every peer
        const int mm = (q + member + (int)(v >> 5)) % h.gs;
        st4(reinterpret_cast<float*>(h.peers[gbase + mm] + h.off_gbar) + j, mean, valid);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_timeout) atomicOr(h.err + kErrTimeout, 1);
    publish_when_last(h.peers, mine, h.off_c2, h.off_d2, h.rank, gbase, h.gs, h.epoch, h.c2_target);
  }
}

// Replica sync (first hierarchical step after bind / set_step): the leader copies its
// x, m and psw into every member's sync buffers and publishes d3; members wait for it
// and take the copy.  Afterwards the members are exact replicas of their leader, which
// is what "the gossiped model parameter of the leader node propagates to other
// workers" leaves them as after every step.
struct SyncArgs {
  HierArgs h;
  float* x;
  float* m;
  float* psw;
  int64_t ld;
  int k;
  uint32_t c3_target;
  size_t off_xsync, off_msync, off_wsync, off_d3, off_c3;
};

__global__ void __launch_bounds__(kHierThreads) k_hier_sync(const SyncArgs sa0) {
  SyncArgs sa = sa0;
  const RankCta rc = rank_cta(sa0.h.vranks, sa0.h.rank);
  sa.h.rank = rc.rank;
  if (sa0.h.vranks > 1) {
    sa.x += (int64_t)rc.rank * sa0.ld;
    sa.m += (int64_t)rc.rank * sa0.ld;
    sa.psw += (int64_t)rc.rank * sa0.k;
  }
  const HierArgs& h = sa.h;
  const int BX = rc.b, GX = rc.G;
  const int grp = h.rank / h.gs, member = h.rank - grp * h.gs, gbase = grp * h.gs;
  char* mine = h.peers[h.rank];
  const int64_t nv = (h.d + 3) / 4;
  const int64_t stride = (int64_t)GX * blockDim.x;
  if (member == 0) {
    for (int c = 1; c < h.gs; ++c) {
      char* dst = h.peers[gbase + c];
      for (int64_t v = (int64_t)BX * blockDim.x + threadIdx.x; v < nv; v += stride) {
        const int64_t j = 4 * v;
        const int valid = (int)imin64(4, h.d - j);
        st4(reinterpret_cast<float*>(dst + sa.off_xsync) + j, ld4_valid(sa.x + j, valid), valid);
        st4(reinterpret_cast<float*>(dst + sa.off_msync) + j, ld4_valid(sa.m + j, valid), valid);
      }
      if (BX == 0)
        for (int s = threadIdx.x; s < sa.k; s += blockDim.x)
          reinterpret_cast<float*>(dst + sa.off_wsync)[s] = sa.psw[s];
    }
    __syncthreads();
    if (threadIdx.x == 0)
      publish_when_last(h.peers, mine, sa.off_c3, sa.off_d3, h.rank, gbase, h.gs, h.epoch, sa.c3_target);
  } else {
    __shared__ int s_timeout;
    if (threadIdx.x == 0) {
      s_timeout = 0;
      if (!wait_acquire(reinterpret_cast<const uint32_t*>(mine + sa.off_d3) + gbase, h.epoch)) s_timeout = 1;
    }
    __syncthreads();
    if (s_timeout) {
      if (threadIdx.x == 0) atomicOr(h.err + kErrTimeout, 1);
      return;
    }
    for (int64_t v = (int64_t)BX * blockDim.x + threadIdx.x; v < nv; v += stride) {
      const int64_t j = 4 * v;
      const int valid = (int)imin64(4, h.d - j);
      st4(sa.x + j, ld4_valid(reinterpret_cast<const float*>(mine + sa.off_xsync) + j, valid), valid);
      st4(sa.m + j, ld4_valid(reinterpret_cast<const float*>(mine + sa.off_msync) + j, valid), valid);
    }
    if (BX == 0)
      for (int s = threadIdx.x; s < sa.k; s += blockDim.x)
        sa.psw[s] = __ldcg(reinterpret_cast<const float*>(mine + sa.off_wsync) + s);
  }
}

// ---------------------------------------------------------------------------
// Hybrid flat step for several workers per GPU (configs 2 at N > 1 and 5).
//
// Restricted to this GPU's workers, each segment's permutation splits into local
// cycles and local chains c0 -> c1 = src(c0) -> ... -> cm, where dst(c0) and
// src(cm) are on other GPUs.  k_hyb_walk is the single-GPU bulk-TMA cycle walk
// (k_gossip_tma) over that structure: cycles are mixed in registers as on one
// GPU; a chain's head additionally stores its y into the inbox of dst(c0) over
// NVLink, and a chain's tail keeps its y in x.  k_hyb_tail then finishes only
// the tails, x = (y + inbox) * 0.5, once every GPU's heads have landed.  HBM
// per parameter: 20 B + 16 B x (fraction of remote-sourced workers), against
// 36 B for the push/mix pair.
constexpr int kHCons = 256;
constexpr int kHThreads = kHCons + 32;
constexpr int kHVPT = kTmaTileMax / (4 * kHCons);
constexpr int kHStages = 4;
constexpr size_t kHStageBytes = 3ull * kTmaTileMax * sizeof(float);
constexpr uint32_t kHStart = 1u << 31, kHEnd = 1u << 30, kHHead = 1u << 29, kHTail = 1u << 28;
constexpr uint32_t kHIdx = (1u << 28) - 1;
constexpr int kHMaxTable = 2048;  // k * n_loc

size_t hyb_smem_bytes(int k, int n_loc) {
  return kHStages * kHStageBytes + sizeof(uint32_t) * 2 * (size_t)k * n_loc +
         sizeof(uint32_t) * 192 * (kHThreads / 32) + sizeof(float) * (size_t)k * n_loc + (size_t)k * n_loc +
         16 + sizeof(float) * kHStages;  // + per-slot LARS rates (4-byte aligned)
}

struct HybArgs {
  float* x;
  float* m;
  const float* g;
  float* psw;
  int64_t ld, d, nq;
  int k, world, n_loc, first, rank, nprocs;
  uint64_t seed;
  uint32_t step;
  const int32_t* given;     // injected topology [k][world] or nullptr
  const int32_t* src_tbl;   // k_topology output [k][world] when !fused
  int fused;
  float lr, mu;
  const TileDesc* tiles;
  int n_tiles;
  char* const* peers;
  size_t off_inbox, off_wbox, off_done, off_pdone, off_count, off_pcount, flag_stride;
  int pieces;
  uint32_t epoch, pdone_target, done_target;
  uint8_t* tail_tbl;        // [k][n_loc]: 1 = the worker's segment source is remote
  int* err;
  int wire;                 // bf16 wire format (reading C-20)
  // deferred merge: the previous step's chain tails (tail_prev, its [k][n_loc] table) are
  // merged with the previous inbox inside this walk, and this step's tails wait for the next
  int fuse;
  const uint8_t* tail_prev;
  // LARS (reading C-18): per-(local worker, layer) rates staged per ring slot; weight decay
  const float* lrs;
  int n_layers;
  float wd;
  const int64_t* bounds;    // [k+1] the segment plan (layer plans move the bounds)
  int vranks;               // > 1: emulated ranks (rows rank*n_loc.. of [vranks*n_loc][ld])
  size_t tbl_stride;        // tail-table bytes per emulated rank
};

// Rank `rank`'s view of hybrid-walk arguments given for rank 0 of an emulated launch.
__device__ __forceinline__ void hyb_view(HybArgs& a, int rank) {
  if (a.vranks <= 1) return;
  const int64_t rows = (int64_t)rank * a.n_loc;
  a.rank = rank;
  a.first = rank * a.n_loc;
  if (a.lrs) a.lrs += rows * a.n_layers;  // (x, m, g, psw: the kernels' own locals)
  if (a.tail_tbl) a.tail_tbl += (size_t)rank * a.tbl_stride;
  if (a.tail_prev) a.tail_prev += (size_t)rank * a.tbl_stride;
}

__global__ void __launch_bounds__(kHThreads, 2) k_hyb_walk(const HybArgs a0) {
  HybArgs a = a0;
  const RankCta rc = rank_cta(a0.vranks, a0.rank);
  hyb_view(a, rc.rank);
  // the rank's rows, computed from the launch arguments (the body uses these locals)
  const int64_t vrows = a0.vranks > 1 ? (int64_t)rc.rank * a0.n_loc : 0;
  float* const aX = a0.x + vrows * a0.ld;
  float* const aM = a0.m + vrows * a0.ld;
  const float* const aG = a0.g + vrows * a0.ld;
  float* const aPSW = a0.psw + vrows * a0.k;
  (void)aM;
  (void)aG;
  const int BX = rc.b, GX = rc.G;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stage_buf = reinterpret_cast<float*>(smem_raw);
  uint32_t* ord = reinterpret_cast<uint32_t*>(smem_raw + kHStages * kHStageBytes);  // [k][n_loc]
  int32_t* head_dst = reinterpret_cast<int32_t*>(ord + a.k * a.n_loc);             // [k][n_loc]
  uint32_t* scratch = reinterpret_cast<uint32_t*>(head_dst + a.k * a.n_loc);         // [warps][192]
  float* cur_w = reinterpret_cast<float*>(scratch + 192 * (kHThreads / 32));         // [k][n_loc]
  uint8_t* tprev = reinterpret_cast<uint8_t*>(cur_w + a.k * a.n_loc);               // [k][n_loc]
  float* srate = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(tprev + a.k * a.n_loc) + 15) & ~uintptr_t(15));
  // deferred merge: 3 stages of x, m, g and the previous inbox tile (the same 12-tile region)
  const int NS = a.fuse ? 3 : kHStages, NA = a.fuse ? 4 : 3;
  __shared__ uint64_t full[kHStages], empty[kHStages];
  __shared__ int s_timeout;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_loc = a.n_loc, first = a.first;
  const int par = (int)(a.epoch & 1u);
  char* mine = a.peers[a.rank];
  volatile int* timeout = &s_timeout;

  if (threadIdx.x == 0) {
    s_timeout = 0;
    for (int s = 0; s < kHStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], kHCons / 32);
    }
    ptx::mbar_fence_init();
  }
  // ---- this step's topology, restricted to this GPU's workers (Alg. 2)
  {
    uint32_t* u = scratch + warp * 192;
    int32_t* srow = reinterpret_cast<int32_t*>(u + 64);   // [<= 64] when fused
    int32_t* dstl = reinterpret_cast<int32_t*>(u + 128);  // [n_loc] dst of local workers
    const int nw = blockDim.x >> 5;
    for (int sg = warp; sg < a.k; sg += nw) {
      const int32_t* row;
      if (a.given != nullptr) {
        row = a.given + (int64_t)sg * a.world;
      } else if (a.fused) {
        warp_alg2_small(a.seed, a.step, sg, a.world, CS_TAG_FLAT, u, srow, a.err);
        row = srow;
      } else {
        row = a.src_tbl + (int64_t)sg * a.world;
      }
      __syncwarp();
      for (int jj = lane; jj < a.world; jj += 32) {  // inverse on the local range: dst
        const int v = row[jj];
        if (v >= first && v < first + n_loc) dstl[v - first] = jj;
      }
      __syncwarp();
      if (lane == 0) {
        uint32_t* o = ord + sg * n_loc;
        uint64_t seen = 0;
        int pos = 0;
        for (int r = 0; r < n_loc; ++r) {  // chains start where the receiver is remote
          const int dg = dstl[r];
          if (dg >= first && dg < first + n_loc) continue;
          head_dst[sg * n_loc + r] = dg;
          int pr = r;
          uint32_t flag = kHStart | kHHead;
          while (true) {
            seen |= 1ull << pr;
            const int sgl = row[first + pr] - first;
            if (sgl < 0 || sgl >= n_loc) {  // source remote: chain tail
              o[pos++] = (uint32_t)pr | flag | kHEnd | kHTail;
              break;
            }
            o[pos++] = (uint32_t)pr | flag;
            flag = 0;
            pr = sgl;
          }
        }
        for (int r0 = 0; r0 < n_loc; ++r0) {  // the rest: cycles of local workers
          if ((seen >> r0) & 1ull) continue;
          int pr = r0;
          uint32_t flag = kHStart;
          do {
            seen |= 1ull << pr;
            const int nx = row[first + pr] - first;
            o[pos++] = (uint32_t)pr | flag | (nx == r0 ? kHEnd : 0u);
            flag = 0;
            pr = nx;
          } while (pr != r0);
        }
      }
      if (BX == 0)
        for (int r = lane; r < n_loc; r += 32) {
          const int sgl = row[first + r] - first;
          a.tail_tbl[sg * n_loc + r] = (sgl < 0 || sgl >= n_loc) ? 1 : 0;
        }
      __syncwarp();
    }
  }
  __syncthreads();
  // ping-pong safety: every GPU finished its mix of epoch e-2 (last reader of this inbox parity)
  if (threadIdx.x < a.nprocs && a.epoch >= 3) {
    const uint32_t* done = reinterpret_cast<const uint32_t*>(mine + a.off_done);
    if (!wait_acquire(done + threadIdx.x, a.epoch - 2)) atomicOr(&s_timeout, 1);
  }
  __syncthreads();
  // the weights each worker holds now: after the previous step's deferred tail merges
  if (a.fuse && threadIdx.x < a.nprocs) {  // every GPU's pushes of epoch e-1 have landed here
    const uint32_t* pd = reinterpret_cast<const uint32_t*>(mine + a.off_pdone);
    if (!wait_acquire(pd + threadIdx.x, a.epoch - 1)) atomicOr(&s_timeout, 1);
  }
  __syncthreads();
  ptx::fence_proxy_async_global();  // the acquired inbox tiles -> the producer's bulk copies
  for (int i = threadIdx.x; i < a.k * n_loc; i += blockDim.x) {
    const int sg = i / n_loc, r = i - sg * n_loc;
    const uint8_t tp = a.fuse ? a.tail_prev[i] : 0;
    const float w = aPSW[(int64_t)r * a.k + sg];
    tprev[i] = tp;
    cur_w[i] = tp ? pair_mean1(w, __ldcg(reinterpret_cast<const float*>(mine + a.off_wbox) +
                                         ((int64_t)(par ^ 1) * n_loc + r) * a.k + sg))
                  : w;
  }
  __syncthreads();
  // push-sum weights of the chain heads go with their y (reading C-11)
  if (BX == 0 && !*timeout)
    for (int i = threadIdx.x; i < a.k * n_loc; i += blockDim.x) {
      const int sg = i / n_loc, r = i - sg * n_loc;
      const int dg = head_dst[sg * n_loc + r];
      const uint32_t* o = ord + sg * n_loc;
      bool head = false;
      for (int pp = 0; pp < n_loc; ++pp)
        if ((o[pp] & kHIdx) == (uint32_t)r && (o[pp] & kHHead)) head = true;
      if (!head) continue;
      const int rp = dg / n_loc, rl = dg - rp * n_loc;
      reinterpret_cast<float*>(a.peers[rp] + a.off_wbox)[((int64_t)par * n_loc + rl) * a.k + sg] = cur_w[i];
    }

  const int64_t ld = a.ld;
  if (warp == kHCons / 32) {
    // ---------------- producer: rows of each tile in walk order ------------------
    if (lane == 0) {
      uint32_t it = 0;
      for (int t = BX; t < a.n_tiles && !*timeout; t += GX) {
        const TileDesc td = a.tiles[t];
        const uint32_t bytes = (uint32_t)(((td.len + 3) & ~3) * sizeof(float));
        const uint32_t* o = ord + td.seg * n_loc;
        for (int p = 0; p < n_loc; ++p, ++it) {
          const int st = (int)(it % NS);
          ptx::mbar_wait(&empty[st], ((it / NS) & 1u) ^ 1u);
          const uint32_t row = o[p] & kHIdx;
          const int64_t off = (int64_t)row * ld + td.c0;
          float* buf = stage_buf + (size_t)st * NA * kTmaTileMax;
          const bool merge = tprev[td.seg * n_loc + row];
          const uint32_t ibytes = a.wire ? (uint32_t)(((td.len + 7) & ~7) * 2) : bytes;
          if (a.lrs) srate[st] = a.lrs[(int64_t)row * a.n_layers + td.layer];  // before the release-arrive
          ptx::mbar_arrive_expect_tx(&full[st], 3 * bytes + (merge ? ibytes : 0u));
          ptx::bulk_g2s(buf, aX + off, bytes, &full[st]);
          ptx::bulk_g2s(buf + kTmaTileMax, aM + off, bytes, &full[st]);
          ptx::bulk_g2s(buf + 2 * kTmaTileMax, aG + off, bytes, &full[st]);
          if (merge && a.wire)  // the previous step's received y of this tail row (bf16 rows)
            ptx::bulk_g2s(buf + 3 * kTmaTileMax,
                          reinterpret_cast<const uint16_t*>(mine + a.off_inbox) +
                              ((int64_t)(par ^ 1) * n_loc + row) * ((ld + 7) & ~7) + td.c0,
                          ibytes, &full[st]);
          else if (merge)
            ptx::bulk_g2s(buf + 3 * kTmaTileMax,
                          reinterpret_cast<const float*>(mine + a.off_inbox) + ((int64_t)(par ^ 1) * n_loc) * ld + off,
                          bytes, &full[st]);
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- consumers: the walk, heads pushed over NVLink, tails kept ------
    bool bad = false;
    uint32_t it = 0;
    for (int t = BX; t < a.n_tiles && !*timeout; t += GX) {
      const TileDesc td = a.tiles[t];
      const uint32_t* o = ord + td.seg * n_loc;
      float4 yfirst[kHVPT], yprev[kHVPT];
      uint32_t prev_row = 0;
      for (int p = 0; p < n_loc; ++p, ++it) {
        const int st = (int)(it % NS);
        ptx::mbar_wait(&full[st], (it / NS) & 1u);
        const float* buf = stage_buf + (size_t)st * NA * kTmaTileMax;
        const uint32_t e = o[p];
        const uint32_t row = e & kHIdx;
        const bool merge = tprev[td.seg * n_loc + row];
        float* inbox = nullptr;
        uint16_t* inboxw = nullptr;
        if (e & kHHead) {
          const int dg = head_dst[td.seg * n_loc + row];
          const int rp = dg / n_loc, rl = dg - rp * n_loc;
          inbox = reinterpret_cast<float*>(a.peers[rp] + a.off_inbox) + ((int64_t)par * n_loc + rl) * ld;
          inboxw = reinterpret_cast<uint16_t*>(a.peers[rp] + a.off_inbox) +
                   ((int64_t)par * n_loc + rl) * ((ld + 7) & ~7);
        }
#pragma unroll
        for (int c = 0; c < kHVPT; ++c) {
          const int v = c * kHCons + threadIdx.x;
          const int valid = td.len - 4 * v;
          if (valid > 0) {
            const int vv = valid < 4 ? valid : 4;
            float4 cx = reinterpret_cast<const float4*>(buf)[v];
            const float4 cm = reinterpret_cast<const float4*>(buf + kTmaTileMax)[v];
            const float4 cg = reinterpret_cast<const float4*>(buf + 2 * kTmaTileMax)[v];
            if (merge)  // the previous step's a5 for this chain tail (Alg.1 l.17)
              cx = mean4(cx, a.wire ? unpack_bf16x4(reinterpret_cast<const uint2*>(buf + 3 * kTmaTileMax)[v])
                                    : reinterpret_cast<const float4*>(buf + 3 * kTmaTileMax)[v]);
            bad |= nonfinite4(cg);
            // LARS (C-18): m' = mu*m + (g + wd*x), y = x - lrs[row][layer]*m'
            const float4 mn = mom4(cm, a.lrs ? decay4(cg, cx, a.wd) : cg, a.mu);
            const float4 y = sgd4(cx, mn, a.lrs ? srate[st] : a.lr);
            const int64_t j = td.c0 + 4 * v;
            st4_cs(aM + (int64_t)row * ld + j, mn, vv);
            if (e & kHStart) {
              yfirst[c] = y;
              if (e & kHHead) {  // NVLink push of the chain head
                if (a.wire) *reinterpret_cast<uint2*>(inboxw + j) = pack_bf16x4(y);
                else st4(inbox + j, y, vv);
              }
            } else {
              st4_cs(aX + (int64_t)prev_row * ld + j, mean4(yprev[c], a.wire ? bf16r4(y) : y), vv);
            }
            if (e & kHEnd) {
              if (e & kHTail) st4(aX + (int64_t)row * ld + j, y, vv);  // finished by k_hyb_tail
              else st4_cs(aX + (int64_t)row * ld + j, mean4(y, a.wire ? bf16r4(yfirst[c]) : yfirst[c]), vv);
            }
            yprev[c] = y;
          }
        }
        prev_row = row;
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&empty[st]);
      }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.err + kErrDiverged, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_timeout) atomicOr(a.err + kErrTimeout, 1);
    __threadfence_system();  // this CTA's NVLink stores before its arrival
    uint32_t* cnt = reinterpret_cast<uint32_t*>(mine + a.off_pcount);
    const uint32_t prev = atomicAdd(cnt, 1u);
    s_timeout = (prev + 1 == a.pdone_target) ? 2 : 0;  // reuse as "last CTA" marker
  }
  __syncthreads();
  if (s_timeout == 2) {
    // last CTA: weights of the workers whose source is local (snapshot: nothing wrote psw yet)
    for (int i = threadIdx.x; i < a.k * n_loc; i += blockDim.x) {
      const int sg = i / n_loc, r = i - sg * n_loc;
      if (a.tail_tbl[sg * n_loc + r]) continue;
      // the local source: the ord entry after r in its cycle (or chain)
      const uint32_t* o = ord + sg * n_loc;
      int pos = 0;
      while ((o[pos] & kHIdx) != (uint32_t)r) ++pos;
      int srcl;
      if (o[pos] & kHEnd) {  // cycle end: closes with its start
        int q = pos;
        while (!(o[q] & kHStart)) --q;
        srcl = (int)(o[q] & kHIdx);
      } else {
        srcl = (int)(o[pos + 1] & kHIdx);
      }
      reinterpret_cast<float*>(stage_buf)[i] = pair_mean1(cur_w[i], cur_w[sg * n_loc + srcl]);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < a.k * n_loc; i += blockDim.x) {
      const int sg = i / n_loc, r = i - sg * n_loc;
      // tails of this step keep their current weight; their merge comes with the next step
      aPSW[(int64_t)r * a.k + sg] = a.tail_tbl[sg * n_loc + r] ? cur_w[i] : reinterpret_cast<const float*>(stage_buf)[i];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      for (int p = 0; p < a.nprocs; ++p) {
        ptx::st_release_sys(reinterpret_cast<uint32_t*>(a.peers[p] + a.off_pdone) + a.rank, a.epoch);
        if (a.fuse)  // the previous inbox is consumed
          ptx::st_release_sys(reinterpret_cast<uint32_t*>(a.peers[p] + a.off_done) + a.rank, a.epoch - 1);
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_hyb_tail(const HybArgs a0) {
  HybArgs a = a0;
  const RankCta rc = rank_cta(a0.vranks, a0.rank);
  hyb_view(a, rc.rank);
  // the rank's rows, computed from the launch arguments (the body uses these locals)
  const int64_t vrows = a0.vranks > 1 ? (int64_t)rc.rank * a0.n_loc : 0;
  float* const aX = a0.x + vrows * a0.ld;
  float* const aM = a0.m + vrows * a0.ld;
  const float* const aG = a0.g + vrows * a0.ld;
  float* const aPSW = a0.psw + vrows * a0.k;
  (void)aM;
  (void)aG;
  const int BX = rc.b, GX = rc.G;
  __shared__ uint8_t tail[kHMaxTable];
  __shared__ int s_timeout;
  char* mine = a.peers[a.rank];
  const int par = (int)(a.epoch & 1u);
  const int n_loc = a.n_loc;
  if (threadIdx.x == 0) s_timeout = 0;
  for (int i = threadIdx.x; i < a.k * n_loc; i += blockDim.x) tail[i] = a.tail_tbl[i];
  __syncthreads();
  if (threadIdx.x < a.nprocs) {  // every GPU's chain heads have landed
    const uint32_t* pd = reinterpret_cast<const uint32_t*>(mine + a.off_pdone);
    if (!wait_acquire(pd + threadIdx.x, a.epoch)) atomicOr(&s_timeout, 1);
  }
  __syncthreads();
  if (!s_timeout) {
    const int64_t nv = (a.d + 3) >> 2;
    const int64_t total = nv * n_loc;
    const float* inbox0 = a.wire
        ? reinterpret_cast<const float*>(reinterpret_cast<const uint16_t*>(mine + a.off_inbox) +
                                         (int64_t)par * n_loc * ((a.ld + 7) & ~7))
        : reinterpret_cast<const float*>(mine + a.off_inbox) + (int64_t)par * n_loc * a.ld;
    for (int64_t idx = (int64_t)BX * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)GX * blockDim.x) {
      const int64_t r = idx / nv, v = idx - r * nv;
      const int64_t j = 4 * v;
      int sg = 0;  // segment of column j: the last plan bound <= j
      for (int lo = 0, hi = a.k - 1; lo <= hi;) {
        const int mid = (lo + hi) >> 1;
        if (a.bounds[mid] <= j) { sg = mid; lo = mid + 1; } else { hi = mid - 1; }
      }
      if (!tail[sg * n_loc + r]) continue;
      const int64_t off = r * a.ld + j;
      const float4 y = __ldcs(reinterpret_cast<const float4*>(aX + off));
      const float4 yi = a.wire ? unpack_bf16x4(__ldcs(reinterpret_cast<const uint2*>(
                                     reinterpret_cast<const uint16_t*>(inbox0) + r * ((a.ld + 7) & ~7) + j)))
                               : __ldcs(reinterpret_cast<const float4*>(inbox0 + off));
      st4_cs(aX + off, mean4(y, yi), (int)imin64(4, a.d - j));
    }
    if (BX == 0)
      for (int i = threadIdx.x; i < a.k * n_loc; i += blockDim.x) {
        const int sg = i / n_loc, r = i - sg * n_loc;
        if (!tail[i]) continue;
        const float* wbox = reinterpret_cast<const float*>(mine + a.off_wbox) + ((int64_t)par * n_loc + r) * a.k;
        float* wp = aPSW + (int64_t)r * a.k + sg;
        *wp = pair_mean1(*wp, __ldcg(wbox + sg));
      }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_timeout) atomicOr(a.err + kErrTimeout, 1);
    publish_when_last(a.peers, mine, a.off_count, a.off_done, a.rank, 0, a.nprocs, a.epoch, a.done_target,
                      a.pieces, a.flag_stride);
  }
}

// ---------------------------------------------------------------------------
// Multi-GPU diagnostics (reading B-3).  GPU q owns columns
// [q*chunk, (q+1)*chunk).  k_diag_scatter sends every local worker's x' of each
// chunk, and its psw row, to the chunk's owner; k_diag_reduce computes the same
// shifted fp64 column sums as the single-GPU kernels over all n workers of its
// chunk and publishes its partial (sum_j sum_i (z - zbar)^2, sum_j zbar) to every
// GPU; k_diag_final adds the partials in rank order (deterministic).
struct DiagArgs {
  const float* x;
  const float* psw;
  char* const* peers;
  int64_t ld, d, nq, chunk;
  const int64_t* bounds;  // [k+1] segment bounds (the plan in use)
  int k, world, n_loc, first, rank, nprocs;
  uint32_t epoch;  // diagnostics epoch (>= 1)
  uint32_t c1_target, c2_target;
  size_t off_dx, off_dw, off_dpart, off_dd1, off_dd2, off_dc1, off_dc2;
  double* partials;  // [gridDim.x][2] scratch of k_diag_reduce
  double* out;       // [2] {CD, mean checksum}
  int* err;
  int vranks;        // > 1: emulated ranks (x, psw: rows rank*n_loc.. of the whole-world buffers)
};

__device__ __forceinline__ void diag_view(DiagArgs& a, int rank, int G) {
  if (a.vranks <= 1) return;
  const int64_t rows = (int64_t)rank * a.n_loc;
  a.rank = rank;
  a.first = rank * a.n_loc;
  (void)rows;  // x, psw: k_diag_scatter's own locals
  a.partials += (size_t)2 * rank * G;
}

__global__ void __launch_bounds__(256) k_diag_scatter(const DiagArgs a0) {
  DiagArgs a = a0;
  const RankCta rc = rank_cta(a0.vranks, a0.rank);
  diag_view(a, rc.rank, rc.G);
  const int BX = rc.b, GX = rc.G;
  const int64_t vrows = a0.vranks > 1 ? (int64_t)rc.rank * a0.n_loc : 0;
  const float* const aX = a0.x + vrows * a0.ld;      // the rank's rows (locals, as in k_hyb_walk)
  const float* const aPSW = a0.psw + vrows * a0.k;
  char* mine = a.peers[a.rank];
  __shared__ int s_timeout;
  if (threadIdx.x == 0) s_timeout = 0;
  __syncthreads();
  // the owners finished reducing the previous diagnostics (their dx is free again)
  if (threadIdx.x < a.nprocs && a.epoch >= 2) {
    const uint32_t* dd2 = reinterpret_cast<const uint32_t*>(mine + a.off_dd2);
    if (!wait_acquire(dd2 + threadIdx.x, a.epoch - 1)) atomicOr(&s_timeout, 1);
  }
  __syncthreads();
  if (!s_timeout) {
    const int64_t cv = a.chunk / 4;
    const int64_t total = (int64_t)a.nprocs * a.n_loc * cv;
    for (int64_t idx = (int64_t)BX * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)GX * blockDim.x) {
      const int q = (int)(idx / ((int64_t)a.n_loc * cv));
      const int64_t rem = idx - (int64_t)q * a.n_loc * cv;
      const int r = (int)(rem / cv);
      const int64_t v = rem - (int64_t)r * cv;
      const int64_t j = q * a.chunk + 4 * v;
      const int valid = (int)imin64(4, a.d - j);
      if (valid <= 0) continue;
      float* dst = reinterpret_cast<float*>(a.peers[q] + a.off_dx) + (int64_t)(a.first + r) * a.chunk + 4 * v;
      st4(dst, ld4_valid(aX + (int64_t)r * a.ld + j, valid), valid);
    }
    if (BX == 0)
      for (int i = threadIdx.x; i < a.nprocs * a.n_loc * a.k; i += blockDim.x) {
        const int q = i / (a.n_loc * a.k), rem = i - q * a.n_loc * a.k;
        const int r = rem / a.k, s = rem - r * a.k;
        reinterpret_cast<float*>(a.peers[q] + a.off_dw)[(int64_t)(a.first + r) * a.k + s] = aPSW[(int64_t)r * a.k + s];
      }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_timeout) atomicOr(a.err + kErrTimeout, 1);
    __threadfence_system();
    publish_when_last(a.peers, mine, a.off_dc1, a.off_dd1, a.rank, 0, a.nprocs, a.epoch, a.c1_target);
  }
}

__global__ void __launch_bounds__(256) k_diag_reduce(const DiagArgs a0) {
  DiagArgs a = a0;
  const RankCta rc = rank_cta(a0.vranks, a0.rank);
  diag_view(a, rc.rank, rc.G);
  const int BX = rc.b, GX = rc.G;
  extern __shared__ double wsum[];  // [k]: 1 / sum_i w_{i,s}
  __shared__ int s_timeout;
  __shared__ double red[2][8];
  char* mine = a.peers[a.rank];
  if (threadIdx.x == 0) s_timeout = 0;
  __syncthreads();
  if (threadIdx.x < a.nprocs) {  // every GPU's columns of this chunk have arrived
    const uint32_t* dd1 = reinterpret_cast<const uint32_t*>(mine + a.off_dd1);
    if (!wait_acquire(dd1 + threadIdx.x, a.epoch)) atomicOr(&s_timeout, 1);
  }
  __syncthreads();
  const float* dx = reinterpret_cast<const float*>(mine + a.off_dx);
  const float* dw = reinterpret_cast<const float*>(mine + a.off_dw);
  for (int s = threadIdx.x; s < a.k; s += blockDim.x) {
    double sum = 0.0;
    for (int i = 0; i < a.world; ++i) sum += (double)__ldcg(dw + (int64_t)i * a.k + s);
    wsum[s] = 1.0 / sum;
  }
  __syncthreads();
  double dacc = 0.0, zacc = 0.0;
  if (!s_timeout) {
    const int64_t c0 = (int64_t)a.rank * a.chunk;
    const int64_t cols = imin64(a.chunk, a.d - c0);
    for (int64_t jj = (int64_t)BX * blockDim.x + threadIdx.x; jj < cols;
         jj += (int64_t)GX * blockDim.x) {
      const int64_t j = c0 + jj;
      int s = 0;  // segment of column j: the last bound <= j (binary search over the plan)
      for (int lo = 0, hi = a.k - 1; lo <= hi;) {
        const int mid = (lo + hi) >> 1;
        if (a.bounds[mid] <= j) { s = mid; lo = mid + 1; } else { hi = mid - 1; }
      }
      double c = 0.0, s1 = 0.0, s2 = 0.0, xs = 0.0;
      for (int i = 0; i < a.world; ++i) {
        const double xv = (double)__ldcg(dx + (int64_t)i * a.chunk + jj);
        const double z = xv / (double)__ldcg(dw + (int64_t)i * a.k + s);
        if (i == 0) c = z;
        const double dz = z - c;
        s1 += dz;
        s2 += dz * dz;
        xs += xv;
      }
      const double zbar = xs * wsum[s];
      const double dm = zbar - c;
      dacc += s2 - 2.0 * dm * s1 + (double)a.world * dm * dm;
      zacc += zbar;
    }
  }
  // fixed-order block reduction -> per-block partial; the last CTA adds them in order
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    dacc += __shfl_xor_sync(0xffffffffu, dacc, off);
    zacc += __shfl_xor_sync(0xffffffffu, zacc, off);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { red[0][warp] = dacc; red[1][warp] = zacc; }
  __syncthreads();
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    double da = 0.0, za = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { da += red[0][w]; za += red[1][w]; }
    a.partials[2 * BX] = da;
    a.partials[2 * BX + 1] = za;
    __threadfence();
    uint32_t* cnt = reinterpret_cast<uint32_t*>(mine + a.off_dc2);
    s_last = (atomicAdd(cnt, 1u) + 1 == a.c2_target);
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    double da = 0.0, za = 0.0;
    for (int b = 0; b < (int)GX; ++b) {
      da += __ldcg(a.partials + 2 * b);
      za += __ldcg(a.partials + 2 * b + 1);
    }
    for (int q = 0; q < a.nprocs; ++q) {
      double* dp = reinterpret_cast<double*>(a.peers[q] + a.off_dpart) + 2 * a.rank;
      dp[0] = da;
      dp[1] = za;
    }
    if (s_timeout) atomicOr(a.err + kErrTimeout, 1);
    __threadfence_system();
    for (int q = 0; q < a.nprocs; ++q)
      ptx::st_release_sys(reinterpret_cast<uint32_t*>(a.peers[q] + a.off_dd2) + a.rank, a.epoch);
  }
}

__global__ void k_diag_final(const DiagArgs a0) {
  DiagArgs a = a0;
  const RankCta rc = rank_cta(a0.vranks, a0.rank);
  diag_view(a, rc.rank, rc.G);
  char* mine = a.peers[a.rank];
  if (threadIdx.x != 0) return;
  for (int q = 0; q < a.nprocs; ++q)
    if (!wait_acquire(reinterpret_cast<const uint32_t*>(mine + a.off_dd2) + q, a.epoch)) {
      atomicOr(a.err + kErrTimeout, 1);
      return;
    }
  double da = 0.0, za = 0.0;
  const double* dp = reinterpret_cast<const double*>(mine + a.off_dpart);
  for (int q = 0; q < a.nprocs; ++q) {
    da += __ldcg(dp + 2 * q);
    za += __ldcg(dp + 2 * q + 1);
  }
  a.out[0] = sqrt(fmax(da, 0.0) / (double)a.world);
  a.out[1] = za;
}

// Launch `fn(arg)` with `grid` CTAs per rank: a plain launch for a real rank, one
// cooperative launch over every emulated rank otherwise (peer_launch).
template <typename Arg>
void plaunch(const PeerState& p, void (*fn)(Arg), int grid, int threads, size_t smem, cudaStream_t st, Arg arg) {
  ++g_peer_launches;
  void* args[] = {&arg};
  peer_launch(p, reinterpret_cast<const void*>(fn), grid, threads, smem, st, args);
}

}  // namespace

const char* peer_error() { return g_peer_err.c_str(); }

int peer_diag(PeerState& p, const PeerStepArgs& a, double* partials, int partials_cap, double* out,
              cudaStream_t st) {
  DiagArgs da;
  da.x = a.x;
  da.psw = a.psw;
  da.peers = p.d_peer_base;
  da.ld = a.ld;
  da.d = a.d;
  da.nq = a.nq;
  da.bounds = p.d_bounds;
  da.chunk = p.diag_chunk;
  da.k = a.k;
  da.world = a.world;
  da.n_loc = a.n_loc;
  da.first = a.first;
  da.rank = a.rank;
  da.nprocs = a.nprocs;
  da.epoch = ++p.diag_epoch;
  da.off_dx = p.off_dx;
  da.off_dw = p.off_dw;
  da.off_dpart = p.off_dpart;
  da.off_dd1 = p.off_dd1;
  da.off_dd2 = p.off_dd2;
  da.off_dc1 = p.off_dc1;
  da.off_dc2 = p.off_dc2;
  da.partials = partials;
  da.out = out;
  da.err = a.err;
  da.vranks = p.vranks;
  partials_cap /= p.vranks;
  const int64_t sv = (int64_t)a.nprocs * a.n_loc * (p.diag_chunk / 4);
  int gs = (int)((sv + 255) / 256);
  if (gs > p.grid_mix) gs = p.grid_mix;
  if (gs < 1) gs = 1;
  int gr = (int)((p.diag_chunk + 255) / 256);
  if (gr > p.grid_mix) gr = p.grid_mix;
  if (gr > partials_cap) gr = partials_cap;
  if (gr < 1) gr = 1;
  da.c1_target = (p.tot_dc1 += (uint32_t)gs);
  da.c2_target = (p.tot_dc2 += (uint32_t)gr);
  plaunch(p, k_diag_scatter, gs, 256, 0, st, da);
  plaunch(p, k_diag_reduce, gr, 256, sizeof(double) * a.k, st, da);
  plaunch(p, k_diag_final, 1, 32, 0, st, da);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CS_OK : perr(CS_ECUDA, "diagnostics launch", e);
}

// Chunk table of the in-step merge kernel for the current tiles (p.h_seg_t0).
int upload_chunks(PeerState& p) {
  const std::vector<int32_t> c = peer_merge_chunks(p.h_seg_t0, kMergeChunk, p.grid_merge);
  if (p.d_chunk_t0) cudaFree(p.d_chunk_t0);
  p.d_chunk_t0 = nullptr;
  p.n_chunks = (int)c.size() - 1;
  if ((int64_t)p.n_tiles * p.n_loc > p.mflag_cap) return CS_OK;  // no room: in-step off (peer_merge_ok)
  cudaError_t e = cudaSuccess;
  if (!p.d_stats) {
    e = cudaMalloc(&p.d_stats, sizeof(unsigned int) * 4);
    if (e == cudaSuccess) e = cudaMemset(p.d_stats, 0, sizeof(unsigned int) * 4);
  }
  if (e == cudaSuccess) e = cudaMalloc(&p.d_chunk_t0, sizeof(int32_t) * c.size());
  if (e == cudaSuccess) e = cudaMemcpy(p.d_chunk_t0, c.data(), sizeof(int32_t) * c.size(), cudaMemcpyHostToDevice);
  return e == cudaSuccess ? CS_OK : perr(CS_ECUDA, "merge chunk table", e);
}

int peer_alloc(PeerState& p, int n_loc, int64_t d, int64_t ld, int k, int nprocs, int rank, int gs, int vranks) {
  p = PeerState();
  p.vranks = vranks > 1 ? vranks : 1;
  if (p.vranks > 1 && (nprocs != p.vranks || rank != 0))
    return perr(CS_EINVAL, "emulated ranks: nprocs must equal vranks, rank 0", cudaSuccess);
  p.nprocs = nprocs;
  p.rank = rank;
  p.n_loc = n_loc;
  p.k = k;
  p.d = d;
  p.ld = ld;
  p.gs = gs;
  // segment bounds (reading C-2) and segment-aligned tiles
  const int64_t nq = (d + kQuantum - 1) / kQuantum;
  std::vector<int64_t> bounds(k + 1);
  std::vector<int32_t> seg_t0(k + 1);
  int n_tiles = 0;
  for (int s = 0; s <= k; ++s) {
    int64_t b = (s == k) ? d : kQuantum * ((s * nq) / k);
    bounds[s] = b < d ? b : d;
  }
  for (int s = 0; s < k; ++s) {
    seg_t0[s] = n_tiles;
    n_tiles += (int)((bounds[s + 1] - bounds[s] + kPeerTile - 1) / kPeerTile);
  }
  seg_t0[k] = n_tiles;
  p.n_tiles = n_tiles;
  p.h_bounds = bounds;
  p.h_seg_t0 = seg_t0;
  if (gs > 0) p.chunk = ((d + gs - 1) / gs + 3) / 4 * 4;

  p.off_inbox = 0;
  p.off_wbox = align_up(p.off_inbox + sizeof(float) * 2 * (size_t)n_loc * ld, 256);
  size_t off = align_up(p.off_wbox + sizeof(float) * 2 * (size_t)n_loc * k, 256);
  if (gs > 0) {
    p.off_gbox = off;
    p.off_gbar = align_up(p.off_gbox + sizeof(float) * (size_t)gs * ld, 256);  // gbox [gs][ld]
    off = align_up(p.off_gbar + sizeof(float) * (size_t)ld, 256);
    p.off_xsync = off;
    p.off_msync = align_up(p.off_xsync + sizeof(float) * (size_t)ld, 256);
    p.off_wsync = align_up(p.off_msync + sizeof(float) * (size_t)ld, 256);
    off = align_up(p.off_wsync + sizeof(float) * (size_t)k, 256);
  }
  // diagnostics: a column chunk per GPU, all workers' x' and psw for it, partials
  p.diag_chunk = ((d + nprocs - 1) / nprocs + 3) / 4 * 4;
  p.off_dx = off;
  off = align_up(off + sizeof(float) * (size_t)(n_loc * nprocs) * p.diag_chunk, 256);
  p.off_dw = off;
  off = align_up(off + sizeof(float) * (size_t)(n_loc * nprocs) * k, 256);
  p.off_dpart = off;
  off = align_up(off + sizeof(double) * 2 * (size_t)nprocs, 256);
  auto flags = [&](size_t& o) {
    o = off;
    off = align_up(off + sizeof(uint32_t) * (size_t)nprocs, 256);
  };
  p.flag_stride = align_up(sizeof(uint32_t) * (size_t)nprocs, 256);
  p.off_done = off;
  off += PeerState::kMaxPieces * p.flag_stride;
  p.off_pdone = off;
  off += PeerState::kMaxPieces * p.flag_stride;
  p.off_d1 = off;  // [kMaxPieces] x [nprocs] each, like done / pdone
  off += PeerState::kMaxPieces * p.flag_stride;
  p.off_d2 = off;
  off += PeerState::kMaxPieces * p.flag_stride;
  flags(p.off_d3);
  flags(p.off_dd1);
  flags(p.off_dd2);
  p.off_count = off;                           // [kMaxPieces] counters, 64 B apart
  p.off_pcount = off + 64 * PeerState::kMaxPieces;
  off += 2 * 64 * PeerState::kMaxPieces;
  p.off_c1 = off;                              // [kMaxPieces] counters, 64 B apart
  p.off_c2 = off + 64 * PeerState::kMaxPieces;
  off += 2 * 64 * PeerState::kMaxPieces;
  p.off_c3 = off;
  p.off_dc1 = off + 64;
  p.off_dc2 = off + 128;
  off += 192;
  // in-step merge schedule (k_push_merge): progress words [2][k][grid_merge]; the grid is
  // the same on every rank (same device model), checked through the header at import
  if (n_loc <= 64 && (int64_t)k * n_loc <= 1024 && k <= 512) {
    const int cap = peer_merge_capacity(k);
    p.grid_merge = cap / p.vranks;
    if (p.grid_merge < 1) p.grid_merge = 0;
  }
  off = align_up(off, 256);
  p.off_claim = off;
  off += 256;
  p.off_mflag = off;
  // trailers per (tile, row): room for a later layer table's extra tiles (one per layer bound,
  // up to 1024 more; a table with more layers runs the split schedule)
  p.mflag_cap = p.grid_merge > 0 ? ((int)((d + kPeerTile - 1) / kPeerTile) + k + 1024) * n_loc : 0;
  off = align_up(off + 16 * 2 * (size_t)p.mflag_cap, 256);
  p.off_hdr = off;
  off += 64;
  p.bytes = align_up(off, 4096);
  cudaError_t e = cudaMalloc(&p.base, p.bytes * p.vranks);
  if (e != cudaSuccess) return perr(CS_ECUDA, "peer region cudaMalloc", e);
  e = cudaMemset(p.base, 0, p.bytes * p.vranks);  // inbox padding is read by 16-byte-rounded bulk copies
  if (e != cudaSuccess) return perr(CS_ECUDA, "peer region memset", e);
  {
    // layout header: every rank must run the same grids over the same tiles
    const int64_t hdr[6] = {0x43524f5353ll, (int64_t)p.grid_merge, (int64_t)p.n_tiles, (int64_t)k, d, (int64_t)p.bytes};
    for (int r = 0; r < p.vranks && e == cudaSuccess; ++r)
      e = cudaMemcpy(p.base + (size_t)r * p.bytes + p.off_hdr, hdr, sizeof(hdr), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return perr(CS_ECUDA, "peer region header", e);
  }
  e = cudaMalloc(&p.d_bounds, sizeof(int64_t) * (k + 1));
  if (e == cudaSuccess) e = cudaMalloc(&p.d_seg_t0, sizeof(int32_t) * (k + 1));
  if (e == cudaSuccess)
    e = cudaMemcpy(p.d_bounds, bounds.data(), sizeof(int64_t) * (k + 1), cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(p.d_seg_t0, seg_t0.data(), sizeof(int32_t) * (k + 1), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return perr(CS_ECUDA, "tile tables", e);

  int dev = 0, sms = 0, occ_push = 0, occ_mix = 0, occ_h = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = push_smem_bytes(k, n_loc);
  e = cudaFuncSetAttribute(k_peer_push, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_push, k_peer_push, kPushThreads, smem);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_mix, k_peer_mix, kMixThreads, 0);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_h, k_hier_reduce, kHierThreads, 0);
  if (e != cudaSuccess || occ_push < 1 || occ_mix < 1 || occ_h < 1) return perr(CS_ECUDA, "occupancy", e);
  const int n_units = p.n_tiles * n_loc;
  // emulated ranks share this GPU: each rank's CTAs are 1/vranks of the co-resident capacity
  const int V = p.vranks;
  p.grid_push_max = std::max(1, sms * occ_push / V);
  p.grid_push = p.grid_push_max < n_units ? p.grid_push_max : n_units;
  p.grid_mix = std::max(1, sms * occ_mix / V);
  p.grid_hier = std::max(1, sms * occ_h / V);
  // hybrid flat step when several workers share a GPU (CS_PEER_HYBRID=0 disables it)
  {
    const char* hy = getenv("CS_PEER_HYBRID");
    p.use_hybrid = n_loc >= 2 && n_loc <= 64 && (int64_t)k * n_loc <= kHMaxTable && !(hy && atoi(hy) == 0);
  }
  if (p.use_hybrid) {
    const size_t hs = hyb_smem_bytes(k, n_loc);
    int occ_w = 0, occ_t = 0;
    e = cudaFuncSetAttribute(k_hyb_walk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hs);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_w, k_hyb_walk, kHThreads, hs);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_t, k_hyb_tail, 256, 0);
    if (e != cudaSuccess || occ_w < 1 || occ_t < 1) return perr(CS_ECUDA, "hybrid occupancy", e);
    p.grid_hyb = std::max(1, sms * occ_w / p.vranks);
    p.grid_tail = std::max(1, sms * occ_t / p.vranks);
    const int T = tma_tile_len(d, p.grid_hyb);
    std::vector<TileDesc> tiles;
    for (int s = 0; s < k; ++s)
      for (int64_t c = bounds[s]; c < bounds[s + 1]; c += T) {
        TileDesc td;
        td.c0 = c;
        td.seg = s;
        td.len = (int32_t)((c + T < bounds[s + 1] ? c + T : bounds[s + 1]) - c);
        td.layer = 0;
        td.pad_ = 0;
        tiles.push_back(td);
      }
    p.n_htiles = (int)tiles.size();
    e = cudaMalloc(&p.d_htiles, sizeof(TileDesc) * tiles.size());
    if (e == cudaSuccess)
      e = cudaMemcpy(p.d_htiles, tiles.data(), sizeof(TileDesc) * tiles.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&p.d_tail_tbl, 2 * (size_t)k * n_loc * p.vranks);  // by step parity, per rank
    if (e != cudaSuccess) return perr(CS_ECUDA, "hybrid tables", e);
  }
  // pieces per step (CS_PEER_PIECES)
  {
    // default 1: measured on 2 B200s (c3), 2 and 3 pieces cost more in repeated push
    // prologues and tails than the mix overlap recovers
    int P = 1;
    const char* env = getenv("CS_PEER_PIECES");
    if (env) P = atoi(env);
    if (P < 1) P = 1;
    if (P > PeerState::kMaxPieces) P = PeerState::kMaxPieces;
    if (P > p.n_tiles) P = p.n_tiles;
    p.pieces = P;
    // hierarchical step with one group: update of piece q overlaps h1 of piece q+1.
    // Default 1: at 4 GPUs (c3 vector) P = 1, 2, 4, 8 measured 399, 409, 445, 558 us; the
    // update kernel takes the SMs the NVLink stores of the next piece need
    int HP = 1;
    const char* henv = getenv("CS_HIER_PIECES");
    if (henv) HP = atoi(henv);
    if (HP < 1) HP = 1;
    if (HP > PeerState::kMaxPieces) HP = PeerState::kMaxPieces;
    if (HP > p.n_tiles) HP = p.n_tiles;
    p.hier_pieces = HP;
    p.fuse = false;  // the schedule (cs_set_schedule) decides; default: merge inside the step
    p.piece_tile.resize(P + 1);
    for (int q = 0; q <= P; ++q) p.piece_tile[q] = (int)((int64_t)q * p.n_tiles / P);
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    e = cudaStreamCreateWithPriority(&p.aux, cudaStreamNonBlocking, hi);
    for (int q = 0; q < PeerState::kMaxPieces && e == cudaSuccess; ++q)
      e = cudaEventCreateWithFlags(&p.ev_push[q], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.ev_mix, cudaEventDisableTiming);
    if (e != cudaSuccess) return perr(CS_ECUDA, "aux stream / events", e);
  }
  p.peer_base.assign(nprocs, nullptr);
  p.peer_base[rank] = p.base;
  for (int r = 1; r < p.vranks; ++r) p.peer_base[r] = p.base + (size_t)r * p.bytes;
  p.allocated = true;
  return p.grid_merge > 0 ? upload_chunks(p) : CS_OK;
}

namespace {
void phase_report();
}  // namespace

void peer_release(PeerState& p) {
  phase_report();
  if (p.imported && p.vranks <= 1) {  // emulated ranks' regions are one local allocation
    for (int r = 0; r < p.nprocs; ++r)
      if (r != p.rank && p.peer_base[r]) cudaIpcCloseMemHandle(p.peer_base[r]);
  }
  if (p.base) cudaFree(p.base);
  if (p.d_peer_base) cudaFree(p.d_peer_base);
  if (p.d_ptiles) cudaFree(p.d_ptiles);
  if (p.d_bounds) cudaFree(p.d_bounds);
  if (p.d_seg_t0) cudaFree(p.d_seg_t0);
  if (p.aux) {
    cudaStreamSynchronize(p.aux);
    cudaStreamDestroy(p.aux);
  }
  for (int q = 0; q < PeerState::kMaxPieces; ++q)
    if (p.ev_push[q]) cudaEventDestroy(p.ev_push[q]);
  if (p.ev_mix) cudaEventDestroy(p.ev_mix);
  if (p.d_htiles) cudaFree(p.d_htiles);
  if (p.d_tail_tbl) cudaFree(p.d_tail_tbl);
  if (p.d_chunk_t0) cudaFree(p.d_chunk_t0);
  if (p.d_stats) cudaFree(p.d_stats);
  if (p.d_nvls_count) cudaFree(p.d_nvls_count);
  nccl_group_release(p);
  p = PeerState();
}

int peer_export(PeerState& p, char* handle_out) {
  if (!p.allocated) return perr(CS_ENOTBOUND, "peer region not allocated", cudaSuccess);
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, p.base);
  if (e != cudaSuccess) return perr(CS_ECUDA, "cudaIpcGetMemHandle", e);
  static_assert(sizeof(cudaIpcMemHandle_t) == CS_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle_out, &h, sizeof(h));
  return CS_OK;
}

int peer_import(PeerState& p, const char* all) {
  if (!p.allocated) return perr(CS_ENOTBOUND, "peer region not allocated", cudaSuccess);
  int64_t mine[6];
  cudaError_t e = cudaMemcpy(mine, p.base + p.off_hdr, sizeof(mine), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return perr(CS_ECUDA, "peer header", e);
  for (int r = 0; r < p.nprocs; ++r) {
    if (r == p.rank) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, all + (size_t)r * CS_IPC_HANDLE_BYTES, sizeof(h));
    void* ptr = nullptr;
    e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return perr(CS_ECUDA, "cudaIpcOpenMemHandle", e);
    p.peer_base[r] = (char*)ptr;
    // the peer's layout must be ours: same offsets, grid and tiles (same-index CTAs pair up)
    int64_t theirs[6];
    e = cudaMemcpy(theirs, p.peer_base[r] + p.off_hdr, sizeof(theirs), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return perr(CS_ECUDA, "peer header read", e);
    if (memcmp(mine, theirs, sizeof(mine)) != 0)
      return perr(CS_EINVAL, "peer exchange region layout differs between ranks (device model, d, k or grid)",
                  cudaSuccess);
  }
  return peer_import_self(p);
}

int peer_import_self(PeerState& p) {
  if (!p.allocated) return perr(CS_ENOTBOUND, "peer region not allocated", cudaSuccess);
  cudaError_t e = cudaMalloc(&p.d_peer_base, sizeof(char*) * p.nprocs);
  if (e == cudaSuccess)
    e = cudaMemcpy(p.d_peer_base, p.peer_base.data(), sizeof(char*) * p.nprocs, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return perr(CS_ECUDA, "peer table", e);
  p.imported = true;
  return CS_OK;
}

namespace {

PeerKernelArgs kernel_args(const PeerState& p, const PeerStepArgs& a, uint32_t epoch, bool final_only) {
  PeerKernelArgs ka;
  ka.s = a;
  ka.peers = p.d_peer_base;
  ka.bounds = p.d_bounds;
  ka.seg_t0 = p.d_seg_t0;
  ka.tiles = p.d_ptiles;
  ka.n_tiles = p.n_tiles;
  ka.epoch = epoch;
  ka.final_only = final_only ? 1 : 0;
  ka.fuse_mix = 0;
  ka.fused_topo = fused_topo_ok(a.gs > 0 ? a.groups : a.world, a.k, a.n_loc) ? 1 : 0;
  ka.vranks = p.vranks;
  ka.off_inbox = p.off_inbox;
  ka.off_wbox = p.off_wbox;
  ka.pieces = p.pieces;
  ka.flag_stride = p.flag_stride;
  ka.off_done = p.off_done;
  ka.off_count = p.off_count;
  ka.off_pdone = p.off_pdone;
  ka.off_pcount = p.off_pcount;
  ka.off_d2 = p.off_d2;
  return ka;
}

int launch_topology_for(const PeerStepArgs& a, int n, int tag, cudaStream_t st) {
  TopoArgs t;
  t.seed = a.seed;
  t.step = a.step;
  t.n = n;
  t.k = a.k;
  t.tag = tag;
  t.given = a.given;
  t.src = a.src;
  t.dst = a.dst;
  t.ord = nullptr;
  t.psw = nullptr;
  t.group_size = 1;
  t.rw = nullptr;
  t.inv_wsum = nullptr;
  t.err = a.err;
  ++g_peer_launches;
  cudaError_t e = launch_topology(t, st);
  return e == cudaSuccess ? CS_OK : perr(CS_ECUDA, "topology launch", e);
}

}  // namespace

int peer_set_layers(PeerState& p, const std::vector<int64_t>& plan, const std::vector<int64_t>& layer_bounds,
                    std::vector<int32_t>& tile_first) {
  const int k = p.k;
  if ((int)plan.size() != k + 1) return perr(CS_EINVAL, "segment plan size", cudaSuccess);
  std::vector<int64_t> lb = layer_bounds.empty() ? std::vector<int64_t>{0, p.d} : layer_bounds;
  const int L = (int)lb.size() - 1;
  std::vector<TileDesc> tiles;
  std::vector<int32_t> seg_t0(k + 1, 0);
  tile_first.assign(L + 1, 0);
  int l = 0;
  for (int s = 0; s < k; ++s) {
    seg_t0[s] = (int32_t)tiles.size();
    int64_t c = plan[s];
    while (c < plan[s + 1]) {
      while (lb[l + 1] <= c) tile_first[++l] = (int32_t)tiles.size();
      const int64_t end = std::min(std::min(plan[s + 1], lb[l + 1]), c + (int64_t)kPeerTile);
      TileDesc td;
      td.c0 = c;
      td.seg = s;
      td.len = (int32_t)(end - c);
      td.layer = l;
      td.pad_ = 0;
      tiles.push_back(td);
      c = end;
    }
  }
  seg_t0[k] = (int32_t)tiles.size();
  while (l < L) tile_first[++l] = (int32_t)tiles.size();
  cudaError_t e = cudaSuccess;
  if (p.d_ptiles) cudaFree(p.d_ptiles);
  p.d_ptiles = nullptr;
  p.h_tile_c0.clear();
  if (layer_bounds.empty()) {
    // back to the closed-form equal split (tiles of kPeerTile)
    int n = 0;
    for (int s = 0; s < k; ++s) {
      seg_t0[s] = n;
      n += (int)((plan[s + 1] - plan[s] + kPeerTile - 1) / kPeerTile);
    }
    seg_t0[k] = n;
  } else {
    e = cudaMalloc(&p.d_ptiles, sizeof(TileDesc) * tiles.size());
    if (e == cudaSuccess)
      e = cudaMemcpy(p.d_ptiles, tiles.data(), sizeof(TileDesc) * tiles.size(), cudaMemcpyHostToDevice);
    p.h_tile_c0.resize(tiles.size() + 1);
    for (size_t t = 0; t < tiles.size(); ++t) p.h_tile_c0[t] = tiles[t].c0;
    p.h_tile_c0[tiles.size()] = p.d;
  }
  if (e == cudaSuccess)
    e = cudaMemcpy(p.d_bounds, plan.data(), sizeof(int64_t) * (k + 1), cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(p.d_seg_t0, seg_t0.data(), sizeof(int32_t) * (k + 1), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return perr(CS_ECUDA, "peer layer tiles", e);
  p.h_bounds = plan;
  p.h_seg_t0 = seg_t0;
  p.n_tiles = seg_t0[k];
  if (p.grid_merge > 0) {
    const int rc = upload_chunks(p);
    if (rc) return rc;
  }
  if (p.use_hybrid) {
    // the hybrid walk's own tiles (TMA-sized), split the same way; LARS norms use them
    const int T = tma_tile_len(p.d, p.grid_hyb);
    std::vector<TileDesc> ht;
    std::vector<int32_t> hfirst(L + 1, 0);
    int hl = 0;
    for (int s2 = 0; s2 < k; ++s2) {
      int64_t c = plan[s2];
      while (c < plan[s2 + 1]) {
        while (lb[hl + 1] <= c) hfirst[++hl] = (int32_t)ht.size();
        const int64_t end = std::min(std::min(plan[s2 + 1], lb[hl + 1]), c + (int64_t)T);
        TileDesc td;
        td.c0 = c;
        td.seg = s2;
        td.len = (int32_t)(end - c);
        td.layer = hl;
        td.pad_ = 0;
        ht.push_back(td);
        c = end;
      }
    }
    while (hl < L) hfirst[++hl] = (int32_t)ht.size();
    if (p.d_htiles) cudaFree(p.d_htiles);
    p.d_htiles = nullptr;
    cudaError_t e2 = cudaMalloc(&p.d_htiles, sizeof(TileDesc) * ht.size());
    if (e2 == cudaSuccess)
      e2 = cudaMemcpy(p.d_htiles, ht.data(), sizeof(TileDesc) * ht.size(), cudaMemcpyHostToDevice);
    if (e2 != cudaSuccess) return perr(CS_ECUDA, "hybrid layer tiles", e2);
    p.n_htiles = (int)ht.size();
    tile_first = hfirst;
  }
  const int units = p.n_tiles * p.n_loc;
  p.grid_push = p.grid_push_max < units ? p.grid_push_max : units;
  // pieces follow the new tile count
  if (p.pieces > p.n_tiles) p.pieces = p.n_tiles;
  p.piece_tile.resize(p.pieces + 1);
  for (int q = 0; q <= p.pieces; ++q) p.piece_tile[q] = (int)((int64_t)q * p.n_tiles / p.pieces);
  if (p.hier_pieces > p.n_tiles) p.hier_pieces = p.n_tiles;
  return CS_OK;
}

// The tiles of the kernel that runs the flat step (LARS norms are computed over them).
const TileDesc* peer_tiles(const PeerState& p) { return p.use_hybrid ? p.d_htiles : p.d_ptiles; }
int peer_tile_count(const PeerState& p) { return p.use_hybrid ? p.n_htiles : p.n_tiles; }

namespace {

int64_t tile_col(const PeerState& p, int t) {
  if (t >= p.n_tiles) return p.d;
  if (!p.h_tile_c0.empty()) return p.h_tile_c0[t];
  int sg = 0;
  while (p.h_seg_t0[sg + 1] <= t) ++sg;
  return p.h_bounds[sg] + (int64_t)(t - p.h_seg_t0[sg]) * kPeerTile;
}

// push(q) on the caller's stream; mix(q) on the aux stream after push(q), so push(q+1)
// overlaps mix(q); the caller's stream finally waits for the last mix.
int launch_push_mix(PeerState& p, const PeerKernelArgs& ka, cudaStream_t st) {
  const int P = ka.final_only ? 1 : p.pieces;
  for (int q = 0; q < P; ++q) {
    PeerKernelArgs kq = ka;
    kq.tile_lo = P == 1 ? 0 : p.piece_tile[q];
    kq.tile_hi = P == 1 ? p.n_tiles : p.piece_tile[q + 1];
    kq.col_lo = tile_col(p, kq.tile_lo);
    kq.col_hi = tile_col(p, kq.tile_hi);
    kq.off_done = p.off_done + q * p.flag_stride;
    kq.off_pdone = p.off_pdone + q * p.flag_stride;
    kq.off_count = p.off_count + 64 * q;
    kq.off_pcount = p.off_pcount + 64 * q;
    const int units = (kq.tile_hi - kq.tile_lo) * ka.s.n_loc;
    const int grid = p.grid_push < units ? p.grid_push : (units > 0 ? units : 1);
    const size_t smem = push_smem_bytes(ka.s.k, ka.s.n_loc);
    if (ka.final_only) {
      kq.done_target = (p.tot_count[q] += (uint32_t)grid);
      plaunch(p, k_peer_push, grid, kPushThreads, smem, st, kq);
      continue;
    }
    kq.pdone_target = (p.tot_pcount[q] += (uint32_t)grid);
    kq.done_target = (p.tot_count[q] += (uint32_t)p.grid_mix);
    plaunch(p, k_peer_push, grid, kPushThreads, smem, st, kq);
    if (P == 1) {
      plaunch(p, k_peer_mix, p.grid_mix, kMixThreads, 0, st, kq);
    } else {
      cudaEventRecord(p.ev_push[q], st);
      cudaStreamWaitEvent(p.aux, p.ev_push[q], 0);
      plaunch(p, k_peer_mix, p.grid_mix, kMixThreads, 0, p.aux, kq);
    }
  }
  if (P > 1) {
    cudaEventRecord(p.ev_mix, p.aux);
    cudaStreamWaitEvent(st, p.ev_mix, 0);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CS_OK : perr(CS_ECUDA, "push/mix launch", e);
}

}  // namespace

namespace {
HybArgs hyb_args(const PeerState& p, const PeerStepArgs& a, uint32_t epoch) {
  HybArgs h;
  h.x = a.x;
  h.m = a.m;
  h.g = a.g;
  h.psw = a.psw;
  h.ld = a.ld;
  h.d = a.d;
  h.nq = a.nq;
  h.k = a.k;
  h.world = a.world;
  h.n_loc = a.n_loc;
  h.first = a.first;
  h.rank = a.rank;
  h.nprocs = a.nprocs;
  h.seed = a.seed;
  h.step = a.step;
  h.given = a.given;
  h.wire = a.wire;
  h.src_tbl = a.src;
  h.fused = a.world <= 64 ? 1 : 0;
  h.lr = a.lr;
  h.mu = a.mu;
  h.tiles = p.d_htiles;
  h.n_tiles = p.n_htiles;
  h.peers = p.d_peer_base;
  h.off_inbox = p.off_inbox;
  h.off_wbox = p.off_wbox;
  h.off_done = p.off_done;
  h.off_pdone = p.off_pdone;
  h.off_count = p.off_count;
  h.off_pcount = p.off_pcount;
  h.flag_stride = p.flag_stride;
  h.pieces = p.pieces;
  h.epoch = epoch;
  h.pdone_target = 0;
  h.done_target = 0;
  h.tail_tbl = nullptr;
  h.err = a.err;
  h.fuse = 0;
  h.tail_prev = nullptr;
  h.lrs = a.lrs;
  h.n_layers = a.n_layers;
  h.wd = a.wd;
  h.bounds = p.d_bounds;
  h.vranks = p.vranks;
  h.tbl_stride = 2 * (size_t)a.k * a.n_loc;
  return h;
}
}  // namespace

int peer_flat_step(PeerState& p, const PeerStepArgs& a, cudaStream_t st, cudaEvent_t ev0,
                   cudaEvent_t ev1) {
  int rc = CS_OK;
  // a flat step gives every worker its own state: the next hierarchical step re-replicates
  // each group's leader to its members first
  p.need_sync = true;
  if (peer_merge_ok(p, a)) {
    // default: the merge completes inside this step's kernel (k_push_merge walks any n_loc)
    p.last_fused = false;
    if (ev0) cudaEventRecord(ev0, st);
    rc = peer_flush(p, st);  // a merge left pending by the deferred schedule
    if (rc) return rc;
    if (a.world > 64) rc = launch_topology_for(a, a.world, CS_TAG_FLAT, st);
    if (rc) return rc;
    PeerStepArgs b = a;
    b.gs = 0;
    b.g_off = 0;
    rc = peer_merge_launch(p, b, ++p.epoch, st);
    if (rc) return perr(rc, "k_push_merge launch", cudaGetLastError());
    if (ev1) cudaEventRecord(ev1, st);
    return CS_OK;
  }
  if (p.use_hybrid) {
    // deferred merge: this step's chain tails are merged inside the next walk (or
    // peer_flush); the previous step's tails are merged here before their update
    const bool fuse = p.fuse && a.lrs == nullptr;  // LARS norms need the merged x
    p.last_fused = fuse;
    if (ev0) cudaEventRecord(ev0, st);
    if (!fuse || (p.pending && (p.pending_args.x != a.x || p.pending_args.psw != a.psw))) {
      rc = peer_flush(p, st);
      if (rc) return rc;
    }
    const bool fused = a.world <= 64;
    if (!fused && a.given == nullptr) rc = launch_topology_for(a, a.world, CS_TAG_FLAT, st);
    if (rc) return rc;
    HybArgs h = hyb_args(p, a, ++p.epoch);
    const size_t tbl = (size_t)a.k * a.n_loc;
    h.tail_tbl = p.d_tail_tbl + (h.epoch & 1u) * tbl;
    h.pdone_target = (p.tot_pcount[0] += (uint32_t)p.grid_hyb);
    if (fuse) {
      h.fuse = p.pending ? 1 : 0;
      h.tail_prev = p.d_tail_tbl + ((h.epoch - 1) & 1u) * tbl;
      plaunch(p, k_hyb_walk, p.grid_hyb, kHThreads, hyb_smem_bytes(a.k, a.n_loc), st, h);
      p.pending = h.epoch;
      p.pending_args = a;
    } else {
      h.done_target = (p.tot_count[0] += (uint32_t)p.grid_tail);
      plaunch(p, k_hyb_walk, p.grid_hyb, kHThreads, hyb_smem_bytes(a.k, a.n_loc), st, h);
      plaunch(p, k_hyb_tail, p.grid_tail, 256, 0, st, h);
    }
    if (ev1) cudaEventRecord(ev1, st);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? CS_OK : perr(CS_ECUDA, "hybrid launch", e);
  }

  // deferred merge (opt-in, kSchedDeferred): this step's push applies the previous step's
  // merge tile by tile, and its own merge waits for the next push (or peer_flush); the
  // separate mix pass and its cross-GPU wait disappear from the step, but params hold y
  // until then
  const bool fuse = p.fuse && p.pieces == 1 && a.lrs == nullptr;
  p.last_fused = fuse;
  if (ev0) cudaEventRecord(ev0, st);
  if (!fuse || (p.pending && (p.pending_args.x != a.x || p.pending_args.psw != a.psw))) {
    rc = peer_flush(p, st);
    if (rc) return rc;
  }
  if (!fused_topo_ok(a.world, a.k, a.n_loc)) rc = launch_topology_for(a, a.world, CS_TAG_FLAT, st);
  if (rc) return rc;
  PeerKernelArgs ka = kernel_args(p, a, ++p.epoch, false);
  ka.s.gs = 0;
  if (fuse) {
    ka.fuse_mix = p.pending != 0 ? 1 : 0;
    ka.tile_lo = 0;
    ka.tile_hi = p.n_tiles;
    ka.col_lo = 0;
    ka.col_hi = p.d;
    const int units = p.n_tiles * a.n_loc;
    const int grid = p.grid_push < units ? p.grid_push : (units > 0 ? units : 1);
    ka.pdone_target = (p.tot_pcount[0] += (uint32_t)grid);
    plaunch(p, k_peer_push, grid, kPushThreads, push_smem_bytes(a.k, a.n_loc), st, ka);
    p.pending = ka.epoch;
    p.pending_args = ka.s;
    rc = cudaGetLastError() == cudaSuccess ? CS_OK : perr(CS_ECUDA, "fused push launch", cudaGetLastError());
  } else {
    rc = launch_push_mix(p, ka, st);
  }
  if (ev1) cudaEventRecord(ev1, st);
  return rc;
}

int peer_set_schedule(PeerState& p, int sched, cudaStream_t st) {
  const int rc = peer_flush(p, st);
  if (rc) return rc;
  p.sched = sched;
  p.fuse = sched == kSchedDeferred;
  return CS_OK;
}

int peer_flush(PeerState& p, cudaStream_t st) {
  if (!p.pending) return CS_OK;
  if (p.use_hybrid) {  // the pending step's chain tails: x = (y + inbox)/2, psw likewise
    HybArgs h = hyb_args(p, p.pending_args, p.pending);
    h.tail_tbl = p.d_tail_tbl + (p.pending & 1u) * (size_t)p.pending_args.k * p.pending_args.n_loc;
    h.done_target = (p.tot_count[0] += (uint32_t)p.grid_tail);
    plaunch(p, k_hyb_tail, p.grid_tail, 256, 0, st, h);
    p.pending = 0;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? CS_OK : perr(CS_ECUDA, "deferred tail merge launch", e);
  }
  PeerKernelArgs ka = kernel_args(p, p.pending_args, p.pending, false);
  ka.s.gs = 0;
  ka.tile_lo = 0;
  ka.tile_hi = p.n_tiles;
  ka.col_lo = 0;
  ka.col_hi = p.d;
  ka.done_target = (p.tot_count[0] += (uint32_t)p.grid_mix);
  plaunch(p, k_peer_mix, p.grid_mix, kMixThreads, 0, st, ka);
  p.pending = 0;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CS_OK : perr(CS_ECUDA, "deferred merge launch", e);
}

// Debug knob CS_PHASE_TIMING=1: events between the hierarchical kernels; the per-phase
// averages are printed to stderr when the peer state is released.
namespace {
struct PhaseTimes {
  std::vector<cudaEvent_t> ev;  // 4 per step: start, after scatter, after reduce, after update
  bool on = false, checked = false;
};
PhaseTimes g_phase;

void phase_record(int i, cudaStream_t st) {
  if (!g_phase.checked) {
    const char* v = getenv("CS_PHASE_TIMING");
    g_phase.on = v && v[0] == '1';
    g_phase.checked = true;
  }
  if (!g_phase.on) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, st);
  g_phase.ev.push_back(e);
  (void)i;
}

void phase_report() {
  if (!g_phase.on || g_phase.ev.size() < 4) return;
  cudaDeviceSynchronize();
  double t[3] = {0, 0, 0};
  const size_t steps = g_phase.ev.size() / 4;
  for (size_t s = 0; s < steps; ++s)
    for (int k = 0; k < 3; ++k) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, g_phase.ev[4 * s + k], g_phase.ev[4 * s + k + 1]);
      t[k] += ms;
    }
  fprintf(stderr, "[cs phase] steps=%zu scatter %.1f us  reduce+allgather %.1f us  update %.1f us\n", steps,
          1e3 * t[0] / steps, 1e3 * t[1] / steps, 1e3 * t[2] / steps);
  for (cudaEvent_t e : g_phase.ev) cudaEventDestroy(e);
  g_phase.ev.clear();
}
}  // namespace

int peer_hier_step(PeerState& p, const PeerStepArgs& a, cudaStream_t st, cudaEvent_t ev0,
                   cudaEvent_t ev1) {
  if (p.gs <= 0 || a.n_loc != 1) return perr(CS_EUNSUPPORTED, "multi-GPU hierarchical step needs one worker per GPU", cudaSuccess);
  const bool exchange = a.groups >= 2;
  if (exchange && !fused_topo_ok(a.groups, a.k, a.n_loc)) {
    int rc = launch_topology_for(a, a.groups, CS_TAG_HIER, st);
    if (rc) return rc;
  }
  // deferred merge of the leader exchange: a pending merge (from the previous hierarchical
  // or flat step) is applied inside this step's push, unless something reads or rewrites x
  // first (replica sync, LARS norms) or there is no exchange to carry it
  // Opt-in (CS_HIER_FUSE=1): at 4 GPUs (2 groups x 2, c4 vector) it measured 546 us against
  // 440 us for push + mix; the next step's reduce-scatter then competes with the pushes
  static const bool hier_fuse = getenv("CS_HIER_FUSE") && getenv("CS_HIER_FUSE")[0] == '1';
  const bool fuse = hier_fuse && p.fuse && exchange && p.pieces == 1 && !a.wire && a.lrs_out == nullptr &&
                    !(p.need_sync && p.gs > 1) &&
                    !(p.pending && (p.pending_args.x != a.x || p.pending_args.psw != a.psw));
  p.last_fused = fuse;
  if (!fuse) {
    int rc0 = peer_flush(p, st);
    if (rc0) return rc0;
  }
  const uint32_t epoch = ++p.epoch;
  HierArgs h;
  h.g = a.g;
  h.peers = p.d_peer_base;
  h.d = a.d;
  h.chunk = p.chunk;
  h.rank = a.rank;
  h.gs = p.gs;
  h.inv_gs = a.inv_gs;
  h.epoch = epoch;
  h.off_gbox = p.off_gbox;
  h.off_gbar = p.off_gbar;
  h.off_d1 = p.off_d1;
  h.off_c1 = p.off_c1;
  h.off_d2 = p.off_d2;
  h.off_c2 = p.off_c2;
  h.err = a.err;
  h.vranks = p.vranks;
  h.ld = a.ld;
  h.pull = 0;
  PeerStepArgs b = a;
  b.g = reinterpret_cast<const float*>(p.base + p.off_gbar);  // the group mean
  b.g_off = p.off_gbar;
  b.gs = p.gs;
  // default schedule: the leader exchange merges inside its own kernel (k_push_merge)
  const bool merge = exchange && !fuse && peer_merge_ok(p, a);
  if (a.lrs_out) {  // LARS with the group-reduced gradient: b.lrs is filled after h1 below
    b.lrs = a.lrs_out;
    if (p.hier_pieces != 1 && !exchange) return perr(CS_EUNSUPPORTED, "hierarchical LARS needs CS_HIER_PIECES=1", cudaSuccess);
  }
  // NVLS h1 (hier_nvls.cu): the group mean by in-switch reduction into this GPU's
  // multicast workspace; the update below then reads a complete gbar
  const bool nvls = p.mc_uc != nullptr && p.vranks <= 1 && a.lrs_out == nullptr && !fuse;
  const float* g_mc = nullptr;
  if (nvls) {
    for (const auto& r : p.mc_grads)
      if (reinterpret_cast<const char*>(a.g) >= r.uc &&
          reinterpret_cast<const char*>(a.g) + (size_t)a.d * sizeof(float) <= r.uc + r.bytes)
        g_mc = reinterpret_cast<const float*>(r.mc + (reinterpret_cast<const char*>(a.g) - r.uc));
    b.g = reinterpret_cast<const float*>(p.mc_uc + nvls_off_gbar());
    b.g_off = 0;
    b.gbar_local = 1;
  }
  p.last_nvls = nvls;
  // NCCL h1 (hier_nccl.cu): ncclAllReduce of the group's gradients into this GPU's gbar; the
  // update scales the sum by fp32(1/|G|)
  const bool nccl = !nvls && p.nccl_comm != nullptr && p.vranks <= 1 && a.lrs_out == nullptr && !fuse;
  p.last_nccl = nccl;
  if (nccl) {
    b.g = reinterpret_cast<const float*>(p.base + p.off_gbar);
    b.gbar_local = 1;
    b.g_scale = a.inv_gs;
  }
  // pulled group mean (one group of 2 GPUs, without NVLS, NCCL, LARS or column pieces):
  // k_hier_reduce keeps each member's mean chunk in its own gbar and the update bulk-loads the
  // chunks from their owners over NVLink, so the all-gather rides in the update's pass.
  // Measured: 285.7 vs 306.8 us at 1 x 2 GPUs, but 440 vs 404 us at 1 x 4 and 450 vs 399 us at
  // 2 x 2 (peer reads are slower than the all-gather's stores once several owners or the leader
  // exchange share the links); CS_HIER_PULL = 0 / 1 forces it off / on
  static const int pull_env = getenv("CS_HIER_PULL") ? atoi(getenv("CS_HIER_PULL")) : -1;
  const bool pull = (pull_env < 0 ? (p.gs == 2 && !exchange) : pull_env == 1) && !nvls && !nccl &&
                    a.lrs_out == nullptr && (exchange || p.hier_pieces == 1) && p.gs > 1;
  if (pull) b.gpull_chunk = ((a.d + p.gs - 1) / p.gs + 3) / 4 * 4;
  PeerKernelArgs ka = kernel_args(p, b, epoch, !exchange);
  if (ev0) cudaEventRecord(ev0, st);
  if (p.need_sync && p.gs > 1) {  // members become exact replicas of their leader
    SyncArgs sa;
    sa.h = h;
    sa.x = a.x;
    sa.m = a.m;
    sa.psw = a.psw;
    sa.ld = a.ld;
    sa.k = a.k;
    sa.c3_target = (p.tot_c3 += (uint32_t)p.grid_hier);
    sa.off_xsync = p.off_xsync;
    sa.off_msync = p.off_msync;
    sa.off_wsync = p.off_wsync;
    sa.off_d3 = p.off_d3;
    sa.off_c3 = p.off_c3;
    plaunch(p, k_hier_sync, p.grid_hier, kHierThreads, 0, st, sa);
  }
  p.need_sync = false;
  // One group (no leader exchange): the vector is cut into P column pieces; h1 of piece
  // q+1 (NVLink-bound) runs on the caller's stream while the update of piece q (HBM-bound,
  // k_peer_push in final_only mode, waiting on piece q's d2 flags) runs on the aux stream.
  const int P = exchange || nvls || nccl ? 1 : p.hier_pieces;
  h.gstride = a.ld;
  int rc = CS_OK;
  for (int q = 0; q < P; ++q) {
    const int t_lo = (int)((int64_t)q * p.n_tiles / P), t_hi = (int)((int64_t)(q + 1) * p.n_tiles / P);
    h.col_lo = tile_col(p, t_lo);
    h.col_hi = tile_col(p, t_hi);
    h.chunk = ((h.col_hi - h.col_lo + p.gs - 1) / p.gs + 3) / 4 * 4;
    h.pull = pull ? 1 : 0;
    h.off_d1 = p.off_d1 + q * p.flag_stride;
    h.off_d2 = p.off_d2 + q * p.flag_stride;
    h.off_c1 = p.off_c1 + 64 * q;
    h.off_c2 = p.off_c2 + 64 * q;
    h.c1_target = (p.tot_c1[q] += (uint32_t)p.grid_hier);
    h.c2_target = (p.tot_c2[q] += (uint32_t)p.grid_hier);
    phase_record(0, st);
    if (nvls) {
      if (nvls_h1(p, a.g, g_mc, a.rank % p.gs, a.inv_gs, a.err, st))
        return perr(CS_ECUDA, "k_hier_nvls launch", cudaGetLastError());
      phase_record(2, st);
    } else if (nccl) {
      if (nccl_h1(p, a.g, reinterpret_cast<float*>(p.base + p.off_gbar), a.d, st))
        return perr(CS_ECUDA, nccl_error(), cudaSuccess);
      phase_record(2, st);
    } else {
      plaunch(p, k_hier_scatter, p.grid_hier, kHierThreads, 0, st, h);
      phase_record(1, st);
      plaunch(p, k_hier_reduce, p.grid_hier, kHierThreads, 0, st, h);
      phase_record(2, st);
    }
    if (a.lrs_out) {  // rates from the leader replica's x and the group mean, once gbar is whole
      LarsWait w;
      if (p.vranks <= 1) {
        w.flags = reinterpret_cast<const uint32_t*>(p.base + p.off_d2);
        w.first = (a.rank / p.gs) * p.gs;
        w.count = p.gs;
        w.epoch = epoch;
        w.err = a.err;
      }
      // emulated ranks: one launch per rank (each has its own group mean); the reduce kernel
      // before them has completed for every rank, so no wait
      for (int r = 0; r < p.vranks; ++r) {
        cudaError_t le = launch_lars_rates(
            a.x + (int64_t)r * a.ld, reinterpret_cast<const float*>(p.peer_base[p.vranks > 1 ? r : a.rank] + p.off_gbar),
            a.ld, p.d_ptiles, p.n_tiles, 1, a.tile_first, a.n_layers, a.lars_part + (size_t)2 * r * p.n_tiles, a.lr,
            a.eta, a.wd, a.eps, a.lrs_out + (int64_t)r * a.n_layers, st, w);
        if (le != cudaSuccess) return perr(CS_ECUDA, "hierarchical LARS rates", le);
      }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return perr(CS_ECUDA, "hierarchical launch", e);
    if (merge) {  // update + exchange + merge of the leaders' step (replicated leader), one kernel
      rc = peer_merge_launch(p, b, epoch, st);
      if (rc) return perr(rc, "k_push_merge launch", cudaGetLastError());
      phase_record(3, st);
      continue;
    }
    if (exchange && fuse) {  // the push only; its merge waits for the next push or a flush
      PeerKernelArgs kf = ka;
      kf.fuse_mix = p.pending ? 1 : 0;
      kf.tile_lo = 0;
      kf.tile_hi = p.n_tiles;
      kf.col_lo = 0;
      kf.col_hi = p.d;
      const int grid = p.grid_push < p.n_tiles ? p.grid_push : (p.n_tiles > 0 ? p.n_tiles : 1);
      kf.pdone_target = (p.tot_pcount[0] += (uint32_t)grid);
      plaunch(p, k_peer_push, grid, kPushThreads, push_smem_bytes(a.k, a.n_loc), st, kf);
      p.pending = epoch;
      p.pending_args = b;
      phase_record(3, st);
      continue;
    }
    if (exchange) {
      rc = launch_push_mix(p, ka, st);
      phase_record(3, st);
      continue;
    }
    PeerKernelArgs kq = ka;
    kq.tile_lo = t_lo;
    kq.tile_hi = t_hi;
    kq.col_lo = h.col_lo;
    kq.col_hi = h.col_hi;
    kq.off_d2 = h.off_d2;
    kq.off_done = p.off_done;
    kq.off_count = p.off_count + 64 * q;
    kq.pieces = q == P - 1 ? p.pieces : 0;  // the last update advances every flat piece's done flag
    const int grid = p.grid_push < (t_hi - t_lo) ? p.grid_push : (t_hi - t_lo > 0 ? t_hi - t_lo : 1);
    kq.done_target = (p.tot_count[q] += (uint32_t)grid);
    const size_t smem = push_smem_bytes(ka.s.k, ka.s.n_loc);
    if (P == 1) {
      plaunch(p, k_peer_push, grid, kPushThreads, smem, st, kq);
    } else {
      cudaEventRecord(p.ev_push[q], st);
      cudaStreamWaitEvent(p.aux, p.ev_push[q], 0);
      plaunch(p, k_peer_push, grid, kPushThreads, smem, p.aux, kq);
    }
    phase_record(3, P == 1 ? st : p.aux);
  }
  if (!exchange && P > 1) {
    cudaEventRecord(p.ev_mix, p.aux);
    cudaStreamWaitEvent(st, p.ev_mix, 0);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return perr(CS_ECUDA, "hierarchical update launch", e);
  if (ev1) cudaEventRecord(ev1, st);
  return rc;
}

}  // namespace cs
