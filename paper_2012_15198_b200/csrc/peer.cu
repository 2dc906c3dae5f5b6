// Multi-GPU flat step over NVLink peer memory (configs 3 and 5).
//
// Workers are partitioned contiguously: worker w lives on GPU w / n_loc.  At step
// t each GPU runs ONE persistent kernel (cooperative launch, so every CTA is
// co-resident).  The work unit is (tile q, local worker r): a segment-aligned
// range of up to kPeerTile columns of one worker's vector, numbered tile-major
// (u = q * n_loc + r); CTA c takes units c, c + G, c + 2G, ... on every GPU.
// Units are cut into waves of exactly G*m units (m per CTA, G*m a multiple of
// n_loc so a tile never straddles two waves), the same on every GPU.
//
// Warp-specialised CTA:
//
//   load warp     bulk-TMA of the x, m, g row-tiles of the next units into a
//                 kStagesA-deep shared-memory ring.
//   push warps    wave w: for each unit, m', y from the staged tiles (a3); m' ->
//                 HBM; y -> x (kept in L2 for the mix) and -> the RECEIVER's
//                 inbox on the receiver's GPU (NVLink store; Alg.1 l.7 isend to
//                 send_to = dst_s(i)); the first tile of a
//                 segment also pushes w_{i,s}.  Then one fence.acq_rel.sys and a
//                 red.add on every GPU's arrival counter of wave w (the irecv
//                 completion, Alg.1 l.14, for a whole wave at once).
//   mix warps     wave w: wait until this GPU's counter of wave w has every CTA
//                 of every GPU (Alg.1 l.12-14 "wait send and recv"), then
//                 x = (y + inbox) * 0.5, w = (w + wbox) * 0.5 (a5, Alg.1 l.17).
//                 y and inbox of a wave are still L2-resident.
//
// The NVLink-bound pushes of wave w overlap the HBM-bound mixes of earlier
// waves.  Deadlock freedom: push warps never wait on another GPU (only on their
// own TMA ring), mix warps only wait for pushes, and all CTAs are resident.
//
// The inbox ping-pongs on step parity; before pushing at epoch e a GPU waits
// until every peer has finished epoch e-2 (the last reader of that parity) —
// the "done" words each GPU writes into every peer's region at the end of a
// step.  Counters and done words carry the monotone epoch, so nothing is reset.
// Spins are bounded (~20 s of %globaltimer) and report CS_ETIMEOUT instead of
// hanging the GPU.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/crossover_sgd.h"
#include "common.cuh"
#include "peer.cuh"
#include "ptx.cuh"

namespace cs {

namespace {

std::string g_peer_err;

int perr(int code, const char* what, cudaError_t e) {
  char buf[256];
  snprintf(buf, sizeof(buf), "%s: %s", what, e == cudaSuccess ? "" : cudaGetErrorString(e));
  g_peer_err = buf;
  return code;
}

constexpr int kGroup = 128;                     // threads per warp group (push / mix)
constexpr int kPeerThreads = 2 * kGroup + 64;   // push warps, mix warps, load warp, release warp
constexpr int kWaveSlots = 8;                   // wave hand-off ring (push warps -> release warp)
constexpr int kPeerTile = 2048;                 // columns per unit: 8 KB of one worker's row
constexpr int kPer = kPeerTile / 4 / kGroup;    // float4 per thread per array
constexpr int kStagesA = 4;                     // x, m, g ring depth (units)
constexpr size_t kTileBytes = sizeof(float) * kPeerTile;
constexpr size_t kRingBytes = kTileBytes * 3 * kStagesA;
constexpr int kMaxDstSmem = 2048;               // receivers table in smem when k*n_loc <= this
constexpr double kWaveBytes = 24.0 * 1024 * 1024;
constexpr uint64_t kSpinLimitNs = 20ull * 1000 * 1000 * 1000;
constexpr int kBarMix = 2;                      // named barrier id of the mix warps

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

size_t peer_smem_bytes(int k, int n_loc) {
  size_t b = kRingBytes + sizeof(int64_t) * (k + 1) + sizeof(int32_t) * (k + 1);
  if ((int64_t)k * n_loc <= kMaxDstSmem) b += sizeof(int32_t) * (size_t)k * n_loc;
  return align_up(b, 16);
}

// wait until (int32)(*p - target) >= 0 polling relaxed, then acquire; false on timeout
__device__ bool wait_acquire(const uint32_t* p, uint32_t target) {
  uint64_t t0 = 0;
  while ((int32_t)(ptx::ld_relaxed_sys(p) - target) < 0) {
    const uint64_t now = ptx::globaltimer();
    if (t0 == 0) t0 = now;
    if (now - t0 > kSpinLimitNs) return false;
    __nanosleep(32);
  }
  ptx::fence_acq_rel_sys();
  return true;
}

struct PeerKernelArgs {
  PeerStepArgs s;
  char* const* peers;       // [nprocs] region bases
  const int64_t* bounds;    // [k+1] segment bounds
  const int32_t* seg_t0;    // [k+1] first tile of each segment (seg_t0[k] = n_tiles)
  int n_tiles;
  int waves;
  int per_wave;             // m: units per CTA per wave
  uint32_t epoch;           // this step's epoch (>= 1)
  int mode;                 // 0 normal; diagnostics (wrong results): 1 local-only, 2 no waits
  int hint;                 // L2 evict-first policy on the x, m, g bulk loads
  size_t off_inbox, off_wbox, off_wave, off_done, off_count;
};

__device__ __forceinline__ float4 mom4(float4 m, float4 g, float mu) {
  return make_float4(__fadd_rn(__fmul_rn(mu, m.x), g.x), __fadd_rn(__fmul_rn(mu, m.y), g.y),
                     __fadd_rn(__fmul_rn(mu, m.z), g.z), __fadd_rn(__fmul_rn(mu, m.w), g.w));
}
__device__ __forceinline__ float4 sgd4(float4 x, float4 m, float lr) {
  return make_float4(__fsub_rn(x.x, __fmul_rn(lr, m.x)), __fsub_rn(x.y, __fmul_rn(lr, m.y)),
                     __fsub_rn(x.z, __fmul_rn(lr, m.z)), __fsub_rn(x.w, __fmul_rn(lr, m.w)));
}
__device__ __forceinline__ float4 mean4(float4 a, float4 b) {
  return make_float4(__fmul_rn(__fadd_rn(a.x, b.x), 0.5f), __fmul_rn(__fadd_rn(a.y, b.y), 0.5f),
                     __fmul_rn(__fadd_rn(a.z, b.z), 0.5f), __fmul_rn(__fadd_rn(a.w, b.w), 0.5f));
}
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
// default-policy store: y (read back by the mix while still in L2), remote inbox
__device__ __forceinline__ void st4(float* p, float4 v, int valid) {
  if (valid == 4) {
    *reinterpret_cast<float4*>(p) = v;
  } else {
    if (valid > 0) p[0] = v.x;
    if (valid > 1) p[1] = v.y;
    if (valid > 2) p[2] = v.z;
  }
}
__device__ __forceinline__ bool nonfinite4(float4 g) {
  const uint32_t e = 0x7f800000u;
  return ((__float_as_uint(g.x) & e) == e) | ((__float_as_uint(g.y) & e) == e) |
         ((__float_as_uint(g.z) & e) == e) | ((__float_as_uint(g.w) & e) == e);
}

// Shared-memory unit metadata and a per-role monotone cursor over segments.
struct Meta {
  const int64_t* bnd;   // [k+1]
  const int32_t* t0;    // [k+1]
  const int32_t* dstl;  // [k][n_loc] global receiver of local worker r in segment s
  bool dst_global;
};

struct Unit {
  int tile, r, seg, len;
  int64_t c0;
  bool first_tile;
};

__device__ __forceinline__ Unit unit_at(const PeerKernelArgs& a, const Meta& M, int u, int& cursor) {
  Unit x;
  x.tile = u / a.s.n_loc;
  x.r = u - x.tile * a.s.n_loc;
  while (M.t0[cursor + 1] <= x.tile) ++cursor;
  x.seg = cursor;
  const int64_t c0 = M.bnd[cursor] + (int64_t)(x.tile - M.t0[cursor]) * kPeerTile;
  const int64_t c1 = c0 + kPeerTile < M.bnd[cursor + 1] ? c0 + kPeerTile : M.bnd[cursor + 1];
  x.c0 = c0;
  x.len = (int)(c1 - c0);
  x.first_tile = x.tile == M.t0[cursor];
  return x;
}

// (receiver GPU, receiver's local index) of local worker r's segment seg
__device__ __forceinline__ void receiver_of(const PeerKernelArgs& a, const Meta& M, int seg, int r, int& rp,
                                            int& rl) {
  const PeerStepArgs& s = a.s;
  if (a.mode == 1) { rp = s.rank; rl = r; return; }
  const int recv = M.dst_global ? s.dst[(int64_t)seg * s.world + s.first + r] : M.dstl[seg * s.n_loc + r];
  rp = recv / s.n_loc;
  rl = recv - rp * s.n_loc;
}

__global__ void __launch_bounds__(kPeerThreads, 1) k_gossip_peer(const PeerKernelArgs a) {
  extern __shared__ __align__(128) float smem_f[];
  float* ringA = smem_f;  // [kStagesA][3][kPeerTile]
  __shared__ uint64_t a_full[kStagesA], a_empty[kStagesA];
  __shared__ uint64_t wave_done[kWaveSlots];
  __shared__ int s_timeout, s_released;

  const PeerStepArgs& s = a.s;
  const uint32_t e = a.epoch;
  const int par = (int)(e & 1u);
  char* mine = a.peers[s.rank];
  const int n_units = a.n_tiles * s.n_loc;
  const int G = gridDim.x;
  const int W = a.waves, m_per = a.per_wave;
  const int n_my = blockIdx.x < n_units ? (n_units - blockIdx.x + G - 1) / G : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  volatile int* timeout = &s_timeout;

  // ---- metadata into shared memory --------------------------------------------------
  int64_t* bnd = reinterpret_cast<int64_t*>(ringA + (size_t)kStagesA * 3 * kPeerTile);
  int32_t* t0 = reinterpret_cast<int32_t*>(bnd + s.k + 1);
  int32_t* dstl = t0 + s.k + 1;
  Meta M;
  M.bnd = bnd;
  M.t0 = t0;
  M.dstl = dstl;
  M.dst_global = (int64_t)s.k * s.n_loc > kMaxDstSmem;
  for (int i = threadIdx.x; i <= s.k; i += blockDim.x) {
    bnd[i] = a.bounds[i];
    t0[i] = a.seg_t0[i];
  }
  if (!M.dst_global)
    for (int i = threadIdx.x; i < s.k * s.n_loc; i += blockDim.x) {
      const int sg = i / s.n_loc, r = i - sg * s.n_loc;
      dstl[i] = s.dst[(int64_t)sg * s.world + s.first + r];
    }
  if (threadIdx.x == 0) {
    s_timeout = 0;
    s_released = 0;
    for (int i = 0; i < kStagesA; ++i) {
      ptx::mbar_init(&a_full[i], 1);
      ptx::mbar_init(&a_empty[i], kGroup / 32);
    }
    for (int i = 0; i < kWaveSlots; ++i) ptx::mbar_init(&wave_done[i], kGroup / 32);
    ptx::mbar_fence_init();
  }
  __syncthreads();
  // ping-pong safety: every receiver finished epoch e-2, the last reader of this parity
  if (threadIdx.x < s.nprocs && e >= 3) {
    const uint32_t* done = reinterpret_cast<const uint32_t*>(mine + a.off_done);
    if (!wait_acquire(done + threadIdx.x, e - 2)) atomicOr(&s_timeout, 1);
  }
  __syncthreads();

  if (warp < kGroup / 32) {
    // ---------------- push warps ------------------------------------------------
    bool bad = false;
    const int tid = threadIdx.x;
    int cur = 0;
    for (int w = 0; w < W; ++w) {
      const int i_end = (w + 1) * m_per < n_my ? (w + 1) * m_per : n_my;
      for (int i = w * m_per; i < i_end && !*timeout; ++i) {
        const Unit U = unit_at(a, M, blockIdx.x + i * G, cur);
        const int st = i % kStagesA;
        while (!ptx::mbar_try(&a_full[st], (uint32_t)((i / kStagesA) & 1)) && !*timeout) {
        }
        if (*timeout) break;
        const float* bx = ringA + (size_t)st * 3 * kPeerTile;
        int rp, rl;
        receiver_of(a, M, U.seg, U.r, rp, rl);
        float* inbox = reinterpret_cast<float*>(a.peers[rp] + a.off_inbox) + ((int64_t)par * s.n_loc + rl) * s.ld;
        const int64_t rowoff = (int64_t)U.r * s.ld;
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
          const int v = tid + q * kGroup;
          const int valid = U.len - 4 * v;
          if (valid > 0) {
            const int vv = valid < 4 ? valid : 4;
            const float4 cx = reinterpret_cast<const float4*>(bx)[v];
            const float4 cm = reinterpret_cast<const float4*>(bx + kPeerTile)[v];
            const float4 cg = reinterpret_cast<const float4*>(bx + 2 * kPeerTile)[v];
            bad |= nonfinite4(cg);
            const float4 mn = mom4(cm, cg, s.mu);
            const float4 y = sgd4(cx, mn, s.lr);
            const int64_t j = U.c0 + 4 * (int64_t)v;
            st4_cs(s.m + rowoff + j, mn, vv);
            st4(s.x + rowoff + j, y, vv);  // y, read back by the mix warps from L2
            st4(inbox + j, y, vv);         // NVLink push
          }
        }
        if (U.first_tile && tid == 0) {
          float* wbox = reinterpret_cast<float*>(a.peers[rp] + a.off_wbox) + ((int64_t)par * s.n_loc + rl) * s.k;
          wbox[U.seg] = s.psw[(int64_t)U.r * s.k + U.seg];
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&a_empty[st]);
      }
      // hand wave w to the release warp (it fences once and signals every GPU)
      __syncwarp();
      if (lane == 0) {
        volatile int* released = &s_released;
        while (*released <= w - kWaveSlots && !*timeout) {
        }
        ptx::mbar_arrive(&wave_done[w % kWaveSlots]);
      }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(s.err + kErrDiverged, 1);
  } else if (warp < 2 * kGroup / 32) {
    // ---------------- mix warps -------------------------------------------------
    const int tid = threadIdx.x - kGroup;
    const uint32_t expect = e * (uint32_t)G * (uint32_t)s.nprocs;  // arrivals per wave, cumulative
    int cur = 0;
    for (int w = 0; w < W; ++w) {
      if (tid == 0 && a.mode != 2) {
        const uint32_t* cnt = reinterpret_cast<const uint32_t*>(mine + a.off_wave) + w;
        if (!wait_acquire(cnt, expect)) *timeout = 1;
      }
      ptx::named_bar_sync(kBarMix, kGroup);
      if (*timeout) break;
      const int i_end = (w + 1) * m_per < n_my ? (w + 1) * m_per : n_my;
      for (int i = w * m_per; i < i_end; i += 2) {  // two units per pass: 4*kPer loads in flight
        Unit U[2];
        bool have[2];
        float4 yo[2][kPer], yi[2][kPer];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          have[h] = i + h < i_end;
          if (!have[h]) continue;
          U[h] = unit_at(a, M, blockIdx.x + (i + h) * G, cur);
          const float* inbox =
              reinterpret_cast<const float*>(mine + a.off_inbox) + ((int64_t)par * s.n_loc + U[h].r) * s.ld;
          const int64_t rowoff = (int64_t)U[h].r * s.ld;
#pragma unroll
          for (int q = 0; q < kPer; ++q) {
            const int vv = tid + q * kGroup;
            if (U[h].len - 4 * vv > 0) {
              const int64_t j = U[h].c0 + 4 * (int64_t)vv;
              yo[h][q] = __ldcg(reinterpret_cast<const float4*>(s.x + rowoff + j));
              yi[h][q] = __ldcg(reinterpret_cast<const float4*>(inbox + j));
            }
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (!have[h]) continue;
          const int64_t rowoff = (int64_t)U[h].r * s.ld;
#pragma unroll
          for (int q = 0; q < kPer; ++q) {
            const int vv = tid + q * kGroup;
            const int valid = U[h].len - 4 * vv;
            if (valid > 0) {
              const int64_t j = U[h].c0 + 4 * (int64_t)vv;
              st4_cs(s.x + rowoff + j, mean4(yo[h][q], yi[h][q]), valid < 4 ? valid : 4);
            }
          }
          if (U[h].first_tile && tid == 0) {
            const float* wbox =
                reinterpret_cast<const float*>(mine + a.off_wbox) + ((int64_t)par * s.n_loc + U[h].r) * s.k;
            float* wp = s.psw + (int64_t)U[h].r * s.k + U[h].seg;
            *wp = __fmul_rn(__fadd_rn(*wp, __ldcg(wbox + U[h].seg)), 0.5f);
          }
        }
      }
    }
  } else if (warp == 2 * kGroup / 32 + 1) {
    // ---------------- release warp: one fence per wave, then every GPU's counter -------
    for (int w = 0; w < W; ++w) {
      if (lane == 0)
        while (!ptx::mbar_try(&wave_done[w % kWaveSlots], (uint32_t)((w / kWaveSlots) & 1)) && !*timeout) {
        }
      __syncwarp();
      if (*timeout) break;
      if (lane < s.nprocs) {  // one fence instruction for the warp, then the arrivals
        ptx::fence_acq_rel_sys();
        uint32_t* cnt = reinterpret_cast<uint32_t*>(a.peers[lane] + a.off_wave) + w;
        ptx::red_add_relaxed_sys(cnt, 1u);
      }
      __syncwarp();
      if (lane == 0) *(volatile int*)&s_released = w + 1;
    }
  } else {
    // ---------------- load warp: x, m, g tiles of the next units ---------------------
    if (lane == 0) {
      const uint64_t pol = ptx::policy_evict_first();
      int cur = 0;
      for (int i = 0; i < n_my && !*timeout; ++i) {
        const Unit U = unit_at(a, M, blockIdx.x + i * G, cur);
        const int st = i % kStagesA;
        while (!ptx::mbar_try(&a_empty[st], (uint32_t)(((i / kStagesA) & 1) ^ 1)) && !*timeout) {
        }
        if (*timeout) break;
        const uint32_t bytes = (uint32_t)(((U.len + 3) & ~3) * 4);
        const int64_t off = (int64_t)U.r * s.ld + U.c0;
        float* buf = ringA + (size_t)st * 3 * kPeerTile;
        ptx::mbar_arrive_expect_tx(&a_full[st], 3 * bytes);
        if (a.hint) {
          ptx::bulk_g2s_hint(buf, s.x + off, bytes, &a_full[st], pol);
          ptx::bulk_g2s_hint(buf + kPeerTile, s.m + off, bytes, &a_full[st], pol);
          ptx::bulk_g2s_hint(buf + 2 * kPeerTile, s.g + off, bytes, &a_full[st], pol);
        } else {
          ptx::bulk_g2s(buf, s.x + off, bytes, &a_full[st]);
          ptx::bulk_g2s(buf + kPeerTile, s.m + off, bytes, &a_full[st]);
          ptx::bulk_g2s(buf + 2 * kPeerTile, s.g + off, bytes, &a_full[st]);
        }
      }
    }
    __syncwarp();
  }

  __syncthreads();
  if (threadIdx.x == 0 && s_timeout) atomicOr(s.err + kErrTimeout, 1);

  // ---- end of step: last CTA tells every peer this GPU finished epoch e ------------
  if (threadIdx.x == 0) {
    __threadfence();
    uint32_t* count = reinterpret_cast<uint32_t*>(mine + a.off_count);
    const uint32_t prevc = atomicAdd(count, 1u);
    if (prevc + 1 == e * gridDim.x) {
      __threadfence_system();
      for (int p = 0; p < s.nprocs; ++p) {
        uint32_t* done = reinterpret_cast<uint32_t*>(a.peers[p] + a.off_done) + s.rank;
        ptx::st_release_sys(done, e);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Two-kernel schedule (algo 2): a pure streaming push kernel, then a streaming
// mix kernel.  No per-tile or per-wave synchronisation at all: one
// system-scope signal per GPU per kernel.
//
//   k_peer_push  per unit (tile, local worker): bulk-TMA x, m, g -> m', y (a3);
//                m' -> HBM, y -> x (local), y -> the receiver's inbox (NVLink,
//                Alg.1 l.7); w_{i,s} -> the receiver's wbox.  The last CTA to
//                finish publishes push_done[rank] = e to every GPU (Alg.1 l.14).
//   k_peer_mix   waits until every GPU published push_done = e, then
//                x = (y + inbox) * 0.5, w = (w + wbox) * 0.5 (a5, Alg.1 l.17);
//                the last CTA publishes done[rank] = e (ping-pong safety).
// ---------------------------------------------------------------------------
constexpr int kPushCompute = 256;
constexpr int kPushThreads = kPushCompute + 32;
constexpr int kPushPer = kPeerTile / 4 / kPushCompute;

struct PushMixArgs {
  PeerKernelArgs k;
  size_t off_pdone, off_pcount;
};

// PULL: y goes only to this GPU's own exchange buffer; receivers pull it in k_peer_mix_pull.
template <bool PULL>
__global__ void __launch_bounds__(kPushThreads, 2) k_peer_push(const PushMixArgs pa) {
  const PeerKernelArgs& a = pa.k;
  extern __shared__ __align__(128) float smem_f[];
  float* ringA = smem_f;
  __shared__ uint64_t a_full[kStagesA], a_empty[kStagesA];
  __shared__ int s_timeout;
  const PeerStepArgs& s = a.s;
  const uint32_t e = a.epoch;
  const int par = (int)(e & 1u);
  char* mine = a.peers[s.rank];
  const int n_units = a.n_tiles * s.n_loc;
  const int G = gridDim.x;
  const int n_my = blockIdx.x < n_units ? (n_units - blockIdx.x + G - 1) / G : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  volatile int* timeout = &s_timeout;

  int64_t* bnd = reinterpret_cast<int64_t*>(ringA + (size_t)kStagesA * 3 * kPeerTile);
  int32_t* t0 = reinterpret_cast<int32_t*>(bnd + s.k + 1);
  int32_t* dstl = t0 + s.k + 1;
  Meta M;
  M.bnd = bnd;
  M.t0 = t0;
  M.dstl = dstl;
  M.dst_global = (int64_t)s.k * s.n_loc > kMaxDstSmem;
  for (int i = threadIdx.x; i <= s.k; i += blockDim.x) {
    bnd[i] = a.bounds[i];
    t0[i] = a.seg_t0[i];
  }
  if (!M.dst_global)
    for (int i = threadIdx.x; i < s.k * s.n_loc; i += blockDim.x) {
      const int sg = i / s.n_loc, r = i - sg * s.n_loc;
      dstl[i] = s.dst[(int64_t)sg * s.world + s.first + r];
    }
  if (threadIdx.x == 0) {
    s_timeout = 0;
    for (int i = 0; i < kStagesA; ++i) {
      ptx::mbar_init(&a_full[i], 1);
      ptx::mbar_init(&a_empty[i], kPushCompute / 32);
    }
    ptx::mbar_fence_init();
  }
  __syncthreads();
  // ping-pong safety: every receiver finished mixing epoch e-2 (last reader of this parity)
  if (threadIdx.x < s.nprocs && e >= 3) {
    const uint32_t* done = reinterpret_cast<const uint32_t*>(mine + a.off_done);
    if (!wait_acquire(done + threadIdx.x, e - 2)) atomicOr(&s_timeout, 1);
  }
  __syncthreads();

  if (warp < kPushCompute / 32) {
    bool bad = false;
    const int tid = threadIdx.x;
    int cur = 0;
    for (int i = 0; i < n_my && !*timeout; ++i) {
      const Unit U = unit_at(a, M, blockIdx.x + i * G, cur);
      const int st = i % kStagesA;
      ptx::mbar_wait(&a_full[st], (uint32_t)((i / kStagesA) & 1));
      const float* bx = ringA + (size_t)st * 3 * kPeerTile;
      int rp, rl;
      receiver_of(a, M, U.seg, U.r, rp, rl);
      float* inbox = PULL ? reinterpret_cast<float*>(mine + a.off_inbox) + ((int64_t)par * s.n_loc + U.r) * s.ld
                          : reinterpret_cast<float*>(a.peers[rp] + a.off_inbox) + ((int64_t)par * s.n_loc + rl) * s.ld;
      const int64_t rowoff = (int64_t)U.r * s.ld;
#pragma unroll
      for (int q = 0; q < kPushPer; ++q) {
        const int v = tid + q * kPushCompute;
        const int valid = U.len - 4 * v;
        if (valid > 0) {
          const int vv = valid < 4 ? valid : 4;
          const float4 cx = reinterpret_cast<const float4*>(bx)[v];
          const float4 cm = reinterpret_cast<const float4*>(bx + kPeerTile)[v];
          const float4 cg = reinterpret_cast<const float4*>(bx + 2 * kPeerTile)[v];
          bad |= nonfinite4(cg);
          const float4 mn = mom4(cm, cg, s.mu);
          const float4 y = sgd4(cx, mn, s.lr);
          const int64_t j = U.c0 + 4 * (int64_t)v;
          st4_cs(s.m + rowoff + j, mn, vv);
          if (!PULL) st4(s.x + rowoff + j, y, vv);
          st4(inbox + j, y, vv);  // PULL: own exchange buffer; else the receiver's inbox (NVLink)
        }
      }
      if (U.first_tile && tid == 0) {
        float* wbox = reinterpret_cast<float*>(a.peers[rp] + a.off_wbox) + ((int64_t)par * s.n_loc + rl) * s.k;
        wbox[U.seg] = s.psw[(int64_t)U.r * s.k + U.seg];
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&a_empty[st]);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(s.err + kErrDiverged, 1);
  } else if (lane == 0) {
    int cur = 0;
    for (int i = 0; i < n_my; ++i) {
      const Unit U = unit_at(a, M, blockIdx.x + i * G, cur);
      const int st = i % kStagesA;
      ptx::mbar_wait(&a_empty[st], (uint32_t)(((i / kStagesA) & 1) ^ 1));
      const uint32_t bytes = (uint32_t)(((U.len + 3) & ~3) * 4);
      const int64_t off = (int64_t)U.r * s.ld + U.c0;
      float* buf = ringA + (size_t)st * 3 * kPeerTile;
      ptx::mbar_arrive_expect_tx(&a_full[st], 3 * bytes);
      ptx::bulk_g2s(buf, s.x + off, bytes, &a_full[st]);
      ptx::bulk_g2s(buf + kPeerTile, s.m + off, bytes, &a_full[st]);
      ptx::bulk_g2s(buf + 2 * kPeerTile, s.g + off, bytes, &a_full[st]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_timeout) atomicOr(s.err + kErrTimeout, 1);
    __threadfence();
    uint32_t* count = reinterpret_cast<uint32_t*>(mine + pa.off_pcount);
    const uint32_t prevc = atomicAdd(count, 1u);
    if (prevc + 1 == e * gridDim.x) {  // every CTA's pushes are issued: publish them
      __threadfence_system();
      for (int p = 0; p < s.nprocs; ++p)
        ptx::st_release_sys(reinterpret_cast<uint32_t*>(a.peers[p] + pa.off_pdone) + s.rank, e);
    }
  }
}

__global__ void __launch_bounds__(256) k_peer_mix(const PushMixArgs pa) {
  const PeerKernelArgs& a = pa.k;
  const PeerStepArgs& s = a.s;
  const uint32_t e = a.epoch;
  const int par = (int)(e & 1u);
  char* mine = a.peers[s.rank];
  __shared__ int s_timeout;
  if (threadIdx.x == 0) s_timeout = 0;
  __syncthreads();
  if (threadIdx.x < s.nprocs && a.mode != 2) {
    const uint32_t* pd = reinterpret_cast<const uint32_t*>(mine + pa.off_pdone);
    if (!wait_acquire(pd + threadIdx.x, e)) atomicOr(&s_timeout, 1);
  }
  __syncthreads();
  if (!s_timeout) {
    const int64_t nv = (s.d + 3) >> 2;
    const int64_t total = nv * s.n_loc;
    const float* inbox0 = reinterpret_cast<const float*>(mine + a.off_inbox) + (int64_t)par * s.n_loc * s.ld;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; base < total; base += 2 * stride) {
      float4 yo[2], yi[2];
      int64_t off[2];
      int valid[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t idx = base + h * stride;
        valid[h] = 0;
        if (idx < total) {
          const int64_t r = idx / nv, v = idx - r * nv;
          const int64_t j = 4 * v;
          valid[h] = (int)imin64(4, s.d - j);
          off[h] = r * s.ld + j;
          yo[h] = __ldcs(reinterpret_cast<const float4*>(s.x + off[h]));
          yi[h] = __ldcs(reinterpret_cast<const float4*>(inbox0 + off[h]));
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (valid[h] > 0) st4_cs(s.x + off[h], mean4(yo[h], yi[h]), valid[h]);
    }
    if (blockIdx.x == 0) {
      for (int i = threadIdx.x; i < s.n_loc * s.k; i += blockDim.x) {
        const int r = i / s.k, sg = i - r * s.k;
        const float* wbox = reinterpret_cast<const float*>(mine + a.off_wbox) + ((int64_t)par * s.n_loc + r) * s.k;
        float* wp = s.psw + (int64_t)r * s.k + sg;
        *wp = __fmul_rn(__fadd_rn(*wp, __ldcg(wbox + sg)), 0.5f);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_timeout) atomicOr(s.err + kErrTimeout, 1);
    __threadfence();
    uint32_t* count = reinterpret_cast<uint32_t*>(mine + a.off_count);
    const uint32_t prevc = atomicAdd(count, 1u);
    if (prevc + 1 == e * gridDim.x) {
      __threadfence_system();
      for (int p = 0; p < s.nprocs; ++p)
        ptx::st_release_sys(reinterpret_cast<uint32_t*>(a.peers[p] + a.off_done) + s.rank, e);
    }
  }
}

// Push kernel with the NVLink transfer handed to the TMA engine (algo 4): compute
// warps write y into a shared-memory ring as well as into x; a store warp issues
// one 1-D bulk copy (cp.async.bulk.global.shared::cta) of each 8 KB y tile into
// the receiver's inbox, so the load/store units only carry the local traffic.
constexpr int kTStagesA = 3, kTSlotsY = 3;
constexpr int kTPushThreads = kPushCompute + 64;  // compute warps, load warp, store warp
constexpr size_t kTRingBytes = kTileBytes * (3 * kTStagesA + kTSlotsY);

size_t push_tma_smem_bytes(int k, int n_loc) {
  size_t b = kTRingBytes + sizeof(int64_t) * (k + 1) + sizeof(int32_t) * (k + 1);
  if ((int64_t)k * n_loc <= kMaxDstSmem) b += sizeof(int32_t) * (size_t)k * n_loc;
  return align_up(b, 16);
}

__global__ void __launch_bounds__(kTPushThreads, 2) k_peer_push_tma(const PushMixArgs pa) {
  const PeerKernelArgs& a = pa.k;
  extern __shared__ __align__(128) float smem_f[];
  float* ringA = smem_f;                                      // [kTStagesA][3][kPeerTile]
  float* ringY = ringA + (size_t)kTStagesA * 3 * kPeerTile;   // [kTSlotsY][kPeerTile]
  __shared__ uint64_t a_full[kTStagesA], a_empty[kTStagesA], y_full[kTSlotsY], y_empty[kTSlotsY];
  __shared__ int s_timeout;
  const PeerStepArgs& s = a.s;
  const uint32_t e = a.epoch;
  const int par = (int)(e & 1u);
  char* mine = a.peers[s.rank];
  const int n_units = a.n_tiles * s.n_loc;
  const int G = gridDim.x;
  const int n_my = blockIdx.x < n_units ? (n_units - blockIdx.x + G - 1) / G : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  volatile int* timeout = &s_timeout;

  int64_t* bnd = reinterpret_cast<int64_t*>(ringY + (size_t)kTSlotsY * kPeerTile);
  int32_t* t0 = reinterpret_cast<int32_t*>(bnd + s.k + 1);
  int32_t* dstl = t0 + s.k + 1;
  Meta M;
  M.bnd = bnd;
  M.t0 = t0;
  M.dstl = dstl;
  M.dst_global = (int64_t)s.k * s.n_loc > kMaxDstSmem;
  for (int i = threadIdx.x; i <= s.k; i += blockDim.x) {
    bnd[i] = a.bounds[i];
    t0[i] = a.seg_t0[i];
  }
  if (!M.dst_global)
    for (int i = threadIdx.x; i < s.k * s.n_loc; i += blockDim.x) {
      const int sg = i / s.n_loc, r = i - sg * s.n_loc;
      dstl[i] = s.dst[(int64_t)sg * s.world + s.first + r];
    }
  if (threadIdx.x == 0) {
    s_timeout = 0;
    for (int i = 0; i < kTStagesA; ++i) {
      ptx::mbar_init(&a_full[i], 1);
      ptx::mbar_init(&a_empty[i], kPushCompute / 32);
    }
    for (int i = 0; i < kTSlotsY; ++i) {
      ptx::mbar_init(&y_full[i], kPushCompute / 32);
      ptx::mbar_init(&y_empty[i], 1);
    }
    ptx::mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x < s.nprocs && e >= 3) {
    const uint32_t* done = reinterpret_cast<const uint32_t*>(mine + a.off_done);
    if (!wait_acquire(done + threadIdx.x, e - 2)) atomicOr(&s_timeout, 1);
  }
  __syncthreads();

  if (warp < kPushCompute / 32) {
    bool bad = false;
    const int tid = threadIdx.x;
    int cur = 0;
    for (int i = 0; i < n_my && !*timeout; ++i) {
      const Unit U = unit_at(a, M, blockIdx.x + i * G, cur);
      const int st = i % kTStagesA, sy = i % kTSlotsY;
      ptx::mbar_wait(&a_full[st], (uint32_t)((i / kTStagesA) & 1));
      ptx::mbar_wait(&y_empty[sy], (uint32_t)(((i / kTSlotsY) & 1) ^ 1));
      const float* bx = ringA + (size_t)st * 3 * kPeerTile;
      float4* yt = reinterpret_cast<float4*>(ringY + (size_t)sy * kPeerTile);
      const int64_t rowoff = (int64_t)U.r * s.ld;
#pragma unroll
      for (int q = 0; q < kPushPer; ++q) {
        const int v = tid + q * kPushCompute;
        const int valid = U.len - 4 * v;
        if (valid > 0) {
          const int vv = valid < 4 ? valid : 4;
          const float4 cx = reinterpret_cast<const float4*>(bx)[v];
          const float4 cm = reinterpret_cast<const float4*>(bx + kPeerTile)[v];
          const float4 cg = reinterpret_cast<const float4*>(bx + 2 * kPeerTile)[v];
          bad |= nonfinite4(cg);
          const float4 mn = mom4(cm, cg, s.mu);
          const float4 y = sgd4(cx, mn, s.lr);
          const int64_t j = U.c0 + 4 * (int64_t)v;
          st4_cs(s.m + rowoff + j, mn, vv);
          st4(s.x + rowoff + j, y, vv);
          yt[v] = y;
        }
      }
      if (U.first_tile && tid == 0) {
        int rp, rl;
        receiver_of(a, M, U.seg, U.r, rp, rl);
        float* wbox = reinterpret_cast<float*>(a.peers[rp] + a.off_wbox) + ((int64_t)par * s.n_loc + rl) * s.k;
        wbox[U.seg] = s.psw[(int64_t)U.r * s.k + U.seg];
      }
      ptx::fence_proxy_async_shared();  // y tile -> the TMA engine's reads
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive(&a_empty[st]);
        ptx::mbar_arrive(&y_full[sy]);
      }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(s.err + kErrDiverged, 1);
  } else if (warp == kPushCompute / 32) {
    if (lane == 0) {  // load warp
      int cur = 0;
      for (int i = 0; i < n_my; ++i) {
        const Unit U = unit_at(a, M, blockIdx.x + i * G, cur);
        const int st = i % kTStagesA;
        ptx::mbar_wait(&a_empty[st], (uint32_t)(((i / kTStagesA) & 1) ^ 1));
        const uint32_t bytes = (uint32_t)(((U.len + 3) & ~3) * 4);
        const int64_t off = (int64_t)U.r * s.ld + U.c0;
        float* buf = ringA + (size_t)st * 3 * kPeerTile;
        ptx::mbar_arrive_expect_tx(&a_full[st], 3 * bytes);
        ptx::bulk_g2s(buf, s.x + off, bytes, &a_full[st]);
        ptx::bulk_g2s(buf + kPeerTile, s.m + off, bytes, &a_full[st]);
        ptx::bulk_g2s(buf + 2 * kPeerTile, s.g + off, bytes, &a_full[st]);
      }
    }
    __syncwarp();
  } else {
    if (lane == 0) {  // store warp: y tiles -> receivers' inboxes over NVLink
      int cur = 0;
      for (int i = 0; i < n_my; ++i) {
        const Unit U = unit_at(a, M, blockIdx.x + i * G, cur);
        const int sy = i % kTSlotsY;
        ptx::mbar_wait(&y_full[sy], (uint32_t)((i / kTSlotsY) & 1));
        int rp, rl;
        receiver_of(a, M, U.seg, U.r, rp, rl);
        float* inbox = reinterpret_cast<float*>(a.peers[rp] + a.off_inbox) + ((int64_t)par * s.n_loc + rl) * s.ld;
        ptx::bulk_s2g(inbox + U.c0, ringY + (size_t)sy * kPeerTile, (uint32_t)(((U.len + 3) & ~3) * 4));
        ptx::bulk_commit();
        ptx::bulk_wait_read<1>();  // groups up to i-1 have read their tiles
        if (i >= 1) ptx::mbar_arrive(&y_empty[(i - 1) % kTSlotsY]);
      }
      ptx::bulk_wait_all();  // every y tile has landed in its receiver's inbox
      asm volatile("fence.proxy.async.global;" ::: "memory");
      if (n_my >= 1) ptx::mbar_arrive(&y_empty[(n_my - 1) % kTSlotsY]);
    }
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_timeout) atomicOr(s.err + kErrTimeout, 1);
    __threadfence();
    uint32_t* count = reinterpret_cast<uint32_t*>(mine + pa.off_pcount);
    const uint32_t prevc = atomicAdd(count, 1u);
    if (prevc + 1 == e * gridDim.x) {  // every CTA's pushes have landed: publish them
      __threadfence_system();
      for (int p = 0; p < s.nprocs; ++p)
        ptx::st_release_sys(reinterpret_cast<uint32_t*>(a.peers[p] + pa.off_pdone) + s.rank, e);
    }
  }
}

// Fused push + mix (algo 5): k_peer_push_tma plus 4 mix warps.  Units are cut into
// W waves of m units per CTA (G*m a multiple of n_loc: a tile never straddles two
// waves).  After the last bulk store of wave w has completed, the store warp
// fences once and adds 1 to wave w's arrival counter on every GPU; the mix warps
// mix wave w once its counter holds every CTA of every GPU, overlapping the
// NVLink-bound pushes of later waves.
constexpr int kMixWarps = 4;
constexpr int kFThreads = kPushCompute + 64 + 32 * kMixWarps;

__global__ void __launch_bounds__(kFThreads, 1) k_peer_fused(const PushMixArgs pa) {
  const PeerKernelArgs& a = pa.k;
  extern __shared__ __align__(128) float smem_f[];
  float* ringA = smem_f;
  float* ringY = ringA + (size_t)kTStagesA * 3 * kPeerTile;
  __shared__ uint64_t a_full[kTStagesA], a_empty[kTStagesA], y_full[kTSlotsY], y_empty[kTSlotsY];
  __shared__ int s_timeout;
  const PeerStepArgs& s = a.s;
  const uint32_t e = a.epoch;
  const int par = (int)(e & 1u);
  char* mine = a.peers[s.rank];
  const int n_units = a.n_tiles * s.n_loc;
  const int G = gridDim.x;
  const int W = a.waves, m_per = a.per_wave;
  const int n_my = blockIdx.x < n_units ? (n_units - blockIdx.x + G - 1) / G : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  volatile int* timeout = &s_timeout;

  int64_t* bnd = reinterpret_cast<int64_t*>(ringY + (size_t)kTSlotsY * kPeerTile);
  int32_t* t0 = reinterpret_cast<int32_t*>(bnd + s.k + 1);
  int32_t* dstl = t0 + s.k + 1;
  Meta M;
  M.bnd = bnd;
  M.t0 = t0;
  M.dstl = dstl;
  M.dst_global = (int64_t)s.k * s.n_loc > kMaxDstSmem;
  for (int i = threadIdx.x; i <= s.k; i += blockDim.x) {
    bnd[i] = a.bounds[i];
    t0[i] = a.seg_t0[i];
  }
  if (!M.dst_global)
    for (int i = threadIdx.x; i < s.k * s.n_loc; i += blockDim.x) {
      const int sg = i / s.n_loc, r = i - sg * s.n_loc;
      dstl[i] = s.dst[(int64_t)sg * s.world + s.first + r];
    }
  if (threadIdx.x == 0) {
    s_timeout = 0;
    for (int i = 0; i < kTStagesA; ++i) {
      ptx::mbar_init(&a_full[i], 1);
      ptx::mbar_init(&a_empty[i], kPushCompute / 32);
    }
    for (int i = 0; i < kTSlotsY; ++i) {
      ptx::mbar_init(&y_full[i], kPushCompute / 32);
      ptx::mbar_init(&y_empty[i], 1);
    }
    ptx::mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x < s.nprocs && e >= 3) {
    const uint32_t* done = reinterpret_cast<const uint32_t*>(mine + a.off_done);
    if (!wait_acquire(done + threadIdx.x, e - 2)) atomicOr(&s_timeout, 1);
  }
  __syncthreads();

  constexpr int kLoadWarp = kPushCompute / 32, kStoreWarp = kLoadWarp + 1, kMix0 = kStoreWarp + 1;
  if (warp < kLoadWarp) {
    // ---------------- compute warps: m', y; y -> x and the y ring --------------------
    bool bad = false;
    const int tid = threadIdx.x;
    int cur = 0;
    for (int i = 0; i < n_my && !*timeout; ++i) {
      const Unit U = unit_at(a, M, blockIdx.x + i * G, cur);
      const int st = i % kTStagesA, sy = i % kTSlotsY;
      ptx::mbar_wait(&a_full[st], (uint32_t)((i / kTStagesA) & 1));
      ptx::mbar_wait(&y_empty[sy], (uint32_t)(((i / kTSlotsY) & 1) ^ 1));
      const float* bx = ringA + (size_t)st * 3 * kPeerTile;
      float4* yt = reinterpret_cast<float4*>(ringY + (size_t)sy * kPeerTile);
      const int64_t rowoff = (int64_t)U.r * s.ld;
#pragma unroll
      for (int q = 0; q < kPushPer; ++q) {
        const int v = tid + q * kPushCompute;
        const int valid = U.len - 4 * v;
        if (valid > 0) {
          const int vv = valid < 4 ? valid : 4;
          const float4 cx = reinterpret_cast<const float4*>(bx)[v];
          const float4 cm = reinterpret_cast<const float4*>(bx + kPeerTile)[v];
          const float4 cg = reinterpret_cast<const float4*>(bx + 2 * kPeerTile)[v];
          bad |= nonfinite4(cg);
          const float4 mn = mom4(cm, cg, s.mu);
          const float4 y = sgd4(cx, mn, s.lr);
          const int64_t j = U.c0 + 4 * (int64_t)v;
          st4_cs(s.m + rowoff + j, mn, vv);
          st4(s.x + rowoff + j, y, vv);
          yt[v] = y;
        }
      }
      if (U.first_tile && tid == 0) {
        int rp, rl;
        receiver_of(a, M, U.seg, U.r, rp, rl);
        float* wbox = reinterpret_cast<float*>(a.peers[rp] + a.off_wbox) + ((int64_t)par * s.n_loc + rl) * s.k;
        wbox[U.seg] = s.psw[(int64_t)U.r * s.k + U.seg];
      }
      ptx::fence_proxy_async_shared();
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive(&a_empty[st]);
        ptx::mbar_arrive(&y_full[sy]);
      }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(s.err + kErrDiverged, 1);
  } else if (warp == kLoadWarp) {
    if (lane == 0) {
      int cur = 0;
      for (int i = 0; i < n_my; ++i) {
        const Unit U = unit_at(a, M, blockIdx.x + i * G, cur);
        const int st = i % kTStagesA;
        ptx::mbar_wait(&a_empty[st], (uint32_t)(((i / kTStagesA) & 1) ^ 1));
        const uint32_t bytes = (uint32_t)(((U.len + 3) & ~3) * 4);
        const int64_t off = (int64_t)U.r * s.ld + U.c0;
        float* buf = ringA + (size_t)st * 3 * kPeerTile;
        ptx::mbar_arrive_expect_tx(&a_full[st], 3 * bytes);
        ptx::bulk_g2s(buf, s.x + off, bytes, &a_full[st]);
        ptx::bulk_g2s(buf + kPeerTile, s.m + off, bytes, &a_full[st]);
        ptx::bulk_g2s(buf + 2 * kPeerTile, s.g + off, bytes, &a_full[st]);
      }
    }
    __syncwarp();
  } else if (warp == kStoreWarp) {
    // ---------------- store warp: y tiles -> inboxes; release each finished wave -----
    if (lane == 0) {
      int cur = 0, i = 0, rel = 0;  // rel: next unit whose y slot goes back to the compute warps
      for (int w = 0; w < W; ++w) {
        const int i_end = (w + 1) * m_per < n_my ? (w + 1) * m_per : n_my;
        for (; i < i_end; ++i) {
          const Unit U = unit_at(a, M, blockIdx.x + i * G, cur);
          const int sy = i % kTSlotsY;
          ptx::mbar_wait(&y_full[sy], (uint32_t)((i / kTSlotsY) & 1));
          int rp, rl;
          receiver_of(a, M, U.seg, U.r, rp, rl);
          float* inbox = reinterpret_cast<float*>(a.peers[rp] + a.off_inbox) + ((int64_t)par * s.n_loc + rl) * s.ld;
          ptx::bulk_s2g(inbox + U.c0, ringY + (size_t)sy * kPeerTile, (uint32_t)(((U.len + 3) & ~3) * 4));
          ptx::bulk_commit();
          ptx::bulk_wait_read<1>();  // groups of units < i have read their tiles
          for (; rel < i; ++rel) ptx::mbar_arrive(&y_empty[rel % kTSlotsY]);
        }
        ptx::bulk_wait_all();  // wave w's tiles have landed
        asm volatile("fence.proxy.async.global;" ::: "memory");
        for (; rel < i; ++rel) ptx::mbar_arrive(&y_empty[rel % kTSlotsY]);
        // the compute warps' x stores of this wave are ordered by y_full (acquire.cta) + the fence below
        ptx::fence_acq_rel_sys();
        for (int p = 0; p < s.nprocs; ++p)
          ptx::red_add_relaxed_sys(reinterpret_cast<uint32_t*>(a.peers[p] + a.off_wave) + w, 1u);
      }
    }
    __syncwarp();
  } else {
    // ---------------- mix warps: wave w once every GPU has pushed it ------------------
    const int tid = threadIdx.x - 32 * kMix0;
    constexpr int kMixThreads = 32 * kMixWarps;
    constexpr int kMixPer = kPeerTile / 4 / kMixThreads;
    const uint32_t expect = e * (uint32_t)G * (uint32_t)s.nprocs;
    int cur = 0;
    for (int w = 0; w < W; ++w) {
      if (tid == 0 && a.mode != 2) {
        const uint32_t* cnt = reinterpret_cast<const uint32_t*>(mine + a.off_wave) + w;
        if (!wait_acquire(cnt, expect)) *timeout = 1;
      }
      ptx::named_bar_sync(kBarMix, kMixThreads);
      if (*timeout) break;
      const int i_end = (w + 1) * m_per < n_my ? (w + 1) * m_per : n_my;
      for (int i = w * m_per; i < i_end; ++i) {
        const Unit U = unit_at(a, M, blockIdx.x + i * G, cur);
        const float* inbox =
            reinterpret_cast<const float*>(mine + a.off_inbox) + ((int64_t)par * s.n_loc + U.r) * s.ld;
        const int64_t rowoff = (int64_t)U.r * s.ld;
        float4 yo[kMixPer], yi[kMixPer];
#pragma unroll
        for (int q = 0; q < kMixPer; ++q) {
          const int vv = tid + q * kMixThreads;
          if (U.len - 4 * vv > 0) {
            const int64_t j = U.c0 + 4 * (int64_t)vv;
            yo[q] = __ldcg(reinterpret_cast<const float4*>(s.x + rowoff + j));
            yi[q] = __ldcg(reinterpret_cast<const float4*>(inbox + j));
          }
        }
#pragma unroll
        for (int q = 0; q < kMixPer; ++q) {
          const int vv = tid + q * kMixThreads;
          const int valid = U.len - 4 * vv;
          if (valid > 0) {
            const int64_t j = U.c0 + 4 * (int64_t)vv;
            st4_cs(s.x + rowoff + j, mean4(yo[q], yi[q]), valid < 4 ? valid : 4);
          }
        }
        if (U.first_tile && tid == 0) {
          const float* wbox =
              reinterpret_cast<const float*>(mine + a.off_wbox) + ((int64_t)par * s.n_loc + U.r) * s.k;
          float* wp = s.psw + (int64_t)U.r * s.k + U.seg;
          *wp = __fmul_rn(__fadd_rn(*wp, __ldcg(wbox + U.seg)), 0.5f);
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_timeout) atomicOr(s.err + kErrTimeout, 1);
    __threadfence();
    uint32_t* count = reinterpret_cast<uint32_t*>(mine + a.off_count);
    const uint32_t prevc = atomicAdd(count, 1u);
    if (prevc + 1 == e * gridDim.x) {
      __threadfence_system();
      for (int p = 0; p < s.nprocs; ++p)
        ptx::st_release_sys(reinterpret_cast<uint32_t*>(a.peers[p] + a.off_done) + s.rank, e);
    }
  }
}

// Pull variant of the mix: x_i = (y_i + y_{src_s(i)}) * 0.5 with y_src read straight
// from the source GPU's exchange buffer over NVLink (128-bit peer loads).
__global__ void __launch_bounds__(256) k_peer_mix_pull(const PushMixArgs pa) {
  const PeerKernelArgs& a = pa.k;
  const PeerStepArgs& s = a.s;
  const uint32_t e = a.epoch;
  const int par = (int)(e & 1u);
  char* mine = a.peers[s.rank];
  __shared__ int s_timeout;
  if (threadIdx.x == 0) s_timeout = 0;
  __syncthreads();
  if (threadIdx.x < s.nprocs && a.mode != 2) {
    const uint32_t* pd = reinterpret_cast<const uint32_t*>(mine + pa.off_pdone);
    if (!wait_acquire(pd + threadIdx.x, e)) atomicOr(&s_timeout, 1);
  }
  __syncthreads();
  if (!s_timeout) {
    const int64_t nv = (s.d + 3) >> 2;
    const int64_t total = nv * s.n_loc;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; base < total; base += 2 * stride) {
      float4 yo[2], yi[2];
      int64_t off[2];
      int valid[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t idx = base + h * stride;
        valid[h] = 0;
        if (idx < total) {
          const int64_t r = idx / nv, v = idx - r * nv;
          const int64_t j = 4 * v;
          const int64_t q = j >> 5;
          const int seg = (int)imin64(s.k - 1, ((q + 1) * s.k - 1) / s.nq);
          const int src = s.src[(int64_t)seg * s.world + s.first + (int)r];
          const int sp = src / s.n_loc, sl = src - sp * s.n_loc;
          valid[h] = (int)imin64(4, s.d - j);
          off[h] = r * s.ld + j;
          yo[h] = __ldcs(reinterpret_cast<const float4*>(mine + a.off_inbox) + (((int64_t)par * s.n_loc + r) * s.ld + j) / 4);
          yi[h] = __ldcg(reinterpret_cast<const float4*>(a.peers[sp] + a.off_inbox) +
                         (((int64_t)par * s.n_loc + sl) * s.ld + j) / 4);
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (valid[h] > 0) st4_cs(s.x + off[h], mean4(yo[h], yi[h]), valid[h]);
    }
    if (blockIdx.x == 0) {
      for (int i = threadIdx.x; i < s.n_loc * s.k; i += blockDim.x) {
        const int r = i / s.k, sg = i - r * s.k;
        const float* wbox = reinterpret_cast<const float*>(mine + a.off_wbox) + ((int64_t)par * s.n_loc + r) * s.k;
        float* wp = s.psw + (int64_t)r * s.k + sg;
        *wp = __fmul_rn(__fadd_rn(*wp, __ldcg(wbox + sg)), 0.5f);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_timeout) atomicOr(s.err + kErrTimeout, 1);
    __threadfence();
    uint32_t* count = reinterpret_cast<uint32_t*>(mine + a.off_count);
    const uint32_t prevc = atomicAdd(count, 1u);
    if (prevc + 1 == e * gridDim.x) {
      __threadfence_system();
      for (int p = 0; p < s.nprocs; ++p)
        ptx::st_release_sys(reinterpret_cast<uint32_t*>(a.peers[p] + a.off_done) + s.rank, e);
    }
  }
}

int gcd_int(int a, int b) {
  while (b) {
    const int t = a % b;
    a = b;
    b = t;
  }
  return a;
}

}  // namespace

const char* peer_error() { return g_peer_err.c_str(); }

int peer_alloc(PeerState& p, int n_loc, int64_t d, int64_t ld, int k, int nprocs, int rank) {
  p = PeerState();
  p.nprocs = nprocs;
  p.rank = rank;
  p.n_loc = n_loc;
  p.k = k;
  p.ld = ld;
  p.tile = kPeerTile;
  const char* mode = getenv("CS_PEER_MODE");
  p.mode = mode ? atoi(mode) : 0;
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

  const size_t smem = peer_smem_bytes(k, n_loc);
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaFuncSetAttribute(k_gossip_peer, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return perr(CS_ECUDA, "smem attribute", e);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gossip_peer, kPeerThreads, smem);
  if (e != cudaSuccess || occ < 1) return perr(CS_ECUDA, "occupancy", e);
  p.grid = sms * occ;
  const int n_units = p.n_tiles * n_loc;
  if (p.grid > n_units) p.grid = n_units;
  const char* algo = getenv("CS_PEER_ALGO");
  p.algo = algo ? atoi(algo) : 0;
  if (p.algo == 5) {  // fused push+mix kernel: its own grid defines the waves
    const size_t smem_f = push_tma_smem_bytes(k, n_loc);
    int occ_f = 0;
    e = cudaFuncSetAttribute(k_peer_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_f);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_f, k_peer_fused, kFThreads, smem_f);
    if (e != cudaSuccess || occ_f < 1) return perr(CS_ECUDA, "fused occupancy", e);
    p.grid = sms * occ_f;
    if (p.grid > n_units) p.grid = n_units;
  }
  // waves of G*m units, G*m a multiple of n_loc (tiles never straddle waves), ~kWaveBytes each
  const int step_m = n_loc / gcd_int(p.grid, n_loc);
  const double unit_bytes = 28.0 * kPeerTile;
  const char* wmb = getenv("CS_PEER_WAVE_MB");  // tuning knob
  const double wave_bytes = wmb ? atof(wmb) * 1024 * 1024 : kWaveBytes;
  int m = (int)(wave_bytes / unit_bytes / p.grid + 0.5);
  if (m < 1) m = 1;
  m = (m + step_m - 1) / step_m * step_m;
  p.per_wave = m;
  p.waves = (n_units + p.grid * m - 1) / (p.grid * m);

  p.off_inbox = 0;
  p.off_wbox = align_up(p.off_inbox + sizeof(float) * 2 * (size_t)n_loc * ld, 256);
  p.off_wave = align_up(p.off_wbox + sizeof(float) * 2 * (size_t)n_loc * k, 256);
  p.off_done = align_up(p.off_wave + sizeof(uint32_t) * (size_t)p.waves, 256);
  p.off_count = align_up(p.off_done + sizeof(uint32_t) * (size_t)nprocs, 256);
  p.off_pdone = align_up(p.off_count + 256, 256);
  p.off_pcount = align_up(p.off_pdone + sizeof(uint32_t) * (size_t)nprocs, 256);
  p.off_flags = p.off_count;  // unused by this protocol
  p.bytes = align_up(p.off_pcount + 256, 4096);
  {
    int occ_push = 0, occ_mix = 0;
    e = cudaFuncSetAttribute(k_peer_push<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_peer_push<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_push, k_peer_push<false>, kPushThreads, smem);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_mix, k_peer_mix, 256, 0);
    if (e != cudaSuccess || occ_push < 1 || occ_mix < 1) return perr(CS_ECUDA, "push/mix occupancy", e);
    if (p.algo == 4) {  // TMA-store push kernel has its own footprint
      const size_t smem_t = push_tma_smem_bytes(k, n_loc);
      e = cudaFuncSetAttribute(k_peer_push_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_t);
      if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_push, k_peer_push_tma, kTPushThreads, smem_t);
      if (e != cudaSuccess || occ_push < 1) return perr(CS_ECUDA, "push-tma occupancy", e);
    }
    p.grid_push = sms * occ_push;
    if (p.grid_push > n_units) p.grid_push = n_units;
    p.grid_mix = sms * occ_mix;
  }
  e = cudaMalloc(&p.base, p.bytes);
  if (e != cudaSuccess) return perr(CS_ECUDA, "peer region cudaMalloc", e);
  e = cudaMemset(p.base, 0, p.bytes);
  if (e != cudaSuccess) return perr(CS_ECUDA, "peer region memset", e);
  e = cudaMalloc(&p.d_bounds, sizeof(int64_t) * (k + 1));
  if (e == cudaSuccess) e = cudaMalloc(&p.d_seg_t0, sizeof(int32_t) * (k + 1));
  if (e == cudaSuccess)
    e = cudaMemcpy(p.d_bounds, bounds.data(), sizeof(int64_t) * (k + 1), cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(p.d_seg_t0, seg_t0.data(), sizeof(int32_t) * (k + 1), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return perr(CS_ECUDA, "tile tables", e);
  p.peer_base.assign(nprocs, nullptr);
  p.peer_base[rank] = p.base;
  p.allocated = true;
  return CS_OK;
}

void peer_release(PeerState& p) {
  if (p.imported) {
    for (int r = 0; r < p.nprocs; ++r)
      if (r != p.rank && p.peer_base[r]) cudaIpcCloseMemHandle(p.peer_base[r]);
  }
  if (p.base) cudaFree(p.base);
  if (p.d_peer_base) cudaFree(p.d_peer_base);
  if (p.d_tiles) cudaFree(p.d_tiles);
  if (p.d_tile_end) cudaFree(p.d_tile_end);
  if (p.d_bounds) cudaFree(p.d_bounds);
  if (p.d_seg_t0) cudaFree(p.d_seg_t0);
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
  for (int r = 0; r < p.nprocs; ++r) {
    if (r == p.rank) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, all + (size_t)r * CS_IPC_HANDLE_BYTES, sizeof(h));
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return perr(CS_ECUDA, "cudaIpcOpenMemHandle", e);
    p.peer_base[r] = (char*)ptr;
  }
  cudaError_t e = cudaMalloc(&p.d_peer_base, sizeof(char*) * p.nprocs);
  if (e == cudaSuccess)
    e = cudaMemcpy(p.d_peer_base, p.peer_base.data(), sizeof(char*) * p.nprocs,
                   cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return perr(CS_ECUDA, "peer table", e);
  p.imported = true;
  return CS_OK;
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

int peer_flat_step(PeerState& p, const PeerStepArgs& a, cudaStream_t st, cudaEvent_t ev0,
                   cudaEvent_t ev1) {
  TopoArgs t;
  t.seed = a.seed;
  t.step = a.step;
  t.n = a.world;
  t.k = a.k;
  t.tag = CS_TAG_FLAT;
  t.given = a.given;
  t.src = a.src;
  t.dst = a.dst;
  t.ord = nullptr;
  t.psw = nullptr;
  t.group_size = 1;
  t.rw = nullptr;
  t.inv_wsum = nullptr;
  t.err = a.err;
  cudaError_t e = launch_topology(t, st);
  if (e != cudaSuccess) return perr(CS_ECUDA, "topology launch", e);

  PeerKernelArgs ka;
  ka.s = a;
  ka.peers = p.d_peer_base;
  ka.bounds = p.d_bounds;
  ka.seg_t0 = p.d_seg_t0;
  ka.n_tiles = p.n_tiles;
  ka.waves = p.waves;
  ka.per_wave = p.per_wave;
  ka.epoch = ++p.epoch;
  ka.mode = p.mode & 3;
  ka.hint = (p.mode & 4) ? 0 : 1;
  ka.off_inbox = p.off_inbox;
  ka.off_wbox = p.off_wbox;
  ka.off_wave = p.off_wave;
  ka.off_done = p.off_done;
  ka.off_count = p.off_count;
  if (p.algo == 5) {
    PushMixArgs pm;
    pm.k = ka;
    pm.off_pdone = p.off_pdone;
    pm.off_pcount = p.off_pcount;
    if (ev0) cudaEventRecord(ev0, st);
    k_peer_fused<<<p.grid, kFThreads, push_tma_smem_bytes(a.k, a.n_loc), st>>>(pm);
    e = cudaGetLastError();
    if (e != cudaSuccess) return perr(CS_ECUDA, "fused launch", e);
    if (ev1) cudaEventRecord(ev1, st);
    return CS_OK;
  }
  if (p.algo == 2 || p.algo == 3 || p.algo == 4) {
    const bool pull = p.algo == 3;
    PushMixArgs pm;
    pm.k = ka;
    pm.off_pdone = p.off_pdone;
    pm.off_pcount = p.off_pcount;
    static const bool time_push_only = getenv("CS_PEER_TIME_PUSH") != nullptr;  // tuning knob
    if (ev0) cudaEventRecord(ev0, st);
    if (p.algo == 4) k_peer_push_tma<<<p.grid_push, kTPushThreads, push_tma_smem_bytes(a.k, a.n_loc), st>>>(pm);
    else if (pull) k_peer_push<true><<<p.grid_push, kPushThreads, peer_smem_bytes(a.k, a.n_loc), st>>>(pm);
    else k_peer_push<false><<<p.grid_push, kPushThreads, peer_smem_bytes(a.k, a.n_loc), st>>>(pm);
    if (ev1 && time_push_only) cudaEventRecord(ev1, st);
    if (pull) k_peer_mix_pull<<<p.grid_mix, 256, 0, st>>>(pm);
    else k_peer_mix<<<p.grid_mix, 256, 0, st>>>(pm);
    e = cudaGetLastError();
    if (e != cudaSuccess) return perr(CS_ECUDA, "push/mix launch", e);
    if (ev1 && !time_push_only) cudaEventRecord(ev1, st);
    return CS_OK;
  }
  void* args[] = {&ka};
  if (ev0) cudaEventRecord(ev0, st);
  e = cudaLaunchCooperativeKernel((const void*)k_gossip_peer, dim3(p.grid), dim3(kPeerThreads), args,
                                  peer_smem_bytes(a.k, a.n_loc), st);
  if (e != cudaSuccess) return perr(CS_ECUDA, "cooperative launch", e);
  if (ev1) cudaEventRecord(ev1, st);
  return CS_OK;
}

}  // namespace cs
