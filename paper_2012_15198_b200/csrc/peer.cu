// Multi-GPU flat step over NVLink peer memory (configs 3 and 5).
//
// Workers are partitioned contiguously: worker w lives on GPU w / n_loc.  At step
// t each GPU runs ONE persistent kernel (cooperative launch, so every CTA is
// co-resident; one CTA per SM).  The work unit is (tile q, local worker r): a
// segment-aligned range of up to kPeerTile columns of one worker's vector.
// Units are numbered tile-major (u = q * n_loc + r) and CTA c takes units
// c, c + G, c + 2G, ... on every GPU.
//
// Warp-specialised CTA, every hand-off through shared-memory mbarriers:
//
//   load warp      bulk-TMA of x, m, g row-tiles of the next units into a
//                  kStagesA-deep ring (cp.async.bulk, 8 KB per array per unit).
//   compute warps  unit i, push: m', y (a3) from the staged tiles; m' -> HBM;
//                  y -> the RECEIVER's inbox on the receiver's GPU (NVLink store;
//                  Alg.1 l.7 isend to send_to = dst_s(i)) and
//                  -> a y ring slot; first tile of a segment also pushes w_{i,s}.
//                  unit i-kLag, mix: x = (y + inbox) * 0.5, w = (w + wbox) * 0.5
//                  (a5, Alg.1 l.17), the inbox tile already staged in smem.
//   signal warp    releases the receivers' flags of every pushed unit (the irecv
//                  completion, Alg.1 l.14) — one fence.acq_rel.sys per batch of
//                  pushed units, then relaxed flag stores; polls its own inbound
//                  flags relaxed and, after one fence per batch, bulk-TMAs the
//                  inbox tiles into the B ring.  It never blocks one queue on the
//                  other.
//
// All unit metadata (segment bounds, first tile of each segment, receivers of
// the local workers) lives in shared memory, so the single-lane producer and
// signal loops issue no dependent global loads.
//
// Deadlock freedom: a push never waits on another GPU; a mix of unit j waits
// for the push of unit j on its source GPU, which is a unit of the same tile;
// every CTA holds at most one unit per tile (G >= n_loc) and visits tiles in
// increasing order on every GPU, all CTAs are resident, so by induction on the
// tile index every push is eventually issued.
//
// The inbox ping-pongs on step parity; before pushing at epoch e a GPU waits
// until every peer has finished epoch e-2 (the last reader of that parity) —
// the "done" words each GPU writes into every peer's region at the end of a
// step.  Flags and done words carry the monotone epoch, so nothing is reset.
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

constexpr int kCompute = 256;                   // 8 compute warps
constexpr int kPeerThreads = kCompute + 64;     // + load warp + signal warp
constexpr int kPeerTile = 2048;                 // columns per unit: 8 KB of one worker's row
constexpr int kPer = kPeerTile / 4 / kCompute;  // float4 per compute thread per array
constexpr int kStagesA = 4;                     // x, m, g ring depth (units)
constexpr int kLag = 3;                         // mix trails push by kLag units
constexpr int kSlotsY = kLag + 1;               // y ring slots
constexpr int kStagesB = 4;                     // inbox ring depth (units)
constexpr size_t kTileBytes = sizeof(float) * kPeerTile;
constexpr size_t kRingBytes = kTileBytes * (3 * kStagesA + kSlotsY + kStagesB);
constexpr int kMaxDstSmem = 4096;               // receivers table in smem when k*n_loc <= this
constexpr uint64_t kSpinLimitNs = 20ull * 1000 * 1000 * 1000;

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

size_t peer_smem_bytes(int k, int n_loc) {
  size_t b = kRingBytes + sizeof(int64_t) * (k + 1) + sizeof(int32_t) * (k + 1);
  if ((int64_t)k * n_loc <= kMaxDstSmem) b += sizeof(int32_t) * (size_t)k * n_loc;
  return align_up(b, 16);
}

// wait until (int32)(*p - target) >= 0; returns false on timeout
__device__ bool spin_until(const uint32_t* p, uint32_t target) {
  if ((int32_t)(ptx::ld_acquire_sys(p) - target) >= 0) return true;
  const uint64_t t0 = ptx::globaltimer();
  while (true) {
    if ((int32_t)(ptx::ld_acquire_sys(p) - target) >= 0) return true;
    if (ptx::globaltimer() - t0 > kSpinLimitNs) return false;
    __nanosleep(32);
  }
}

struct PeerKernelArgs {
  PeerStepArgs s;
  char* const* peers;       // [nprocs] region bases
  const int64_t* bounds;    // [k+1] segment bounds
  const int32_t* seg_t0;    // [k+1] first tile of each segment (seg_t0[k] = n_tiles)
  int n_tiles;
  uint32_t epoch;           // this step's epoch (>= 1)
  int mode;                 // 0 normal; diagnostics (wrong results): 1 local-only, 2 no waits
  size_t off_inbox, off_wbox, off_flags, off_done, off_count;
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
__device__ __forceinline__ void st4(float* p, float4 v, int valid) {
  if (valid == 4) {
    __stcs(reinterpret_cast<float4*>(p), v);
  } else {
    if (valid > 0) p[0] = v.x;
    if (valid > 1) p[1] = v.y;
    if (valid > 2) p[2] = v.z;
  }
}
__device__ __forceinline__ void st4_remote(float* p, float4 v, int valid) {
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
  const int32_t* dstl;  // [k][n_loc] global receiver of local worker r in segment s (or global table)
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

__device__ __forceinline__ uint32_t tile_bytes(const Unit& U) { return (uint32_t)(((U.len + 3) & ~3) * 4); }

__global__ void __launch_bounds__(kPeerThreads, 1) k_gossip_peer(const PeerKernelArgs a) {
  extern __shared__ __align__(128) float smem_f[];
  float* ringA = smem_f;                                   // [kStagesA][3][kPeerTile]
  float* ringY = ringA + (size_t)kStagesA * 3 * kPeerTile; // [kSlotsY][kPeerTile]
  float* ringB = ringY + (size_t)kSlotsY * kPeerTile;      // [kStagesB][kPeerTile]
  __shared__ uint64_t a_full[kStagesA], a_empty[kStagesA];
  __shared__ uint64_t b_full[kStagesB], b_empty[kStagesB];
  __shared__ uint64_t pushed[kSlotsY];
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

  // ---- metadata into shared memory --------------------------------------------------
  int64_t* bnd = reinterpret_cast<int64_t*>(ringB + (size_t)kStagesB * kPeerTile);
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
      ptx::mbar_init(&a_empty[i], kCompute / 32);
    }
    for (int i = 0; i < kStagesB; ++i) {
      ptx::mbar_init(&b_full[i], 1);
      ptx::mbar_init(&b_empty[i], kCompute / 32);
    }
    for (int i = 0; i < kSlotsY; ++i) ptx::mbar_init(&pushed[i], kCompute / 32);
    ptx::mbar_fence_init();
  }
  __syncthreads();
  // ping-pong safety: every receiver finished epoch e-2, the last reader of this parity
  if (threadIdx.x < s.nprocs && e >= 3) {
    const uint32_t* done = reinterpret_cast<const uint32_t*>(mine + a.off_done);
    if (!spin_until(done + threadIdx.x, e - 2)) atomicOr(&s_timeout, 1);
  }
  __syncthreads();

  if (warp < kCompute / 32) {
    // ---------------- compute warps ---------------------------------------------
    bool bad = false;
    const int tid = threadIdx.x;
    int cur_push = 0, cur_mix = 0;
    for (int i = 0; i < n_my + kLag && !*timeout; ++i) {
      if (i < n_my) {  // push unit i
        const Unit U = unit_at(a, M, blockIdx.x + i * G, cur_push);
        const int st = i % kStagesA;
        while (!ptx::mbar_try(&a_full[st], (uint32_t)((i / kStagesA) & 1)) && !*timeout) {
        }
        if (*timeout) break;
        const float* bx = ringA + (size_t)st * 3 * kPeerTile;
        float4* yslot = reinterpret_cast<float4*>(ringY + (size_t)(i % kSlotsY) * kPeerTile);
        int rp, rl;
        receiver_of(a, M, U.seg, U.r, rp, rl);
        float* inbox = reinterpret_cast<float*>(a.peers[rp] + a.off_inbox) + ((int64_t)par * s.n_loc + rl) * s.ld;
        const int64_t rowoff = (int64_t)U.r * s.ld;
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
          const int v = tid + q * kCompute;
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
            st4(s.m + rowoff + j, mn, vv);
            st4_remote(inbox + j, y, vv);
            yslot[v] = y;
          }
        }
        if (U.first_tile && tid == 0) {
          float* wbox = reinterpret_cast<float*>(a.peers[rp] + a.off_wbox) + ((int64_t)par * s.n_loc + rl) * s.k;
          wbox[U.seg] = s.psw[(int64_t)U.r * s.k + U.seg];
        }
        __syncwarp();
        if (lane == 0) {
          ptx::mbar_arrive(&a_empty[st]);
          ptx::mbar_arrive(&pushed[i % kSlotsY]);
        }
      }
      if (i >= kLag) {  // mix unit j
        const int j = i - kLag;
        const Unit U = unit_at(a, M, blockIdx.x + j * G, cur_mix);
        const int sb = j % kStagesB;
        while (!ptx::mbar_try(&b_full[sb], (uint32_t)((j / kStagesB) & 1)) && !*timeout) {
        }
        if (*timeout) break;
        const float4* yslot = reinterpret_cast<const float4*>(ringY + (size_t)(j % kSlotsY) * kPeerTile);
        const float4* yin = reinterpret_cast<const float4*>(ringB + (size_t)sb * kPeerTile);
        const int64_t rowoff = (int64_t)U.r * s.ld;
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
          const int v = tid + q * kCompute;
          const int valid = U.len - 4 * v;
          if (valid > 0) {
            const int64_t jj = U.c0 + 4 * (int64_t)v;
            st4(s.x + rowoff + jj, mean4(yslot[v], yin[v]), valid < 4 ? valid : 4);
          }
        }
        if (U.first_tile && tid == 0) {
          const float* wbox = reinterpret_cast<const float*>(mine + a.off_wbox) + ((int64_t)par * s.n_loc + U.r) * s.k;
          float* w = s.psw + (int64_t)U.r * s.k + U.seg;
          *w = __fmul_rn(__fadd_rn(*w, __ldcg(wbox + U.seg)), 0.5f);
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&b_empty[sb]);
      }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(s.err + kErrDiverged, 1);
  } else if (warp == kCompute / 32) {
    // ---------------- load warp: x, m, g tiles ahead -------------------------------
    if (lane == 0) {
      int cur = 0;
      for (int i = 0; i < n_my && !*timeout; ++i) {
        const Unit U = unit_at(a, M, blockIdx.x + i * G, cur);
        const int st = i % kStagesA;
        while (!ptx::mbar_try(&a_empty[st], (uint32_t)(((i / kStagesA) & 1) ^ 1)) && !*timeout) {
        }
        if (*timeout) break;
        const uint32_t bytes = tile_bytes(U);
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
    // ---------------- signal warp: flags out, flags in, inbox tiles ---------------
    if (lane == 0) {
      int nrel = 0, nacq = 0, cur_rel = 0, cur_acq = 0;
      uint64_t tstall = 0;
      while (nacq < n_my) {
        bool progress = false;
        // release every unit the compute warps have pushed: one system fence per batch
        int cnt = 0;
        while (nrel + cnt < n_my && cnt < kSlotsY &&
               ptx::mbar_test(&pushed[(nrel + cnt) % kSlotsY], (uint32_t)(((nrel + cnt) / kSlotsY) & 1)))
          ++cnt;
        if (cnt > 0) {
          ptx::fence_acq_rel_sys();
          for (int c = 0; c < cnt; ++c) {
            const Unit U = unit_at(a, M, blockIdx.x + (nrel + c) * G, cur_rel);
            int rp, rl;
            receiver_of(a, M, U.seg, U.r, rp, rl);
            uint32_t* flag =
                reinterpret_cast<uint32_t*>(a.peers[rp] + a.off_flags) + (int64_t)U.tile * s.n_loc + rl;
            ptx::st_relaxed_sys(flag, e);
          }
          nrel += cnt;
          progress = true;
        }
        // acquire inbound units whose flag is set and whose B slot is free: one fence per batch
        int got = 0;
        int cur_probe = cur_acq;
        while (nacq + got < nrel && got < kStagesB &&
               ptx::mbar_test(&b_empty[(nacq + got) % kStagesB], (uint32_t)((((nacq + got) / kStagesB) & 1) ^ 1))) {
          const Unit U = unit_at(a, M, blockIdx.x + (nacq + got) * G, cur_probe);
          const uint32_t* flag =
              reinterpret_cast<const uint32_t*>(mine + a.off_flags) + (int64_t)U.tile * s.n_loc + U.r;
          if (a.mode != 2 && (int32_t)(ptx::ld_relaxed_sys(flag) - e) < 0) break;
          ++got;
        }
        if (got > 0) {
          ptx::fence_acq_rel_sys();
          ptx::fence_proxy_async_global();
          for (int c = 0; c < got; ++c) {
            const Unit U = unit_at(a, M, blockIdx.x + (nacq + c) * G, cur_acq);
            const int sb = (nacq + c) % kStagesB;
            const uint32_t bytes = tile_bytes(U);
            const float* src = reinterpret_cast<const float*>(mine + a.off_inbox) +
                               ((int64_t)par * s.n_loc + U.r) * s.ld + U.c0;
            ptx::mbar_arrive_expect_tx(&b_full[sb], bytes);
            ptx::bulk_g2s(ringB + (size_t)sb * kPeerTile, src, bytes, &b_full[sb]);
          }
          nacq += got;
          progress = true;
        }
        if (progress) {
          tstall = 0;
        } else {
          const uint64_t now = ptx::globaltimer();
          if (tstall == 0) tstall = now;
          if (now - tstall > kSpinLimitNs) {  // give up: the other warps poll s_timeout
            *timeout = 1;
            break;
          }
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
  p.off_inbox = 0;
  p.off_wbox = align_up(p.off_inbox + sizeof(float) * 2 * (size_t)n_loc * ld, 256);
  p.off_flags = align_up(p.off_wbox + sizeof(float) * 2 * (size_t)n_loc * k, 256);
  p.off_done = align_up(p.off_flags + sizeof(uint32_t) * (size_t)p.n_tiles * n_loc, 256);
  p.off_count = align_up(p.off_done + sizeof(uint32_t) * (size_t)nprocs, 256);
  p.bytes = align_up(p.off_count + 256, 4096);
  cudaError_t e = cudaMalloc(&p.base, p.bytes);
  if (e != cudaSuccess) return perr(CS_ECUDA, "peer region cudaMalloc", e);
  e = cudaMemset(p.base, 0, p.bytes);  // inbox padding is read by 16-byte-rounded bulk copies
  if (e != cudaSuccess) return perr(CS_ECUDA, "peer region memset", e);
  e = cudaMalloc(&p.d_bounds, sizeof(int64_t) * (k + 1));
  if (e == cudaSuccess) e = cudaMalloc(&p.d_seg_t0, sizeof(int32_t) * (k + 1));
  if (e == cudaSuccess)
    e = cudaMemcpy(p.d_bounds, bounds.data(), sizeof(int64_t) * (k + 1), cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(p.d_seg_t0, seg_t0.data(), sizeof(int32_t) * (k + 1), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return perr(CS_ECUDA, "tile tables", e);
  const size_t smem = peer_smem_bytes(k, n_loc);
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaFuncSetAttribute(k_gossip_peer, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return perr(CS_ECUDA, "smem attribute", e);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gossip_peer, kPeerThreads, smem);
  if (e != cudaSuccess || occ < 1) return perr(CS_ECUDA, "occupancy", e);
  p.grid = sms * occ;
  const int n_units = p.n_tiles * n_loc;
  if (p.grid > n_units) p.grid = n_units;
  if (p.grid < n_loc) return perr(CS_EUNSUPPORTED, "more local workers than resident CTAs", cudaSuccess);
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
  ka.epoch = ++p.epoch;
  ka.mode = p.mode;
  ka.off_inbox = p.off_inbox;
  ka.off_wbox = p.off_wbox;
  ka.off_flags = p.off_flags;
  ka.off_done = p.off_done;
  ka.off_count = p.off_count;
  void* args[] = {&ka};
  if (ev0) cudaEventRecord(ev0, st);
  e = cudaLaunchCooperativeKernel((const void*)k_gossip_peer, dim3(p.grid), dim3(kPeerThreads), args,
                                  peer_smem_bytes(a.k, a.n_loc), st);
  if (e != cudaSuccess) return perr(CS_ECUDA, "cooperative launch", e);
  if (ev1) cudaEventRecord(ev1, st);
  return CS_OK;
}

}  // namespace cs
