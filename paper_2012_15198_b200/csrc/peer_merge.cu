// k_push_merge: one multi-GPU step (one worker per GPU) whose merge a5 completes inside
// the step's own kernel, so params and psw hold the merged x', w' when the step's enqueued
// work completes ("parameter averaging is processed after the gradient is applied",
// PAPER.md:122; Alg. 1 l.12-17: wait for the segments, then average).
//
// Work units are chunks of up to kMergeChunk segment-aligned tiles, numbered in segment
// order.  Every GPU runs a persistent grid whose CTAs claim chunks from a per-GPU counter
// (dynamic: with a static split, per-CTA timestamps showed SMs finishing between 90 and
// 160 us), so all GPUs sweep the vector front to back at the same pace and tile t of a
// receiver is pushed by its sender at about the time the receiver updates it.
// Warp roles of a CTA:
//
//   x/m/g warp        claims chunks, bulk-loads the x, m, g tiles (3-stage ring)
//   update warps (8)  a3: m' = mu*m + g, y = x - lr*m'; m' -> HBM; y -> params (through L2:
//                     the mix re-reads it soon) and into the push ring (bf16 on the bf16
//                     wire), with two 32-bit checksums of the pushed words
//   store warp        a4 (Alg.1 l.7 isend): one bulk copy per y tile into the inbox of the
//                     tile's receiver over NVLink; once the copy has completed
//                     (cp.async.bulk.wait_group) a 16-byte trailer for the tile
//                     {epoch, xor ^ w, weighted sum, w} (w = the push-sum weight on a
//                     segment's first tile) goes to the receiver
//   inbox warp        waits for the tile's trailer epoch (Alg.1 l.14 "wait until ...
//                     communication is completed", per tile), stages the received tile and
//                     the own y tile (Alg.1 l.8 irecv)
//   mix warps (4)     verify the received words against the trailer's checksums (re-read
//                     from memory until they match), then a5: x' = fl(fl(y + y_recv) * 0.5)
//                     -> params; a segment's first tile also merges psw (C-11)
//
// Why trailers and not release/acquire flags: a system-scope fence waits for the SM's
// in-flight NVLink copies, and under this load each one took ~13 us (measured: the
// signalling warp spent 130 of 160 us in fences), so a per-chunk release lagged the merge
// by tens of microseconds.  A trailer is written only after its tile's copy completed;
// the receiver accepts the tile only when its words reproduce both checksums of that
// exact trailer, so a tile is never mixed from partially arrived or stale data, whatever
// order the fabric delivers writes in (a stale tile would have to match two 32-bit
// checksums of new data).
//
// Nothing that produces a tile (claim, update, push) waits for another GPU's progress in the
// step: only the inbox warp and the mix do, and nothing waits for the mix.  So the merge
// may trail the update by any distance, and the step has no grid-wide or cross-GPU barrier.
// HBM per parameter: 12 B read (x, m, g) + 4 B m' + 4 B x' + 4 B inbox written by the
// sender + 4 B inbox read = 28 B, + 8 B for y (write, re-read) where L2 does not absorb it;
// NVLink 4 B out and 4 B in (+16 B per 8 KB tile of trailer).
//
// Ping-pong: inbox and trailers are indexed by the epoch parity.  Before writing parity
// e & 1 into a receiver, the store warp checks that every rank consumed epoch e - 2 (its
// done word, published with a release by its last CTA of that step; the same word the
// other multi-GPU kernels publish, so schedules can follow one another).  Deadlock freedom:
// producers never wait on the current epoch of another GPU, and every CTA is resident
// (persistent grid; in the single-GPU emulation, one cooperative launch).  Every cross-GPU
// wait is bounded; on timeout the kernel still drains its pipeline (results undefined) and
// reports CS_ETIMEOUT.
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "../../include/crossover_sgd.h"
#include "arith.cuh"
#include "common.cuh"
#include "peer.cuh"
#include "peer_dev.cuh"
#include "ptx.cuh"
#include "topo_device.cuh"

namespace cs {

namespace {

constexpr int kT = kPeerTile;                         // columns per tile
constexpr int kUpd = 256;                             // update warps' threads
constexpr int kMix = 128;                             // mix warps' threads
constexpr int kMThreads = kUpd + kMix + 96;           // + x/m/g loader, inbox loader, store warp
constexpr int kWarps = kMThreads / 32;
constexpr int kNA = 3, kNI = 3, kNY = 4;              // ring depths: x/m/g stages, inbox + own y, push
constexpr int kLand = 1;                              // copies in flight before the store warp checks completion
constexpr int kMaxK = 512;                            // segments (smem tables)
constexpr int kMaxClaims = 1024;                      // chunks one CTA may claim per step (smem list)
constexpr int kWLoadXmg = (kUpd + kMix) / 32, kWLoadIn = kWLoadXmg + 1, kWStore = kWLoadXmg + 2;
constexpr int kPerU = kT / 4 / kUpd;                  // float4 per update thread per tile
constexpr int kPerM = kT / 4 / kMix;                  // float4 per mix thread per tile
constexpr int kMixBar = 1;                            // named barrier of the mix warps

size_t smem_bytes(int k) {
  size_t b = sizeof(float) * (size_t)kT * (3 * kNA + 2 * kNI + kNY);
  b += sizeof(int64_t) * (k + 1) + sizeof(int32_t) * (k + 1) + sizeof(int32_t) * (size_t)k;
  b += sizeof(int32_t) * kMaxClaims;
  b = (b + 15) & ~size_t(15);
  b += sizeof(uint32_t) * 128 * kWarps;  // per-warp Alg. 2 scratch
  return b;
}

struct MergeArgs {
  PeerStepArgs s;
  char* const* peers;       // [nprocs] region bases
  const int64_t* bounds;    // [k+1]
  const int32_t* seg_t0;    // [k+1] first tile of each segment
  const TileDesc* tiles;    // explicit tiles (layer table) or nullptr
  const int32_t* chunk_t0;  // [n_chunks+1] first tile of each chunk (chunks never cross segments)
  int n_tiles, n_chunks;
  int trl_cap;              // trailer slots per parity
  int lag;                  // the inbox warp stages position j once the update is at j + lag
  int vranks;
  uint32_t epoch;
  int fused_topo;
  unsigned long long* trace;  // measurement only (CS_MERGE_TRACE): per-CTA timestamps [G][8]
  unsigned int* retries;      // tiles whose first read failed verification (diagnostic counter)
  uint32_t done_target;     // arrival total at which this step's last CTA publishes done = epoch
  size_t off_inbox, off_trl, off_done, off_count, off_claim, off_d2;
};

struct MTile {
  int64_t c0;
  int len, seg, layer;
  bool first;   // first tile of its segment (carries the push-sum weight)
};

__device__ __forceinline__ MTile mtile(const MergeArgs& a, const int64_t* bnd, const int32_t* t0, int t, int& cur) {
  MTile u;
  while (t0[cur + 1] <= t) ++cur;  // tiles of a CTA only increase: a cursor suffices
  u.seg = cur;
  u.first = t == t0[cur];
  if (a.tiles != nullptr) {
    const TileDesc td = a.tiles[t];
    u.c0 = td.c0;
    u.len = td.len;
    u.layer = td.layer;
  } else {
    u.c0 = bnd[cur] + (int64_t)(t - t0[cur]) * kT;
    const int64_t c1 = u.c0 + kT < bnd[cur + 1] ? u.c0 + kT : bnd[cur + 1];
    u.len = (int)(c1 - u.c0);
    u.layer = 0;
  }
  return u;
}

// A role's walk over the CTA's claimed chunks: position i -> tile.  claims[] is written by
// the x/m/g warp before the first tile of a chunk is released to the pipeline (every other
// role reaches that position after an acquire that follows the write).
struct Walk {
  int ci = -1, t = 0, t_end = 0, chunk = -1;
  __device__ __forceinline__ bool next(const int32_t* claims, const int32_t* chunk_t0) {
    if (t + 1 < t_end) {
      ++t;
      return true;
    }
    ++ci;
    chunk = claims[ci];
    if (chunk < 0) return false;
    t = __ldg(chunk_t0 + chunk);
    t_end = __ldg(chunk_t0 + chunk + 1);
    return true;
  }
};

__device__ __forceinline__ void st4(float* p, float4 v, int valid) {
  if (valid == 4) {
    *reinterpret_cast<float4*>(p) = v;
  } else {
    if (valid > 0) p[0] = v.x;
    if (valid > 1) p[1] = v.y;
    if (valid > 2) p[2] = v.z;
  }
}
__device__ __forceinline__ void st4_cs(float* p, float4 v, int valid) {
  if (valid == 4) {
    __stcs(reinterpret_cast<float4*>(p), v);
  } else {
    if (valid > 0) p[0] = v.x;
    if (valid > 1) p[1] = v.y;
    if (valid > 2) p[2] = v.z;
  }
}
__device__ __forceinline__ void red_add_release_cta(uint32_t* p, uint32_t v) {
  asm volatile("red.release.cta.shared::cta.add.u32 [%0], %1;" ::"r"(ptx::smem_addr(p)), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_cta(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(ptx::smem_addr(p)) : "memory");
  return v;
}
// memory reads that bypass L1 (another GPU writes these words)
__device__ __forceinline__ uint4 ld_volatile4(const void* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ uint2 ld_volatile2(const void* p) {
  uint2 v;
  asm volatile("ld.volatile.global.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_volatile1(const void* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile4(void* p, uint4 v) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// The two checksums of a tile's pushed words w_i (i = word index in the tile):
// xor of all w_i, and sum of w_i * (2i + 1) mod 2^32 (position-sensitive).
__device__ __forceinline__ void ck_add(uint32_t& cx, uint32_t& cs, uint32_t w, uint32_t i) {
  cx ^= w;
  cs += w * (2u * i + 1u);
}

__global__ void __launch_bounds__(kMThreads, 1) k_push_merge(const MergeArgs a) {
  extern __shared__ __align__(128) float smem_f[];
  float* ringA = smem_f;                                   // [kNA][3][kT]  x, m, g
  float* ringI = ringA + (size_t)kNA * 3 * kT;             // [kNI][2][kT]  received y (fp32/bf16), own y
  float* ringY = ringI + (size_t)kNI * 2 * kT;             // [kNY][kT]     y to push (fp32 or bf16)
  const PeerStepArgs& s0 = a.s;
  const bool wire = s0.wire != 0;
  int64_t* bnd = reinterpret_cast<int64_t*>(ringY + (size_t)kNY * kT);
  int32_t* t0 = reinterpret_cast<int32_t*>(bnd + s0.k + 1);
  int32_t* recv = t0 + s0.k + 1;                           // [k] rank receiving my segment s
  int32_t* claims = recv + s0.k;                           // [kMaxClaims] chunks claimed, -1 ends
  uint32_t* scratch = reinterpret_cast<uint32_t*>(
      (reinterpret_cast<uintptr_t>(claims + kMaxClaims) + 15) & ~uintptr_t(15));  // [kWarps][128]
  __shared__ uint64_t a_full[kNA], a_empty[kNA], i_full[kNI], i_empty[kNI], y_full[kNY], y_free[kNY];
  __shared__ uint32_t ck_upd[kNY][kUpd / 32][2];  // per update warp: checksums of its pushed words
  __shared__ uint32_t w_upd[kNY];                 // push-sum weight bits sent with the tile (0: none)
  __shared__ uint4 meta[kNI];                     // trailer of the staged received tile (bulk-loaded)
  __shared__ uint4 meta_re;                       // trailer re-read by the mix after a failed check
  __shared__ uint32_t ck_mix[2][kMix / 32][2];    // per mix warp, double-buffered by tile parity
  __shared__ uint32_t y_stored;  // update-warp arrivals: position j's y is in params at >= 8 (j + 1)
  __shared__ int s_end;          // number of positions (tiles) this CTA processes; INT_MAX until known
  __shared__ int s_timeout;
  volatile int* timeout = &s_timeout;
  volatile int* end_pos = &s_end;

  const unsigned long long t_entry = a.trace ? ptx::globaltimer() : 0;
  const RankCta rc = rank_cta(a.vranks, s0.rank);
  PeerStepArgs s = s0;
  rank_view(s, a.peers, a.vranks, rc.rank);
  const int b = rc.b, G = rc.G;
  const uint32_t e = a.epoch;
  const int par = (int)(e & 1u);
  char* mine = a.peers[s.rank];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ld_bf = (s.ld + 7) & ~int64_t(7);

  for (int i = threadIdx.x; i <= s.k; i += blockDim.x) {
    bnd[i] = a.bounds[i];
    t0[i] = a.seg_t0[i];
  }
  if (threadIdx.x == 0) {
    s_timeout = 0;
    s_end = 0x7fffffff;
    y_stored = 0;
    for (int i = 0; i < kNA; ++i) {
      ptx::mbar_init(&a_full[i], 1);
      ptx::mbar_init(&a_empty[i], kUpd / 32);
    }
    for (int i = 0; i < kNI; ++i) {
      ptx::mbar_init(&i_full[i], 1);
      ptx::mbar_init(&i_empty[i], kMix / 32);
    }
    for (int i = 0; i < kNY; ++i) {
      ptx::mbar_init(&y_full[i], kUpd / 32);
      ptx::mbar_init(&y_free[i], 1);  // the store warp's copy has read the slot
    }
    ptx::mbar_fence_init();
  }
  // this step's receivers: Alg. 2 per segment, one warp per segment,
  // then send_to = the rank that receives from me (Alg.1 l.6)
  {
    const int ntop = s.gs > 0 ? s.groups : s.world;
    const int grp = s.gs > 0 ? s.rank / s.gs : 0;
    const int target = s.gs > 0 ? grp : s.rank;
    uint32_t* u = scratch + warp * 128;
    int32_t* srow = reinterpret_cast<int32_t*>(u + 64);
    for (int sg = warp; sg < s.k; sg += kWarps) {
      if (!a.fused_topo) {
        if (lane == 0) recv[sg] = receiver_worker(s, sg, 0);
        continue;
      }
      const int32_t* row = srow;
      if (s.given != nullptr) row = s.given + (int64_t)sg * ntop;
      else warp_alg2_small(s.seed, s.step, sg, ntop, s.gs > 0 ? CS_TAG_HIER : CS_TAG_FLAT, u, srow, s.err);
      __syncwarp();
      for (int jj = lane; jj < ntop; jj += 32)
        if (row[jj] == target) recv[sg] = s.gs > 0 ? jj * s.gs + (s.rank - grp * s.gs) : jj;
      __syncwarp();
    }
  }
  __syncthreads();
  unsigned long long* tr = a.trace ? a.trace + ((size_t)s.rank * G + b) * 8 : nullptr;
  if (tr && threadIdx.x == 0) {
    tr[0] = ptx::globaltimer();
    tr[5] = t_entry;
  }
  uint4* trl_in = reinterpret_cast<uint4*>(mine + a.off_trl) + (size_t)par * a.trl_cap;

  if (warp < kUpd / 32) {
    // ---------------- update warps: a3 ------------------------------------------------
    const int tid = threadIdx.x;
    bool bad = false;
    int cur = 0;
    Walk w;
    for (int i = 0;; ++i) {
      const int st = i % kNA, sy = i % kNY;
      ptx::mbar_wait(&a_full[st], (uint32_t)((i / kNA) & 1));
      ptx::mbar_wait(&y_free[sy], (uint32_t)(((i / kNY) & 1) ^ 1));
      if (!w.next(claims, a.chunk_t0)) {  // end marker: pass it on to the store warp
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&y_full[sy]);
        break;
      }
      const MTile U = mtile(a, bnd, t0, w.t, cur);
      const float* bx = ringA + (size_t)st * 3 * kT;
      float4* yt = reinterpret_cast<float4*>(ringY + (size_t)sy * kT);
      const float rate = s.lrs ? __ldg(s.lrs + U.layer) : s.lr;
      const uint32_t nw = wire ? (uint32_t)(U.len + 1) / 2 : (uint32_t)U.len;  // pushed words checked
      uint32_t cx = 0, cs = 0;
#pragma unroll
      for (int q = 0; q < kPerU; ++q) {
        const int v = tid + q * kUpd;
        const int valid = U.len - 4 * v;
        if (valid > 0) {
          const int vv = valid < 4 ? valid : 4;
          const float4 cxv = reinterpret_cast<const float4*>(bx)[v];
          const float4 cm = reinterpret_cast<const float4*>(bx + kT)[v];
          const float4 cg = reinterpret_cast<const float4*>(bx + 2 * kT)[v];
          bad |= nonfinite4(cg);
          // LARS (C-18): m' = mu*m + (g + wd*x), y = x - lrs[layer]*m'
          const float4 mn = mom4(cm, s.lrs ? decay4(cg, cxv, s.wd) : cg, s.mu);
          const float4 y = sgd4(cxv, mn, rate);
          st4_cs(s.m + U.c0 + 4 * v, mn, vv);
          st4(s.x + U.c0 + 4 * v, y, vv);  // default policy: stays in L2 for the mix
          if (wire) {  // what the receiver gets (C-20)
            const uint2 pw = pack_bf16x4(y);
            reinterpret_cast<uint2*>(yt)[v] = pw;
            if (2u * v < nw) ck_add(cx, cs, pw.x, 2u * v);
            if (2u * v + 1 < nw) ck_add(cx, cs, pw.y, 2u * v + 1);
          } else {
            yt[v] = y;
            const uint32_t wv[4] = {__float_as_uint(y.x), __float_as_uint(y.y), __float_as_uint(y.z),
                                    __float_as_uint(y.w)};
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (c < vv) ck_add(cx, cs, wv[c], 4u * v + c);
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        cx ^= __shfl_xor_sync(0xffffffffu, cx, o);
        cs += __shfl_xor_sync(0xffffffffu, cs, o);
      }
      if (lane == 0) {
        ck_upd[sy][warp][0] = cx;
        ck_upd[sy][warp][1] = cs;
      }
      // the push-sum weight travels with the segment's first tile
      if (tid == 0) w_upd[sy] = U.first ? __float_as_uint(s.psw[U.seg]) : 0u;
      ptx::fence_proxy_async_shared();  // push tile -> the store warp's bulk copy
      ptx::fence_proxy_async_global();  // y in params -> the inbox warp's bulk copy
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive(&a_empty[st]);
        ptx::mbar_arrive(&y_full[sy]);
        red_add_release_cta(&y_stored, 1u);
      }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(s.err + kErrDiverged, 1);
    if (tr && threadIdx.x == 0) tr[1] = ptx::globaltimer();
  } else if (warp < (kUpd + kMix) / 32) {
    // ---------------- mix warps: verify, then a5 ------------------------------------
    const int tm = threadIdx.x - kUpd, mw = tm >> 5;
    const float* inbox_f = reinterpret_cast<const float*>(mine + a.off_inbox) + par * s.ld;
    const uint16_t* inbox_w = reinterpret_cast<const uint16_t*>(mine + a.off_inbox) + par * ld_bf;
    int cur = 0, retried = 0, round = 0;  // round: checksum reductions so far (buffer parity)
    Walk w;
    for (int j = 0;; ++j) {
      const int si = j % kNI;
      ptx::mbar_wait(&i_full[si], (uint32_t)((j / kNI) & 1));
      if (!w.next(claims, a.chunk_t0)) break;
      const MTile U = mtile(a, bnd, t0, w.t, cur);
      const float* it = ringI + (size_t)si * 2 * kT;
      const float4* yt = reinterpret_cast<const float4*>(it + kT);
      const uint32_t nw = wire ? (uint32_t)(U.len + 1) / 2 : (uint32_t)U.len;
      uint4 tl = meta[si];
      uint4 raw[kPerM];  // the received words as pushed (fp32 bits, or 2 x 2 bf16 in .x .y)
#pragma unroll
      for (int q = 0; q < kPerM; ++q) {
        const int v = tm + q * kMix;
        if (wire) {
          const uint2 pw = reinterpret_cast<const uint2*>(it)[v];
          raw[q] = make_uint4(pw.x, pw.y, 0u, 0u);
        } else {
          raw[q] = reinterpret_cast<const uint4*>(it)[v];
        }
      }
      for (int attempt = 0;; ++attempt) {
        uint32_t cx = 0, cs = 0;
#pragma unroll
        for (int q = 0; q < kPerM; ++q) {
          const int v = tm + q * kMix;
          if (4 * v < U.len) {
            if (wire) {
              if (2u * v < nw) ck_add(cx, cs, raw[q].x, 2u * v);
              if (2u * v + 1 < nw) ck_add(cx, cs, raw[q].y, 2u * v + 1);
            } else {
              const uint32_t wv[4] = {raw[q].x, raw[q].y, raw[q].z, raw[q].w};
#pragma unroll
              for (int c = 0; c < 4; ++c)
                if (4 * v + c < U.len) ck_add(cx, cs, wv[c], 4u * v + c);
            }
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          cx ^= __shfl_xor_sync(0xffffffffu, cx, o);
          cs += __shfl_xor_sync(0xffffffffu, cs, o);
        }
        const int pb = round++ & 1;
        if (lane == 0) {
          ck_mix[pb][mw][0] = cx;
          ck_mix[pb][mw][1] = cs;
        }
        ptx::named_bar_sync(kMixBar, kMix);
        uint32_t X = 0, S = 0;
#pragma unroll
        for (int m2 = 0; m2 < kMix / 32; ++m2) {
          X ^= ck_mix[pb][m2][0];
          S += ck_mix[pb][m2][1];
        }
        if (((X ^ tl.w) == tl.y && S == tl.z && tl.x == e) || *timeout) break;
        // not (yet) the tile the trailer describes: wait for this epoch's trailer, then read
        // trailer and words again from memory
        if (tm == 0) {
          if (tl.x == e) ++retried;  // the trailer had arrived but the words had not
          const uint32_t* ep = reinterpret_cast<const uint32_t*>(trl_in + w.t);
          const uint64_t tin = tr ? ptx::globaltimer() : 0;
          uint64_t tw = 0;
          while ((int32_t)(ld_volatile1(ep) - e) < 0) {
            const uint64_t now = ptx::globaltimer();
            if (tw == 0) tw = now;
            if (now - tw > ptx::kSpinLimitNs) {
              *timeout = 1;
              break;
            }
            __nanosleep(64);
          }
          if (tr) tr[4] += ptx::globaltimer() - tin;
          if (attempt > 0) __nanosleep(256);
          meta_re = ld_volatile4(trl_in + w.t);
        }
        ptx::named_bar_sync(kMixBar, kMix);
        tl = meta_re;
#pragma unroll
        for (int q = 0; q < kPerM; ++q) {
          const int v = tm + q * kMix;
          if (4 * v < U.len) {
            if (wire) {
              const uint2 pw = ld_volatile2(inbox_w + U.c0 + 4 * v);
              raw[q] = make_uint4(pw.x, pw.y, 0u, 0u);
            } else {
              raw[q] = ld_volatile4(inbox_f + U.c0 + 4 * v);
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < kPerM; ++q) {
        const int v = tm + q * kMix;
        const int valid = U.len - 4 * v;
        if (valid > 0) {
          const float4 yr = wire ? unpack_bf16x4(make_uint2(raw[q].x, raw[q].y))
                                 : make_float4(__uint_as_float(raw[q].x), __uint_as_float(raw[q].y),
                                               __uint_as_float(raw[q].z), __uint_as_float(raw[q].w));
          st4_cs(s.x + U.c0 + 4 * v, mean4(yt[v], yr), valid < 4 ? valid : 4);  // Alg.1 l.17
        }
      }
      if (U.first && tm == 0) s.psw[U.seg] = pair_mean1(s.psw[U.seg], __uint_as_float(tl.w));
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&i_empty[si]);
    }
    if (tm == 0 && retried && a.retries) atomicAdd(a.retries, (unsigned)retried);
    if (tr && tm == 0) tr[6] = ptx::globaltimer();
  } else if (warp == kWLoadXmg) {
    // ---------------- claims + x, m, g loader ----------------------------------------
    if (s.gs > 0 && lane < s.gs) {  // hierarchical: the group mean is complete on this GPU
      const uint32_t* d2 = reinterpret_cast<const uint32_t*>(mine + a.off_d2);
      const int gbase = (s.rank / s.gs) * s.gs;
      if (!ptx::wait_geq_sys(d2 + gbase + lane, e)) atomicOr(&s_timeout, 1);
    }
    __syncwarp();
    if (lane == 0) {
      ptx::fence_proxy_async_global();
      // claim counters by epoch parity: this step's starts at 0 (reset by the previous step)
      uint32_t* counter = reinterpret_cast<uint32_t*>(mine + a.off_claim) + par;
      int cur = 0, n_claims = 0, t = 0, t_end = 0;
      for (int i = 0;; ++i) {
        const int st = i % kNA;
        ptx::mbar_wait(&a_empty[st], (uint32_t)(((i / kNA) & 1) ^ 1));
        if (t == t_end) {  // claim the next chunk (segment order: the pace every GPU keeps)
          const int c = n_claims < kMaxClaims - 1 ? (int)atomicAdd(counter, 1u) : a.n_chunks;
          if (c >= a.n_chunks) {  // nothing left (or this CTA's list is full): end marker
            claims[n_claims] = -1;
            *end_pos = i;
            ptx::mbar_arrive(&a_full[st]);
            break;
          }
          claims[n_claims++] = c;
          t = __ldg(a.chunk_t0 + c);
          t_end = __ldg(a.chunk_t0 + c + 1);
        }
        const MTile U = mtile(a, bnd, t0, t, cur);
        ++t;
        const uint32_t bytes = (uint32_t)(((U.len + 3) & ~3) * 4);
        float* buf = ringA + (size_t)st * 3 * kT;
        ptx::mbar_arrive_expect_tx(&a_full[st], 3 * bytes);
        ptx::bulk_g2s(buf, s.x + U.c0, bytes, &a_full[st]);
        ptx::bulk_g2s(buf + kT, s.m + U.c0, bytes, &a_full[st]);
        ptx::bulk_g2s(buf + 2 * kT, s.g + U.c0, bytes, &a_full[st]);
      }
    }
    __syncwarp();
  } else if (warp == kWLoadIn) {
    // ---------------- inbox loader: wait for the tile's trailer, stage the tiles -------
    if (lane == 0) {
      int cur = 0;
      Walk w;
      for (int j = 0;; ++j) {
        const int si = j % kNI;
        // this CTA's own y of position j + lag is in params (the sender's copy of j has
        // probably completed by then), or the walk ends before it
        bool more = true;
        while ((int32_t)(ld_acquire_cta(&y_stored) - (uint32_t)(kUpd / 32) * (uint32_t)(j + 1 + a.lag)) < 0) {
          const int ep = *end_pos;
          if (ep <= j + a.lag) {
            more = ep > j;
            if (more)  // the end is near: wait only for position j itself
              while ((int32_t)(ld_acquire_cta(&y_stored) - (uint32_t)(kUpd / 32) * (uint32_t)(j + 1)) < 0) {
              }
            break;
          }
        }
        ptx::mbar_wait(&i_empty[si], (uint32_t)(((j / kNI) & 1) ^ 1));
        if (!more) {  // end marker for the mix warps
          ptx::mbar_arrive(&i_full[si]);
          break;
        }
        w.next(claims, a.chunk_t0);
        const MTile U = mtile(a, bnd, t0, w.t, cur);
        // no wait here: the trailer is staged with the tiles and checked by the mix, which
        // polls only when it finds the trailer of an older epoch
        ptx::fence_proxy_async_global();  // own y written by the update warps -> this bulk copy
        float* buf = ringI + (size_t)si * 2 * kT;
        const uint32_t yb = (uint32_t)(((U.len + 3) & ~3) * 4);
        const uint32_t ib = wire ? (uint32_t)(((U.len + 7) & ~7) * 2) : yb;
        ptx::mbar_arrive_expect_tx(&i_full[si], ib + yb + 16u);
        ptx::bulk_g2s(&meta[si], trl_in + w.t, 16u, &i_full[si]);
        if (wire)
          ptx::bulk_g2s(buf, reinterpret_cast<const uint16_t*>(mine + a.off_inbox) + par * ld_bf + U.c0, ib,
                        &i_full[si]);
        else
          ptx::bulk_g2s(buf, reinterpret_cast<const float*>(mine + a.off_inbox) + par * s.ld + U.c0, yb,
                        &i_full[si]);
        ptx::bulk_g2s(buf + kT, s.x + U.c0, yb, &i_full[si]);
      }
    }
    __syncwarp();
  } else if (warp == kWStore) {
    // ---------------- store warp: push y tiles, then each completed tile's trailer ------
    // every rank consumed epoch e-2 (the last reader of the inbox parity written now):
    // relaxed polls by the lanes, one acquire fence
    if (e >= 3) {
      const uint32_t* dn = reinterpret_cast<const uint32_t*>(mine + a.off_done);
      bool ok = true;
      for (int q = lane; q < s.nprocs; q += 32) {
        uint64_t tw = 0;
        while ((int32_t)(ptx::ld_relaxed_sys(dn + q) - (e - 2)) < 0) {
          const uint64_t now = ptx::globaltimer();
          if (tw == 0) tw = now;
          if (now - tw > ptx::kSpinLimitNs) {
            ok = false;
            break;
          }
          __nanosleep(64);
        }
      }
      if (!__all_sync(0xffffffffu, ok) && lane == 0) *timeout = 1;
      if (lane == 0) ptx::fence_acq_rel_sys();
    }
    if (lane == 0) {
      uint4* pend_dst[kLand + 1] = {};
      uint4 pend_trl[kLand + 1] = {};
      int cur = 0, n = 0;
      Walk w;
      auto completed = [&](int j) {  // copy j has completed: its trailer may go (Alg.1 l.14)
        const int q = j % (kLand + 1);
        st_volatile4(pend_dst[q], pend_trl[q]);
      };
      for (int i = 0;; ++i) {
        const int sy = i % kNY;
        ptx::mbar_wait(&y_full[sy], (uint32_t)((i / kNY) & 1));
        if (!w.next(claims, a.chunk_t0)) break;
        const MTile U = mtile(a, bnd, t0, w.t, cur);
        const int rp = recv[U.seg];
        if (wire)
          ptx::bulk_s2g(reinterpret_cast<uint16_t*>(a.peers[rp] + a.off_inbox) + par * ld_bf + U.c0,
                        ringY + (size_t)sy * kT, (uint32_t)(((U.len + 7) & ~7) * 2));
        else
          ptx::bulk_s2g(reinterpret_cast<float*>(a.peers[rp] + a.off_inbox) + par * s.ld + U.c0,
                        ringY + (size_t)sy * kT, (uint32_t)(((U.len + 3) & ~3) * 4));
        ptx::bulk_commit();
        uint32_t X = 0, S = 0;
#pragma unroll
        for (int u = 0; u < kUpd / 32; ++u) {
          X ^= ck_upd[sy][u][0];
          S += ck_upd[sy][u][1];
        }
        const uint32_t wb = w_upd[sy];
        const int q = i % (kLand + 1);
        pend_dst[q] = reinterpret_cast<uint4*>(a.peers[rp] + a.off_trl) + (size_t)par * a.trl_cap + w.t;
        pend_trl[q] = make_uint4(e, X ^ wb, S, wb);
        ptx::bulk_wait_read<1>();
        if (i >= 1) ptx::mbar_arrive(&y_free[(i - 1) % kNY]);
        if (i >= kLand) {  // copies <= i - kLand have completed
          ptx::bulk_wait<kLand>();
          ptx::fence_proxy_async_global();  // their async-proxy writes -> the trailer store
          completed(i - kLand);
        }
        n = i + 1;
      }
      ptx::bulk_wait_all();
      ptx::fence_proxy_async_global();
      if (tr) tr[2] = ptx::globaltimer();
      if (n >= 1) ptx::mbar_arrive(&y_free[(n - 1) % kNY]);
      for (int j = n - kLand > 0 ? n - kLand : 0; j < n; ++j) completed(j);
      if (tr) tr[3] = ptx::globaltimer();
    }
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // this CTA consumed its tiles of epoch e; the last CTA releases parity e & 1 to every
    // sender: done[rank] = e on every GPU.  The arrival is an acq_rel atomic, so the last
    // CTA's system-scope release is cumulative over every CTA's reads and writes.
    if (s_timeout) atomicOr(s.err + kErrTimeout, 1);
    if (tr) tr[7] = ptx::globaltimer();
    const uint32_t prev = ptx::atom_add_acq_rel_gpu(reinterpret_cast<uint32_t*>(mine + a.off_count), 1u);
    if (prev + 1 == a.done_target) {
      // every CTA of this rank is past its claims: the next step's counter starts at 0
      reinterpret_cast<uint32_t*>(mine + a.off_claim)[par ^ 1] = 0u;
      for (int q = 0; q < s.nprocs; ++q)
        ptx::st_release_sys(reinterpret_cast<uint32_t*>(a.peers[q] + a.off_done) + s.rank, e);
      if (a.trace) a.trace[(size_t)a.vranks * G * 8 + s.rank] = ptx::globaltimer();
    }
  }
}

}  // namespace

size_t peer_merge_smem(int k, bool wire) {
  (void)wire;
  return smem_bytes(k);
}

int peer_merge_capacity(int k) {
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = smem_bytes(k < kMaxK ? k : kMaxK);
  if (cudaFuncSetAttribute(k_push_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_push_merge, kMThreads, smem) != cudaSuccess) return 0;
  return sms * occ;
}

// Chunks never crossing a segment, in tile order: chunk_t0 [n_chunks + 1].  Guided sizes:
// `chunk` tiles while plenty remain, shrinking to 1 tile over the last ~4 tiles per CTA of
// the grid, so the CTAs (whose SMs differ in speed) finish together.
std::vector<int32_t> peer_merge_chunks(const std::vector<int32_t>& seg_t0, int chunk, int grid) {
  if (getenv("CS_MERGE_CHUNK")) chunk = atoi(getenv("CS_MERGE_CHUNK")) > 0 ? atoi(getenv("CS_MERGE_CHUNK")) : chunk;
  std::vector<int32_t> c;
  const int k = (int)seg_t0.size() - 1;
  const int total = seg_t0[k];
  const int g4 = 4 * (grid > 0 ? grid : 1);
  for (int s = 0; s < k; ++s)
    for (int t = seg_t0[s]; t < seg_t0[s + 1];) {
      c.push_back(t);
      int len = (total - t) / g4;
      len = len < 1 ? 1 : (len > chunk ? chunk : len);
      t = t + len < seg_t0[s + 1] ? t + len : seg_t0[s + 1];
    }
  c.push_back(seg_t0[k]);
  return c;
}

bool peer_merge_ok(const PeerState& p, const PeerStepArgs& a) {
  return p.sched == kSchedInStep && a.n_loc == 1 && a.k <= kMaxK && p.grid_merge > 0 && p.d_chunk_t0 != nullptr &&
         // every CTA's claims fit its list even if one CTA took 4x its share
         (int64_t)p.n_chunks < (int64_t)(kMaxClaims - 1) * p.grid_merge / 4;
}

cudaError_t peer_launch(const PeerState& p, const void* fn, int grid_per_rank, int threads, size_t smem,
                        cudaStream_t st, void** args) {
  if (p.vranks <= 1) return cudaLaunchKernel(fn, dim3(grid_per_rank), dim3(threads), args, smem, st);
  return cudaLaunchCooperativeKernel(fn, dim3(grid_per_rank * p.vranks), dim3(threads), args, smem, st);
}

int peer_merge_launch(PeerState& p, const PeerStepArgs& a, uint32_t epoch, cudaStream_t st) {
  MergeArgs ma;
  ma.s = a;
  ma.peers = p.d_peer_base;
  ma.bounds = p.d_bounds;
  ma.seg_t0 = p.d_seg_t0;
  ma.tiles = p.d_ptiles;
  ma.chunk_t0 = p.d_chunk_t0;
  ma.n_tiles = p.n_tiles;
  ma.n_chunks = p.n_chunks;
  ma.vranks = p.vranks;
  ma.epoch = epoch;
  const int ntop = a.gs > 0 ? a.groups : a.world;
  ma.fused_topo = ntop <= 64 ? 1 : 0;
  ma.off_inbox = p.off_inbox;
  ma.off_trl = p.off_mflag;
  ma.trl_cap = p.mflag_cap;
  static const int lag = getenv("CS_MERGE_LAG") ? atoi(getenv("CS_MERGE_LAG")) : 2;
  ma.lag = lag < 0 ? 0 : lag;
  ma.retries = p.d_stats;
  ma.off_done = p.off_done;
  ma.off_count = p.off_count;
  ma.off_claim = p.off_claim;
  ma.off_d2 = p.off_d2;
  ma.done_target = (p.tot_count[0] += (uint32_t)p.grid_merge);
  // CS_MERGE_TRACE=E: per-CTA timestamps of epoch E, summarised on stderr
  static const long trace_epoch = getenv("CS_MERGE_TRACE") ? atol(getenv("CS_MERGE_TRACE")) : -1;
  static unsigned long long* d_trace = nullptr;
  ma.trace = nullptr;
  if (trace_epoch >= 0 && (long)epoch == trace_epoch) {
    const size_t n = (size_t)p.grid_merge * p.vranks * 8 + 64;
    if (!d_trace) cudaMalloc(&d_trace, n * sizeof(unsigned long long));
    cudaMemsetAsync(d_trace, 0, n * sizeof(unsigned long long), st);
    ma.trace = d_trace;
  }
  void* args[] = {&ma};
  cudaError_t e = peer_launch(p, (const void*)k_push_merge, p.grid_merge, kMThreads, smem_bytes(a.k), st, args);
  if (e != cudaSuccess) {
    fprintf(stderr, "k_push_merge launch: %s\n", cudaGetErrorString(e));
    return CS_ECUDA;
  }
  if (ma.trace) {
    const int n = p.grid_merge * p.vranks;
    std::vector<unsigned long long> h((size_t)n * 8 + 64);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), ma.trace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < n; ++c) t0 = h[c * 8] && h[c * 8] < t0 ? h[c * 8] : t0;
    const char* names[8] = {"start", "update_end", "push_landed", "trailers_end", "trailer_wait_us", "entry",
                            "mix_end", "cta_end"};
    unsigned int retr = 0;
    if (p.d_stats) cudaMemcpy(&retr, p.d_stats, sizeof(retr), cudaMemcpyDeviceToHost);
    fprintf(stderr, "[k_push_merge trace] tiles re-read after a failed verification so far: %u\n", retr);
    fprintf(stderr, "[k_push_merge trace] rank %d epoch %u, %d CTAs (us from the first start)\n", a.rank, epoch, n);
    for (int c = 0; c < n; ++c) t0 = h[c * 8 + 5] && h[c * 8 + 5] < t0 ? h[c * 8 + 5] : t0;
    fprintf(stderr, "  r%d done_published %8.2f (us from the first CTA entry)\n", a.rank,
            (h[(size_t)n * 8 + (p.vranks > 1 ? 0 : a.rank)] - t0) * 1e-3);
    for (int f = 0; f < 8; ++f) {
      std::vector<double> v;
      for (int c = 0; c < n; ++c) {
        const unsigned long long x = h[c * 8 + f];
        if (f == 4 || f == 5) v.push_back(x * 1e-3);
        else if (x) v.push_back((x - t0) * 1e-3);
      }
      if (v.empty()) continue;
      std::sort(v.begin(), v.end());
      fprintf(stderr, "  r%d %-13s min %8.2f  median %8.2f  max %8.2f\n", a.rank, names[f], v.front(),
              v[v.size() / 2], v.back());
    }
  }
  return CS_OK;
}

}  // namespace cs
