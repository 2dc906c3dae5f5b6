// k_push_merge: one multi-GPU flat step (or the leader exchange of a hierarchical step)
// whose merge a5 completes inside the step's own kernel, so params and psw hold the merged
// x', w' when the step's enqueued work completes ("parameter averaging is processed after
// the gradient is applied"; Alg. 1 l.12-17: wait for the
// segments, then average).  Any number n_loc of workers per GPU.
//
// Work: for every segment-aligned tile (2048 columns) the CTA walks the n_loc local rows in
// the order of that segment's permutation restricted to this GPU (built in the prologue
// from Alg. 2): local cycles c0 <- c1 <- ... (x'_{c_p} = mean(y_{c_p},
// y_{c_{p+1}}), all in registers), and chains whose head's receiver and whose tail's
// source are on other GPUs.  Per row that is one update (a3); a chain head's y goes to its
// receiver's inbox over NVLink (a4), a chain tail merges with the y it receives (a5).
// With one worker per GPU every row is a one-element chain (push and merge).
//
// Tiles are claimed in chunks from a per-GPU counter (dynamic: with a static split,
// per-CTA timestamps showed SMs finishing between 90 and 160 us), in segment order, so
// all GPUs sweep the vector front to back at the same pace.  Warp roles of a CTA:
//
//   x/m/g warp        claims chunks, bulk-loads the x, m, g row-tiles in walk order
//   update warps (8)  a3 + the walk: m' -> HBM; x' of local pairs -> HBM; a chain tail's y
//                     -> params (plain stores: L1/L2); a head's y into the push ring (bf16 on
//                     the bf16 wire) with two 32-bit checksums of its words
//   store warp        a head's tile: one bulk copy into its receiver's inbox row; once the
//                     copy has completed (cp.async.bulk.wait_group) a 16-byte trailer
//                     {epoch, xor ^ w, weighted sum, w} (w: the push-sum weight on a
//                     segment's first tile) goes to the receiver
//   inbox warp        for a chain tail: stages the tile's trailer, the received tile and the
//                     own y tile (Alg.1 l.8 irecv), once every update warp released the position
//   mix warps (4)     take the tails in the order the inbox warp staged them (each slot carries
//                     the tail's row and tile; an end marker closes the step), and
//                     verify the received words against the trailer's checksums (polling
//                     the trailer and re-reading the words until they match: Alg.1 l.14
//                     "wait until ... communication is completed", per tile), then
//                     a5: x' = fl(fl(y + y_recv) * 0.5) -> params and the tail's psw
//
// Why trailers and not release/acquire flags: a system-scope fence waits for the SM's
// in-flight NVLink copies, and under this load each one took ~13 us (measured: the
// signalling warp spent 130 of 160 us in fences), so a per-chunk release lagged the merge
// by tens of microseconds.  A trailer is written only after its tile's copy completed; the
// receiver accepts the tile only when its words reproduce both checksums of that exact
// trailer, so a tile is never mixed from partially arrived or stale data, whatever order
// the fabric delivers writes in (a stale tile would have to match two 32-bit checksums of
// new data).  Measured: ~1.7 % of tiles are first read before their words are visible.
//
// Nothing that produces a tile (claim, update, push) waits for another GPU's progress in the
// step: only the inbox warp and the mix do, and nothing waits for the mix.  So the merge may
// trail the update by any distance, and the step has no grid-wide or cross-GPU barrier.
// HBM per parameter: 20 B (read x, m, g; write m', x') + for a tail 4 B inbox written by
// the sender + 4 B inbox read (+ 8 B y write and re-read where L2 does not absorb it);
// NVLink 4 B out per head parameter (+16 B per 8 KB tile of trailer).
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
constexpr int kNA = 4, kNI = 3, kNY = 5;              // ring depths: x/m/g stages, inbox + own y, y out
constexpr int kReadLag = kNY - 1;                     // y-out slots whose copies may still be reading
constexpr int kQ = 8;                                 // store warp: positions with copies in flight (max)
constexpr int kMaxK = 512;                            // segments (smem tables)
constexpr int kMaxLoc = 64;                           // workers per GPU (64-bit walk masks)
constexpr int kMaxKN = 1024;                          // k * n_loc (smem walk tables)
constexpr int kMaxClaims = 1024;                      // chunks one CTA may claim per step (smem list)
constexpr int kWLoadXmg = (kUpd + kMix) / 32, kWLoadIn = kWLoadXmg + 1, kWStore = kWLoadXmg + 2;
constexpr int kPerU = kT / 4 / kUpd;                  // float4 per update thread per tile
constexpr int kPerM = kT / 4 / kMix;                  // float4 per mix thread per tile
constexpr int kMixBar = 1;                            // named barrier of the mix warps
// walk-order entries: local row | flags
constexpr uint32_t kWStart = 1u << 31, kWEnd = 1u << 30, kWHead = 1u << 29, kWTail = 1u << 28;
constexpr uint32_t kWIdx = (1u << 28) - 1;

size_t smem_bytes(int k, int n_loc, bool wire) {
  size_t b = sizeof(float) * (size_t)kT * (3 * kNA + 2 * kNI + kNY) + (wire ? sizeof(uint16_t) * (size_t)kT * kNY : 0);
  b += sizeof(int64_t) * (k + 1) + sizeof(int32_t) * (k + 1);
  b += 2 * sizeof(uint32_t) * (size_t)k * n_loc;  // walk order, head receivers
  b += sizeof(int32_t) * kMaxClaims;
  b += sizeof(float) * kMaxLoc;                    // psw snapshot of a segment's first tile
  return (b + 15) & ~size_t(15);                   // (the prologue's Alg. 2 scratch aliases the inbox ring)
}
static_assert(sizeof(float) * kT * (3 * kNA + 2 * kNI + kNY) + sizeof(uint16_t) * kT * kNY +
                      (sizeof(int64_t) + sizeof(int32_t)) * (kMaxK + 1) + 2 * sizeof(uint32_t) * kMaxKN +
                      sizeof(int32_t) * kMaxClaims + sizeof(float) * kMaxLoc + 16 + 2048 <=
                  227 * 1024,
              "k_push_merge shared memory exceeds 227 KB");
static_assert(sizeof(uint32_t) * 192 * kWarps <= sizeof(float) * kT * 2 * kNI, "Alg. 2 scratch fits the inbox ring");

struct MergeArgs {
  PeerStepArgs s;
  char* const* peers;       // [nprocs] region bases
  const int64_t* bounds;    // [k+1]
  const int32_t* seg_t0;    // [k+1] first tile of each segment
  const TileDesc* tiles;    // explicit tiles (layer table) or nullptr
  const int32_t* chunk_t0;  // [n_chunks+1] first tile of each chunk (chunks never cross segments)
  int n_tiles, n_chunks;
  int trl_cap;              // trailer slots per parity (tiles x n_loc)
  int lag;                  // the inbox warp stages position j once the update is at j + lag
  int read_lag;             // y-out slots left unfreed while their copies may still read them (0..kNY-1)
  int land;                 // > 0: positions whose copies stay in flight before the store warp awaits them (<= 7)
  int vranks;
  uint32_t epoch;
  int fused_topo;           // draw Alg. 2 in the prologue (<= 64 ranks), else read s.src
  unsigned long long* trace;  // measurement only (CS_MERGE_TRACE): per-CTA timestamps [G][8]
  unsigned int* retries;      // tiles whose first read failed verification (diagnostic counter)
  uint32_t done_target;     // arrival total at which this step's last CTA publishes done = epoch
  size_t off_inbox, off_trl, off_done, off_count, off_claim, off_d2;
};

struct MixMeta {   // what the mix needs of a staged tail (written before the slot's i_full arrive)
  int64_t c0;
  int len, seg, first, row, t;
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

// A role's walk over the CTA's positions: claimed chunks -> tiles -> the n_loc rows of a
// tile in walk order (p).  claims[] is written by the x/m/g warp before the first tile of a
// chunk is released to the pipeline (every other role reaches that position after an
// acquire that follows the write).
struct Walk {
  int ci = -1, t = 0, t_end = 0, chunk = -1, p = 0;
  __device__ __forceinline__ void init(int n_loc) { p = n_loc - 1; }
  __device__ __forceinline__ bool next(const int32_t* claims, const int32_t* chunk_t0, int n_loc) {
    if (++p < n_loc) return true;
    p = 0;
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

// wait until at most n (runtime, 0..4) bulk groups of this thread still read their source
__device__ __forceinline__ void bulk_wait_read_n(int n) {
  switch (n) {
    case 0: ptx::bulk_wait_read<0>(); break;
    case 1: ptx::bulk_wait_read<1>(); break;
    case 2: ptx::bulk_wait_read<2>(); break;
    case 3: ptx::bulk_wait_read<3>(); break;
    default: ptx::bulk_wait_read<4>(); break;
  }
}

// wait until at most n (runtime, 0..7) bulk groups of this thread are still writing
__device__ __forceinline__ void bulk_wait_n(int n) {
  switch (n) {
    case 0: ptx::bulk_wait<0>(); break;
    case 1: ptx::bulk_wait<1>(); break;
    case 2: ptx::bulk_wait<2>(); break;
    case 3: ptx::bulk_wait<3>(); break;
    case 4: ptx::bulk_wait<4>(); break;
    case 5: ptx::bulk_wait<5>(); break;
    case 6: ptx::bulk_wait<6>(); break;
    default: ptx::bulk_wait<7>(); break;
  }
}

// The two checksums of a tile's pushed words w_i (i = word index in the tile):
// xor of all w_i, and sum of w_i * (2i + 1) mod 2^32 (position-sensitive).
__device__ __forceinline__ void ck_add(uint32_t& cx, uint32_t& cs, uint32_t w, uint32_t i) {
  cx ^= w;
  cs += w * (2u * i + 1u);
}

// Wait until the update warps finished position j (true), or the walk ends before it (false).
// Position j is done when EVERY update warp has released it: each warp counts its own
// positions (a shared total would let warps that run ahead -- up to kNA stages -- stand in for
// one still storing its part of position j).  false once j is past the CTA's last position.
// Position j is done when EVERY update warp has released it (each counts its own positions:
// a shared total would let warps running up to kNA stages ahead stand in for one still
// storing its slice of position j).  Relaxed polls, one acquire fence; false once j is past
// the CTA's last position.  Only the inbox warp waits here (the mix follows its slots).
__device__ __forceinline__ bool wait_position(const uint32_t* y_stored, volatile int* end_pos, int j) {
  const volatile uint32_t* ys = y_stored;
  for (;;) {
    bool all = true;
#pragma unroll
    for (int w = 0; w < kUpd / 32; ++w) all &= (int32_t)(ys[w] - (uint32_t)(j + 1)) >= 0;
    if (all) break;
    if (*end_pos <= j) return false;
  }
  asm volatile("fence.acq_rel.cta;" ::: "memory");
  return true;
}

__global__ void __launch_bounds__(kMThreads, 1) k_push_merge(const MergeArgs a) {
  extern __shared__ __align__(128) float smem_f[];
  float* ringA = smem_f;                                   // [kNA][3][kT]  x, m, g
  float* ringI = ringA + (size_t)kNA * 3 * kT;             // [kNI][2][kT]  received y (fp32/bf16), own y
  float* ringY = ringI + (size_t)kNI * 2 * kT;             // [kNY][kT]     y out (fp32)
  uint16_t* ringW = reinterpret_cast<uint16_t*>(ringY + (size_t)kNY * kT);  // [kNY][kT] bf16 image (wire)
  const PeerStepArgs& s0 = a.s;
  const bool wire = s0.wire != 0;
  const int n_loc = s0.n_loc;
  int64_t* bnd = reinterpret_cast<int64_t*>(wire ? reinterpret_cast<float*>(ringW + (size_t)kNY * kT)
                                                 : ringY + (size_t)kNY * kT);
  int32_t* t0 = reinterpret_cast<int32_t*>(bnd + s0.k + 1);
  uint32_t* ord = reinterpret_cast<uint32_t*>(t0 + s0.k + 1);  // [k][n_loc] walk order per segment
  int32_t* hdst = reinterpret_cast<int32_t*>(ord + s0.k * n_loc);  // [k][n_loc] receiver of a head row
  int32_t* claims = hdst + s0.k * n_loc;                   // [kMaxClaims] chunks claimed, -1 ends
  float* wsnap = reinterpret_cast<float*>(claims + kMaxClaims);  // [kMaxLoc] psw of a first tile's segment
  // [kWarps][192] prologue scratch in the inbox ring: nothing is staged there before the
  // topology barrier (the x/m/g warp, which may start early, uses its own ring)
  uint32_t* scratch = reinterpret_cast<uint32_t*>(ringI);
  __shared__ uint64_t a_full[kNA], a_empty[kNA], i_full[kNI], i_empty[kNI], y_full[kNY], y_free[kNY];
  __shared__ uint32_t ck_upd[kNY][kUpd / 32][2];  // per update warp: checksums of its pushed words
  __shared__ uint32_t w_upd[kNY];                 // push-sum weight bits sent with the tile (0: none)
  __shared__ int32_t dst_upd[kNY];                // receiving worker of a head's tile (-1: not a head)
  __shared__ uint4 meta[kNI];                     // trailer of the staged received tile (bulk-loaded)
  __shared__ uint4 meta_re;                       // trailer re-read by the mix after a failed check
  __shared__ uint32_t ck_mix[2][kMix / 32][2];    // per mix warp, double-buffered by round parity
  __shared__ uint32_t y_stored[kUpd / 32];  // per update warp: positions it has released
  __shared__ MixMeta mmeta[kNI];            // the tail staged in each inbox slot (row < 0: end)
  __shared__ int s_end;          // number of positions this CTA processes; INT_MAX until known
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
  // the rank's rows as locals (computed from the launch arguments)
  const int64_t vrows = a.vranks > 1 ? (int64_t)rc.rank * n_loc : 0;
  float* const X = s0.x + vrows * s0.ld;
  float* const M = s0.m + vrows * s0.ld;
  float* const PSW = s0.psw + vrows * s0.k;

  for (int i = threadIdx.x; i <= s.k; i += blockDim.x) {
    bnd[i] = a.bounds[i];
    t0[i] = a.seg_t0[i];
  }
  if (threadIdx.x == 0) {
    s_timeout = 0;
    s_end = 0x7fffffff;
    for (int w = 0; w < kUpd / 32; ++w) y_stored[w] = 0;
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
      ptx::mbar_init(&y_free[i], 1);  // the store warp is done with the slot
    }
    ptx::mbar_fence_init();
  }
  __syncthreads();  // mbarriers and segment tables ready
  const unsigned long long t_topo = a.trace ? ptx::globaltimer() : 0;
  // With one worker per GPU the walk is one row (a one-element chain): the x/m/g warp starts
  // loading at once, while the others draw the topology
  const bool solo = n_loc == 1;
  const int topo_threads = solo ? kMThreads - 32 : kMThreads;
  // ---- this step's topology restricted to this GPU's workers (Alg. 2):
  // per segment the walk order (chains first, from their heads, then the local cycles) and
  // the receiver of every chain head (send_to, Alg.1 l.6)
  {
    uint32_t* u = scratch + warp * 192;
    int32_t* srow = reinterpret_cast<int32_t*>(u + 64);   // [<= 64] the drawn row when fused
    int32_t* dstl = reinterpret_cast<int32_t*>(u + 128);  // [n_loc] receiver of each local worker
    const int ntop = s.gs > 0 ? s.groups : s.world;
    const int tw0 = solo ? (warp < kWLoadXmg ? warp : warp - 1) : warp, tnw = solo ? kWarps - 1 : kWarps;
    for (int sg = (solo && warp == kWLoadXmg) ? s.k : tw0; sg < s.k; sg += tnw) {
      if (s.gs > 0) {  // hierarchical leader exchange (one worker per GPU, replicated leader)
        if (lane == 0) dstl[0] = -1;
        __syncwarp();
        const int grp = s.rank / s.gs, member = s.rank - grp * s.gs;
        const int32_t* row;
        if (s.given != nullptr) row = s.given + (int64_t)sg * ntop;
        else if (a.fused_topo) {
          warp_alg2_small(s.seed, s.step, sg, ntop, CS_TAG_HIER, u, srow, s.err);
          row = srow;
        } else row = s.src + (int64_t)sg * ntop;
        __syncwarp();
        for (int jj = lane; jj < ntop; jj += 32)
          if (row[jj] == grp) dstl[0] = jj * s.gs + member;  // the member of the same index
        __syncwarp();
        if (lane == 0) {
          ord[sg] = 0u | kWStart | kWHead | kWEnd | kWTail;
          hdst[sg] = dstl[0];
        }
        __syncwarp();
        continue;
      }
      const int32_t* row;
      if (s.given != nullptr) row = s.given + (int64_t)sg * ntop;
      else if (a.fused_topo) {
        warp_alg2_small(s.seed, s.step, sg, ntop, CS_TAG_FLAT, u, srow, s.err);
        row = srow;
      } else row = s.src + (int64_t)sg * ntop;
      __syncwarp();
      const int first = s.first;
      for (int jj = lane; jj < ntop; jj += 32) {  // inverse on the local range: receivers
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
          hdst[sg * n_loc + r] = dg;
          int pr = r;
          uint32_t flag = kWStart | kWHead;
          while (true) {
            seen |= 1ull << pr;
            const int sgl = row[first + pr] - first;
            if (sgl < 0 || sgl >= n_loc) {  // source remote: chain tail
              o[pos++] = (uint32_t)pr | flag | kWEnd | kWTail;
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
          uint32_t flag = kWStart;
          do {
            seen |= 1ull << pr;
            const int nx = row[first + pr] - first;
            o[pos++] = (uint32_t)pr | flag | (nx == r0 ? kWEnd : 0u);
            flag = 0;
            pr = nx;
          } while (pr != r0);
        }
      }
      __syncwarp();
    }
  }
  if (!(solo && warp == kWLoadXmg)) ptx::named_bar_sync(2, topo_threads);
  unsigned long long* tr = a.trace ? a.trace + ((size_t)s.rank * G + b) * 8 : nullptr;
  if (tr && threadIdx.x == 0) {
    tr[0] = ptx::globaltimer();
    tr[3] = t_topo;
    tr[5] = t_entry;
  }
  uint4* trl_in = reinterpret_cast<uint4*>(mine + a.off_trl) + (size_t)par * a.trl_cap;

  if (warp < kUpd / 32) {
    // ---------------- update warps: a3 and the walk ---------------------------------
    const int tid = threadIdx.x;
    bool bad = false;
    int cur = 0;
    Walk w;
    w.init(n_loc);
    float4 yfirst[kPerU], yprev[kPerU];
    uint32_t prev_row = 0;
    int c = 0;  // positions with copies (chain heads and tails) so far: the y-out ring index
    for (int i = 0;; ++i) {
      const int st = i % kNA;
      ptx::mbar_wait(&a_full[st], (uint32_t)((i / kNA) & 1));
      if (!w.next(claims, a.chunk_t0, n_loc)) {  // end marker: pass it on to the store warp
        const int sy = c % kNY;
        ptx::mbar_wait(&y_free[sy], (uint32_t)(((c / kNY) & 1) ^ 1));
        if (tid == 0) dst_upd[sy] = -2;
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&y_full[sy]);
        break;
      }
      const MTile U = mtile(a, bnd, t0, w.t, cur);
      const uint32_t e_w = ord[U.seg * n_loc + w.p];
      const uint32_t row = e_w & kWIdx;
      const bool head = (e_w & kWHead) != 0, tail = (e_w & kWTail) != 0;
      const bool copy = head;  // the store warp has work for this position (a push)
      const int sy = c % kNY;
      if (copy) ptx::mbar_wait(&y_free[sy], (uint32_t)(((c / kNY) & 1) ^ 1));
      const float* bx = ringA + (size_t)st * 3 * kT;
      float4* yt = reinterpret_cast<float4*>(ringY + (size_t)sy * kT);
      const float rate = s.lrs ? __ldg(s.lrs + (int64_t)row * s.n_layers + U.layer) : s.lr;
      const uint32_t nw = wire ? (uint32_t)(U.len + 1) / 2 : (uint32_t)U.len;  // pushed words checked
      const int64_t rowoff = (int64_t)row * s.ld;
      if (U.first && w.p == 0 && tid == 0)  // the segment's psw before any merge of this step
        for (int r = 0; r < n_loc; ++r) wsnap[r] = PSW[(int64_t)r * s.k + U.seg];
      uint32_t cx = 0, cs = 0;
#pragma unroll
      for (int q = 0; q < kPerU; ++q) {
        const int v = tid + q * kUpd;
        const int valid = U.len - 4 * v;
        if (valid > 0) {
          const int vv = valid < 4 ? valid : 4;
          const int64_t j = U.c0 + 4 * (int64_t)v;
          const float4 cxv = reinterpret_cast<const float4*>(bx)[v];
          const float4 cm = reinterpret_cast<const float4*>(bx + kT)[v];
          float4 cg = reinterpret_cast<const float4*>(bx + 2 * kT)[v];
          if (s.g_scale != 1.f) cg = scale4(cg, s.g_scale);  // NCCL h1: the group sum -> mean
          bad |= nonfinite4(cg);
          // LARS (C-18): m' = mu*m + (g + wd*x), y = x - lrs[row][layer]*m'
          const float4 mn = mom4(cm, s.lrs ? decay4(cg, cxv, s.wd) : cg, s.mu);
          const float4 y = sgd4(cxv, mn, rate);
          st4_cs(M + rowoff + j, mn, vv);
          // the walk: x'_{prev} = mean(y_prev, y) (this row is prev's source, Alg.1 l.17),
          // a cycle closes with its first y; what a worker receives is bf16 on the bf16 wire
          if (e_w & kWStart) yfirst[q] = y;
          else st4_cs(X + (int64_t)prev_row * s.ld + j, mean4(yprev[q], wire ? bf16r4(y) : y), vv);
          if ((e_w & kWEnd) && !tail)
            st4_cs(X + rowoff + j, mean4(y, wire ? bf16r4(yfirst[q]) : yfirst[q]), vv);
          // a chain tail's y waits in params for the mix; the inbox warp bulk-loads it back
          // after every update warp released this position (proxy fence below)
          if (tail) st4(X + rowoff + j, y, vv);
          yprev[q] = y;
          if (head) {
            if (wire) {  // what the receiver gets (C-20)
              const uint2 pw = pack_bf16x4(y);
              reinterpret_cast<uint2*>(ringW + (size_t)sy * kT)[v] = pw;
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
      }
      prev_row = row;
      if (head) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          cx ^= __shfl_xor_sync(0xffffffffu, cx, o);
          cs += __shfl_xor_sync(0xffffffffu, cs, o);
        }
        if (lane == 0) {
          ck_upd[sy][warp][0] = cx;
          ck_upd[sy][warp][1] = cs;
        }
      }
      if (tid == 0) {
        // a head's tile goes to its receiver with the segment's weight on the first tile
        if (copy) {  // this position's slot (a position without a push has none)
          dst_upd[sy] = hdst[U.seg * n_loc + row];
          w_upd[sy] = U.first ? __float_as_uint(wsnap[row]) : 0u;
        }
        if (U.first && w.p == n_loc - 1)  // psw of the rows with a local source
          for (int p = 0; p < n_loc; ++p) {
            const uint32_t o = ord[U.seg * n_loc + p];
            if (o & kWTail) continue;  // merged with the received weight by the mix
            const uint32_t src = (o & kWEnd) ? 0xffffffffu : (ord[U.seg * n_loc + p + 1] & kWIdx);
            uint32_t sl = src;
            if (o & kWEnd) {  // a cycle's last member's source is the cycle's first
              int q2 = p;
              while (!(ord[U.seg * n_loc + q2] & kWStart)) --q2;
              sl = ord[U.seg * n_loc + q2] & kWIdx;
            }
            const uint32_t r = o & kWIdx;
            PSW[(int64_t)r * s.k + U.seg] = pair_mean1(wsnap[r], wsnap[sl]);
          }
      }
      if (copy) ptx::fence_proxy_async_shared();  // y tile -> the store warp's bulk copies
      if (tail) ptx::fence_proxy_async_global();  // y in params -> the inbox warp's bulk read
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive(&a_empty[st]);
        if (copy) ptx::mbar_arrive(&y_full[sy]);
      }
      if (lane == 0) red_add_release_cta(&y_stored[warp], 1u);  // this warp's part of the position
      if (copy) ++c;
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(s.err + kErrDiverged, 1);
    if (tr && threadIdx.x == 0) tr[1] = ptx::globaltimer();
  } else if (warp < (kUpd + kMix) / 32) {
    // ---------------- mix warps: a chain tail's verify + a5 -------------------------
    const int tm = threadIdx.x - kUpd, mw = tm >> 5;
    int retried = 0, round = 0, q = 0;  // round: checksum reductions (buffer parity); q: tails
    for (;;) {  // the tails in the order the inbox warp stages them
      const int si = q % kNI;
      ptx::mbar_wait(&i_full[si], (uint32_t)((q / kNI) & 1));
      ++q;
      const MixMeta mm = mmeta[si];
      if (mm.row < 0) break;  // end marker
      MTile U;
      U.c0 = mm.c0;
      U.len = mm.len;
      U.seg = mm.seg;
      U.first = mm.first != 0;
      const uint32_t row = (uint32_t)mm.row;
      const float* it = ringI + (size_t)si * 2 * kT;
      const uint32_t nw = wire ? (uint32_t)(U.len + 1) / 2 : (uint32_t)U.len;
      const float* inbox_f = reinterpret_cast<const float*>(mine + a.off_inbox) + ((int64_t)par * n_loc + row) * s.ld;
      const uint16_t* inbox_w =
          reinterpret_cast<const uint16_t*>(mine + a.off_inbox) + ((int64_t)par * n_loc + row) * ld_bf;
      const uint4* trl = trl_in + (size_t)mm.t * n_loc + row;
      uint4 tl = meta[si];
      uint4 raw[kPerM];  // the received words as pushed (fp32 bits, or 2 x 2 bf16 in .x .y)
      float4 yo[kPerM];  // the tail's own y (staged by the inbox warp)
#pragma unroll
      for (int qq = 0; qq < kPerM; ++qq) yo[qq] = reinterpret_cast<const float4*>(it + kT)[tm + qq * kMix];
#pragma unroll
      for (int qq = 0; qq < kPerM; ++qq) {
        const int v = tm + qq * kMix;
        if (wire) {
          const uint2 pw = reinterpret_cast<const uint2*>(it)[v];
          raw[qq] = make_uint4(pw.x, pw.y, 0u, 0u);
        } else {
          raw[qq] = reinterpret_cast<const uint4*>(it)[v];
        }
      }
      for (int attempt = 0;; ++attempt) {
        uint32_t cx = 0, cs = 0;
#pragma unroll
        for (int qq = 0; qq < kPerM; ++qq) {
          const int v = tm + qq * kMix;
          if (4 * v < U.len) {
            if (wire) {
              if (2u * v < nw) ck_add(cx, cs, raw[qq].x, 2u * v);
              if (2u * v + 1 < nw) ck_add(cx, cs, raw[qq].y, 2u * v + 1);
            } else {
              const uint32_t wv[4] = {raw[qq].x, raw[qq].y, raw[qq].z, raw[qq].w};
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
        uint32_t Xc = 0, Sc = 0;
#pragma unroll
        for (int m2 = 0; m2 < kMix / 32; ++m2) {
          Xc ^= ck_mix[pb][m2][0];
          Sc += ck_mix[pb][m2][1];
        }
        if (((Xc ^ tl.w) == tl.y && Sc == tl.z && tl.x == e) || *timeout) break;
        // not (yet) the tile the trailer describes: wait for this epoch's trailer, then read
        // trailer and words again from memory
        if (tm == 0) {
          if (tl.x == e) ++retried;  // the trailer had arrived but the words had not
          const uint64_t tin = tr ? ptx::globaltimer() : 0;
          uint64_t tw = 0;
          while ((int32_t)(ld_volatile1(trl) - e) < 0) {
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
          meta_re = ld_volatile4(trl);
        }
        ptx::named_bar_sync(kMixBar, kMix);
        tl = meta_re;
#pragma unroll
        for (int qq = 0; qq < kPerM; ++qq) {
          const int v = tm + qq * kMix;
          if (4 * v < U.len) {
            if (wire) {
              const uint2 pw = ld_volatile2(inbox_w + U.c0 + 4 * v);
              raw[qq] = make_uint4(pw.x, pw.y, 0u, 0u);
            } else {
              raw[qq] = ld_volatile4(inbox_f + U.c0 + 4 * v);
            }
          }
        }
      }
#pragma unroll
      for (int qq = 0; qq < kPerM; ++qq) {
        const int v = tm + qq * kMix;
        const int valid = U.len - 4 * v;
        if (valid > 0) {
          const float4 yr = wire ? unpack_bf16x4(make_uint2(raw[qq].x, raw[qq].y))
                                 : make_float4(__uint_as_float(raw[qq].x), __uint_as_float(raw[qq].y),
                                               __uint_as_float(raw[qq].z), __uint_as_float(raw[qq].w));
          st4_cs(X + (int64_t)row * s.ld + U.c0 + 4 * v, mean4(yo[qq], yr), valid < 4 ? valid : 4);  // Alg.1 l.17
        }
      }
      if (U.first && tm == 0) PSW[(int64_t)row * s.k + U.seg] = pair_mean1(PSW[(int64_t)row * s.k + U.seg],
                                                                          __uint_as_float(tl.w));
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&i_empty[si]);
    }
    if (tm == 0 && retried && a.retries) atomicAdd(a.retries, (unsigned)retried);
    if (tr && tm == 0) tr[6] = ptx::globaltimer();
  } else if (warp == kWLoadXmg) {
    // ---------------- claims + x, m, g loader ----------------------------------------
    if (s.gs > 0 && !s.gbar_local && lane < s.gs) {  // hierarchical: the group mean is complete on this GPU
      const uint32_t* d2 = reinterpret_cast<const uint32_t*>(mine + a.off_d2);
      const int gbase = (s.rank / s.gs) * s.gs;
      if (!ptx::wait_geq_sys(d2 + gbase + lane, e)) atomicOr(&s_timeout, 1);
    }
    __syncwarp();
    if (lane == 0) {
      ptx::fence_proxy_async_global();
      // claim counters by epoch parity: this step's starts at 0 (reset by the previous step)
      uint32_t* counter = reinterpret_cast<uint32_t*>(mine + a.off_claim) + par;
      const float* Gr = s.g;
      const float* Mr = M;
      int cur = 0, n_claims = 0, t = 0, t_end = 0, p = n_loc - 1;
      for (int i = 0;; ++i) {
        const int st = i % kNA;
        ptx::mbar_wait(&a_empty[st], (uint32_t)(((i / kNA) & 1) ^ 1));
        if (++p == n_loc) {
          p = 0;
          if (++t >= t_end) {  // claim the next chunk (segment order: the pace every GPU keeps)
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
        }
        const MTile U = mtile(a, bnd, t0, t, cur);
        const int64_t off = (solo ? 0 : (int64_t)(ord[U.seg * n_loc + p] & kWIdx)) * s.ld + U.c0;
        const uint32_t bytes = (uint32_t)(((U.len + 3) & ~3) * 4);
        float* buf = ringA + (size_t)st * 3 * kT;
        ptx::mbar_arrive_expect_tx(&a_full[st], 3 * bytes);
        ptx::bulk_g2s(buf, X + off, bytes, &a_full[st]);
        ptx::bulk_g2s(buf + kT, Mr + off, bytes, &a_full[st]);
        if (s.gpull_chunk > 0) bulk_load_g(s, a.peers, buf + 2 * kT, off, U.c0, bytes / 4, &a_full[st]);
        else ptx::bulk_g2s(buf + 2 * kT, Gr + off, bytes, &a_full[st]);
      }
    }
    __syncwarp();
  } else if (warp == kWLoadIn) {
    // ---------------- inbox loader: a chain tail's trailer, received and own y tiles ---
    // (lane 0 bulk-loads the trailer, the received tile and the tail's own y; the update warps'
    // generic stores of that y precede their fence.proxy.async and per-warp release, which
    // this warp acquires for every update warp before the bulk read)
    {
      int cur = 0, q = 0;
      Walk w;
      w.init(n_loc);
      for (int j = 0;; ++j) {
        if (!wait_position(y_stored, end_pos, j)) break;
        w.next(claims, a.chunk_t0, n_loc);
        const MTile U = mtile(a, bnd, t0, w.t, cur);
        const uint32_t e_w = ord[U.seg * n_loc + w.p];
        if (!(e_w & kWTail)) continue;
        const uint32_t row = e_w & kWIdx;
        // stage it once the update is `lag` positions further (the sender's copy has probably
        // completed by then), or at the end; the mix polls if the trailer is still old
        if (a.lag > 0) wait_position(y_stored, end_pos, j + a.lag);
        const int si = q % kNI;
        ptx::mbar_wait(&i_empty[si], (uint32_t)(((q / kNI) & 1) ^ 1));
        ++q;
        float* buf = ringI + (size_t)si * 2 * kT;
        const uint32_t yb = (uint32_t)(((U.len + 3) & ~3) * 4);
        const uint32_t ib = wire ? (uint32_t)(((U.len + 7) & ~7) * 2) : yb;
        if (lane == 0) {
          mmeta[si] = MixMeta{U.c0, U.len, U.seg, U.first ? 1 : 0, (int)row, w.t};  // published by the arrive
          ptx::mbar_arrive_expect_tx(&i_full[si], ib + yb + 16u);
          ptx::bulk_g2s(buf + kT, X + (int64_t)row * s.ld + U.c0, yb, &i_full[si]);  // own y
          ptx::bulk_g2s(&meta[si], trl_in + (size_t)w.t * n_loc + row, 16u, &i_full[si]);
          if (wire)
            ptx::bulk_g2s(buf, reinterpret_cast<const uint16_t*>(mine + a.off_inbox) +
                                   ((int64_t)par * n_loc + row) * ld_bf + U.c0,
                          ib, &i_full[si]);
          else
            ptx::bulk_g2s(buf, reinterpret_cast<const float*>(mine + a.off_inbox) +
                                   ((int64_t)par * n_loc + row) * s.ld + U.c0,
                          yb, &i_full[si]);
        }
      }
      // end marker for the mix (a plain arrive completes the slot's phase)
      const int si = q % kNI;
      ptx::mbar_wait(&i_empty[si], (uint32_t)(((q / kNI) & 1) ^ 1));
      if (lane == 0) {
        mmeta[si].row = -1;
        ptx::mbar_arrive(&i_full[si]);
      }
    }
    __syncwarp();
  } else if (warp == kWStore) {
    // ---------------- store warp: push head tiles, then each completed tile's trailer ---
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
      // positions whose copies were issued but are not yet known complete, oldest first: a
      // head's trailer waits for its copy, a tail's release to the inbox warp for its own
      // copies in flight before completion is awaited (c3 at 2 GPUs: 194.2 / 192.0 / 191.6 /
      // 191.3 us for 1 / 2 / 4 / 7; bf16 wire 198.2 -> 186.0 us; profiles/r02/m16)
      const int land = a.land > 0 ? a.land : 4;
      uint4* pend_dst[kQ] = {};
      uint4 pend_trl[kQ] = {};
      int pend_head = 0, npend = 0, cur = 0;
      int unfreed = 0, free_next = 0;  // y-out slots whose copies may still read them, oldest first
      auto free_oldest = [&]() {
        ptx::mbar_arrive(&y_free[free_next]);
        free_next = (free_next + 1) % kNY;
        --unfreed;
      };
      Walk w;
      w.init(n_loc);
      auto complete_oldest = [&]() {  // Alg.1 l.14: that position's copies have completed
        if (pend_dst[pend_head]) st_volatile4(pend_dst[pend_head], pend_trl[pend_head]);
        pend_head = (pend_head + 1) % kQ;
        --npend;
      };
      for (int c = 0;; ++c) {  // positions with copies only (chain heads and tails)
        const int sy = c % kNY;
        const uint32_t ph = (uint32_t)((c / kNY) & 1);
        if ((npend > 0 || unfreed > 0) && !ptx::mbar_test(&y_full[sy], ph)) {  // idle: finish what is in flight
          ptx::bulk_wait_all();
          ptx::fence_proxy_async_global();  // their async-proxy writes -> the trailer stores
          while (npend > 0) complete_oldest();
          while (unfreed > 0) free_oldest();
        }
        ptx::mbar_wait(&y_full[sy], ph);
        const int dg = dst_upd[sy];
        if (dg == -2) break;  // end marker
        MTile U;
        do {  // this slot's position: the next one with copies
          w.next(claims, a.chunk_t0, n_loc);
          U = mtile(a, bnd, t0, w.t, cur);
        } while (!(ord[U.seg * n_loc + w.p] & kWHead));
        const int q = (pend_head + npend) % kQ;
        pend_dst[q] = nullptr;
        if (dg >= 0) {  // a head: its y tile to the receiver's inbox row over NVLink (a4)
          const int rp = dg / n_loc, rl = dg - rp * n_loc;
          if (wire)
            ptx::bulk_s2g(reinterpret_cast<uint16_t*>(a.peers[rp] + a.off_inbox) + ((int64_t)par * n_loc + rl) * ld_bf +
                              U.c0,
                          ringW + (size_t)sy * kT, (uint32_t)(((U.len + 7) & ~7) * 2));
          else
            ptx::bulk_s2g(reinterpret_cast<float*>(a.peers[rp] + a.off_inbox) + ((int64_t)par * n_loc + rl) * s.ld +
                              U.c0,
                          ringY + (size_t)sy * kT, (uint32_t)(((U.len + 3) & ~3) * 4));
          uint32_t Xc = 0, Sc = 0;
#pragma unroll
          for (int u = 0; u < kUpd / 32; ++u) {
            Xc ^= ck_upd[sy][u][0];
            Sc += ck_upd[sy][u][1];
          }
          const uint32_t wb = w_upd[sy];
          pend_dst[q] = reinterpret_cast<uint4*>(a.peers[rp] + a.off_trl) + (size_t)par * a.trl_cap +
                        (size_t)w.t * n_loc + rl;
          pend_trl[q] = make_uint4(e, Xc ^ wb, Sc, wb);
        }
        ptx::bulk_commit();
        ++npend;
        ++unfreed;
        // slots are freed once their copies have read them, up to kReadLag positions late (the
        // update warps may run kNY copy positions ahead, so this never waits on them)
        bulk_wait_read_n(a.read_lag);
        while (unfreed > a.read_lag) free_oldest();
        if (npend > land) {  // all but the newest `land` positions' copies have completed
          bulk_wait_n(land);
          ptx::fence_proxy_async_global();
          while (npend > land) complete_oldest();
        }
      }
      ptx::bulk_wait_all();
      ptx::fence_proxy_async_global();
      if (tr) tr[2] = ptx::globaltimer();
      while (npend > 0) complete_oldest();
      while (unfreed > 0) free_oldest();
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
      ptx::fence_acq_rel_sys();  // one release for all the done words (relaxed stores after it)
      for (int q = 0; q < s.nprocs; ++q)
        ptx::st_relaxed_sys(reinterpret_cast<uint32_t*>(a.peers[q] + a.off_done) + s.rank, e);
      if (a.trace) a.trace[(size_t)a.vranks * G * 8 + s.rank] = ptx::globaltimer();
    }
  }
}

}  // namespace

size_t peer_merge_smem(int k, int n_loc) { return smem_bytes(k, n_loc, true); }

int peer_merge_capacity(int k) {
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = smem_bytes(1, kMaxKN, true);  // the largest walk tables, bf16 image
  cudaError_t e = cudaFuncSetAttribute(k_push_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_push_merge, kMThreads, smem);
  if (e != cudaSuccess || occ < 1) {  // never silently: the in-step schedule would be off
    fprintf(stderr, "crossover_sgd: k_push_merge cannot be resident (%s, smem %zu); in-step merge disabled\n",
            cudaGetErrorString(e), smem);
    cudaGetLastError();
    return 0;
  }
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
  return p.sched == kSchedInStep && a.n_loc <= kMaxLoc && (int64_t)a.k * a.n_loc <= kMaxKN && a.k <= kMaxK &&
         p.grid_merge > 0 && p.d_chunk_t0 != nullptr && (int64_t)p.n_tiles * a.n_loc <= p.mflag_cap &&
         // every CTA's claims fit its list even if one CTA took 4x its share
         (int64_t)p.n_chunks < (int64_t)(kMaxClaims - 1) * p.grid_merge / 4;
}

cudaError_t peer_launch(const PeerState& p, const void* fn, int grid_per_rank, int threads, size_t smem,
                        cudaStream_t st, void** args) {
  ++g_peer_launches;
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
  static const int lag = getenv("CS_MERGE_LAG") ? atoi(getenv("CS_MERGE_LAG")) : 4;  // c3 at 2 GPUs: 188.5 / 185.2 / 180.5 us for 0 / 2 / 4 (profiles/r02/m18)
  ma.lag = lag < 0 ? 0 : lag;
  static const int read_lag = getenv("CS_MERGE_READLAG") ? atoi(getenv("CS_MERGE_READLAG")) : kReadLag;
  ma.read_lag = read_lag < 0 ? 0 : (read_lag > kReadLag ? kReadLag : read_lag);
  static const int land = getenv("CS_MERGE_LAND") ? atoi(getenv("CS_MERGE_LAND")) : 0;
  ma.land = land < 0 ? 0 : (land > kQ - 1 ? kQ - 1 : land);
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
  cudaError_t e = peer_launch(p, (const void*)k_push_merge, p.grid_merge, kMThreads, smem_bytes(a.k, a.n_loc, a.wire != 0), st, args);
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
    const char* names[8] = {"start", "update_end", "push_landed", "topo_begin", "trailer_wait_us", "entry",
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
