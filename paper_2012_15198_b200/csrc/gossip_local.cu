// Single-GPU hot path: every worker co-resident in this GPU's HBM (configs 1, 2;
// the paper itself ran "multiple processes for each GPU").
//
// ONE launch per step.  k_gossip_local fuses, per float4 column (4 consecutive
// parameters), for all n workers:
//   a2  (prologue, every CTA) the k per-segment topologies of this step — Alg. 2
//       from the shared seed, PAPER.md:165-191 — and their cycle order, into
//       shared memory (no communication, no separate topology kernel)
//   a3  m_i <- fl(fl(mu*m_i) + g_i);  y_i <- fl(x_i - fl(lr*m_i))   (C-8, C-9)
//   a4  receive y_{src_s(i)} — here an HBM row already in flight in this thread
//   a5  x_i <- fl(fl(y_i + y_{src_s(i)}) * 0.5)                    (Alg.1 l.17)
//       and (epilogue, last CTA) psw_{i,s} <- (psw_{i,s} + psw_{src,s}) * 0.5
//   a6  (DIAG) fp64 shifted sums of z = x'/w' per column -> per-block partials,
//       reduced in a fixed order by the last CTA (deterministic)
//
// Column-owner cycle walk: the thread that owns column j visits the workers of
// segment s(j) in the cycle order of src_s, so y_{c_p} and y_{c_{p+1}} =
// y_{src(c_p)} are both in registers when x'_{c_p} is written; each of x, m, g
// is read exactly once and x, m written exactly once: the algorithmic 20 B per
// parameter per worker, in place, with no ping-pong buffer (every element is
// read by its owner before its owner writes it).  The loads of the next PF
// workers' rows are issued before the current row's arithmetic (register
// pipeline) to keep enough bytes in flight per SM.
//
// All fp32 arithmetic uses __fmul_rn/__fadd_rn/__fsub_rn: never contracted to
// FMA, so results are bit-identical to the oracle's separately rounded ops.
#include <stdlib.h>

#include "arith.cuh"
#include "common.cuh"
#include "ptx.cuh"
#include "philox.cuh"
#include "topo_device.cuh"

namespace cs {

namespace {

__device__ __forceinline__ float4 ld_stream(const float* p) {
  return __ldcs(reinterpret_cast<const float4*>(p));
}

__device__ __forceinline__ void st_stream(float* p, const float4 v, int valid) {
  if (valid == 4) {
    __stcs(reinterpret_cast<float4*>(p), v);
  } else {
    if (valid > 0) p[0] = v.x;
    if (valid > 1) p[1] = v.y;
    if (valid > 2) p[2] = v.z;
  }
}



// index of the last bound <= j among bounds[0 .. count) (bounds ascending, bounds[0] = 0)
__device__ __forceinline__ int last_bound_le(const int64_t* bounds, int count, int64_t j) {
  int s = 0;
  for (int lo = 0, hi = count - 1; lo <= hi;) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(bounds + mid) <= j) { s = mid; lo = mid + 1; } else { hi = mid - 1; }
  }
  return s;
}

// LARS carry helpers: fp64 sum of squares of the first `valid` lanes, fixed-order warp sum
__device__ __forceinline__ double sumsq4(double acc, float4 v, int valid) {
  acc = __dadd_rn(acc, __dmul_rn((double)v.x, (double)v.x));
  if (valid > 1) acc = __dadd_rn(acc, __dmul_rn((double)v.y, (double)v.y));
  if (valid > 2) acc = __dadd_rn(acc, __dmul_rn((double)v.z, (double)v.z));
  if (valid > 3) acc = __dadd_rn(acc, __dmul_rn((double)v.w, (double)v.w));
  return acc;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}





// Per-column fp64 accumulators for the consensus diagnostics, shifted by the
// first value c seen in the column so the variance does not cancel near consensus.
struct ColDiag {
  double c[4], s1[4], s2[4], xs[4];
  __device__ __forceinline__ void reset() {
#pragma unroll
    for (int e = 0; e < 4; ++e) { c[e] = 0.0; s1[e] = 0.0; s2[e] = 0.0; xs[e] = 0.0; }
  }
  // add `mult` identical workers with value x' and 1/w' = rw
  __device__ __forceinline__ void add(float4 xv, double rw, bool first, double mult) {
    const float xa[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      double z = (double)xa[e] * rw;
      if (first) c[e] = z;
      double dz = z - c[e];
      s1[e] += mult * dz;
      s2[e] += mult * dz * dz;
      xs[e] += mult * (double)xa[e];
    }
  }
  // column j's contribution: sum_i (z_ij - zbar_j)^2 = S2 - 2(zbar-c)S1 + n(zbar-c)^2, and zbar_j
  __device__ __forceinline__ void finish(double inv_wsum, double n, int valid, double& dacc,
                                         double& zacc) const {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (e < valid) {
        double zbar = xs[e] * inv_wsum;
        double dm = zbar - c[e];
        dacc += s2[e] - 2.0 * dm * s1[e] + n * dm * dm;
        zacc += zbar;
      }
    }
  }
};

__device__ __forceinline__ void block_reduce_store(double a, double b, double* out) {
  __shared__ double red[2][32];
  const unsigned FULL = 0xffffffffu;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    a += __shfl_xor_sync(FULL, a, off);
    b += __shfl_xor_sync(FULL, b, off);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { red[0][warp] = a; red[1][warp] = b; }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    a = lane < nw ? red[0][lane] : 0.0;
    b = lane < nw ? red[1][lane] : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      a += __shfl_xor_sync(FULL, a, off);
      b += __shfl_xor_sync(FULL, b, off);
    }
    if (lane == 0) { out[2 * blockIdx.x] = a; out[2 * blockIdx.x + 1] = b; }
  }
}

// Shared-memory tables of the fused prologue.
struct SmemTopo {
  double* rw;       // [k][n]   1 / w'_{rank,s}  (DIAG)
  double* iws;      // [k]      1 / sum_rows w'_{.,s}  (DIAG)
  uint32_t* ord;    // [k][n]   cycle order
  int32_t* src;     // [k][n]
  float* wsn;       // [n][k]   psw snapshot of each rank's (leader) row
  uint32_t* scratch;  // [warps][64] Philox words
};

__host__ __device__ inline size_t fused_smem_bytes(int n, int k, int warps, bool diag) {
  size_t b = 0;
  if (diag) b += sizeof(double) * ((size_t)k * n + k);
  b += sizeof(uint32_t) * (size_t)k * n;  // ord
  b += sizeof(int32_t) * (size_t)k * n;   // src
  b += sizeof(float) * (size_t)n * k;     // wsn
  b += sizeof(uint32_t) * 64 * warps;     // scratch
  return b;
}

__device__ SmemTopo carve(unsigned char* base, int n, int k, bool diag) {
  SmemTopo t;
  size_t off = 0;
  if (diag) {
    t.rw = reinterpret_cast<double*>(base);
    off += sizeof(double) * (size_t)k * n;
    t.iws = reinterpret_cast<double*>(base + off);
    off += sizeof(double) * k;
  } else {
    t.rw = nullptr;
    t.iws = nullptr;
  }
  t.ord = reinterpret_cast<uint32_t*>(base + off);
  off += sizeof(uint32_t) * (size_t)k * n;
  t.src = reinterpret_cast<int32_t*>(base + off);
  off += sizeof(int32_t) * (size_t)k * n;
  t.wsn = reinterpret_cast<float*>(base + off);
  off += sizeof(float) * (size_t)n * k;
  t.scratch = reinterpret_cast<uint32_t*>(base + off);
  return t;
}

// w'_{i,s} from the snapshot (n >= 2 mixes with the source; a single leader keeps its weight)
__device__ __forceinline__ float mixed_weight(const SmemTopo& t, int n, int k, int s, int i) {
  const float wi = t.wsn[i * k + s];
  return n >= 2 ? pair_mean1(wi, t.wsn[t.src[s * n + i] * k + s]) : wi;
}

// Prologue of the fused kernels: every CTA builds this step's tables.
template <bool DIAG>
__device__ void build_topology_smem(const LocalArgs& a, const SmemTopo& t) {
  const int n = a.n, k = a.k, gs = a.group_size;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int e = threadIdx.x; e < n * k; e += blockDim.x) {
    const int i = e / k, s = e - i * k;
    t.wsn[e] = a.psw[(int64_t)i * gs * k + s];
  }
  for (int s = wid; s < k; s += nwarps) {
    int32_t* srow = t.src + s * n;
    if (a.given != nullptr) {
      for (int i = lane; i < n; i += 32) srow[i] = a.given[(int64_t)s * n + i];
      __syncwarp();
    } else if (n == 1) {
      if (lane == 0) srow[0] = 0;
      __syncwarp();
    } else {
      warp_alg2_small(a.seed, a.step, s, n, a.tag, t.scratch + 64 * wid, srow, a.err);
    }
    if (lane == 0) {  // cycle order: c0, src(c0), src(src(c0)), ...
      uint64_t seen = 0;
      int pos = 0;
      for (int i0 = 0; i0 < n; ++i0) {
        if ((seen >> i0) & 1ull) continue;
        int p = i0;
        uint32_t flag = kOrdStart;
        do {
          seen |= 1ull << p;
          const int nx = srow[p];
          t.ord[s * n + pos++] = (uint32_t)p | flag | (nx == i0 ? kOrdEnd : 0u);
          flag = 0;
          p = nx;
        } while (p != i0);
      }
    }
  }
  __syncthreads();
  if (DIAG) {
    for (int e = threadIdx.x; e < n * k; e += blockDim.x) {
      const int s = e / n, i = e - s * n;
      t.rw[e] = 1.0 / (double)mixed_weight(t, n, k, s, i);
    }
    for (int s = threadIdx.x; s < k; s += blockDim.x) {
      double sum = 0.0;
      for (int i = 0; i < n; ++i) sum += (double)mixed_weight(t, n, k, s, i) * (double)gs;
      t.iws[s] = 1.0 / sum;
    }
    __syncthreads();
  }
}

// Epilogue: the last CTA to arrive writes the mixed push-sum weights (fused path)
// and reduces the diagnostics partials in a fixed order.
template <bool DIAG, bool FUSED>
__device__ void finish_step(const LocalArgs& a, const SmemTopo& t, double dacc, double zacc) {
  __shared__ int s_last;
  if (DIAG) block_reduce_store(dacc, zacc, a.partials);
  if (!DIAG && !FUSED) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(a.counter, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int n = a.n, k = a.k, gs = a.group_size;
  if (FUSED && !a.skip_psw) {
    for (int e = threadIdx.x; e < n * k; e += blockDim.x) {
      const int i = e / k, s = e - i * k;
      const float wn = mixed_weight(t, n, k, s, i);
      for (int r = 0; r < gs; ++r) a.psw[((int64_t)i * gs + r) * k + s] = wn;
    }
  }
  if (DIAG && threadIdx.x < 32) {
    double da = 0.0, za = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) {
      da += __ldcg(a.partials + 2 * b);
      za += __ldcg(a.partials + 2 * b + 1);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      da += __shfl_xor_sync(0xffffffffu, da, off);
      za += __shfl_xor_sync(0xffffffffu, za, off);
    }
    if (threadIdx.x == 0) {
      a.diag_out[0] = sqrt(fmax(da, 0.0) / ((double)n * gs));
      a.diag_out[1] = za;
    }
  }
  if (threadIdx.x == 0) {
    if (a.claim_next) *a.claim_next = 0u;  // the next launch's tile counter
    *a.counter = 0u;
  }
}

}  // namespace

constexpr int kThreads = 256;

template <int PF, bool DIAG, bool FUSED>
__global__ void __launch_bounds__(kThreads) k_gossip_local(const LocalArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int n = a.n;
  const int64_t ld = a.ld, d = a.d;
  const int64_t nvec = (d + 3) >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const float mu = a.mu, lr = a.lr;
  double dacc = 0.0, zacc = 0.0;
  bool bad = false;

  SmemTopo t = carve(smem_raw, n, a.k, DIAG && FUSED);
  if (FUSED) build_topology_smem<DIAG>(a, t);
  const uint32_t* ord_all = FUSED ? t.ord : a.ord;
  const double* rw_all = FUSED ? t.rw : a.rw;
  const double* iws_all = FUSED ? t.iws : a.inv_wsum;

  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += stride) {
    const int64_t j = v << 2;
    const int valid = (int)imin64(4, d - j);
    // segment of column j (reading C-2): the largest s with 32*floor(s*nq/k) <= j
    const int64_t q = j >> 5;
    const int s = (int)imin64(a.k - 1, ((q + 1) * a.k - 1) / a.nq);
    const uint32_t* ord = ord_all + (int64_t)s * n;
    const double* rw = DIAG ? rw_all + (int64_t)s * n : nullptr;

    float4 bx[PF], bm[PF], bg[PF];
    uint32_t be[PF];
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      if (u < n) {
        be[u] = ord[u];
        const int64_t off = (int64_t)(be[u] & kOrdIdx) * ld + j;
        bx[u] = ld_stream(a.x + off);
        bm[u] = ld_stream(a.m + off);
        bg[u] = ld_stream(a.g + off);
      }
    }
    float4 yfirst = make_float4(0.f, 0.f, 0.f, 0.f), yprev = yfirst;
    int64_t prev_off = 0;
    uint32_t prev_row = 0;
    ColDiag cd;
    if (DIAG) cd.reset();
    bool first_diag = true;

    for (int p0 = 0; p0 < n; p0 += PF) {
#pragma unroll
      for (int u = 0; u < PF; ++u) {
        const int p = p0 + u;
        if (p < n) {
          const float4 cx = bx[u], cm = bm[u], cg = bg[u];
          const uint32_t e = be[u];
          if (p + PF < n) {  // refill this slot with the row PF ahead
            be[u] = ord[p + PF];
            const int64_t off2 = (int64_t)(be[u] & kOrdIdx) * ld + j;
            bx[u] = ld_stream(a.x + off2);
            bm[u] = ld_stream(a.m + off2);
            bg[u] = ld_stream(a.g + off2);
          }
          const uint32_t row = e & kOrdIdx;
          const int64_t off = (int64_t)row * ld + j;
          bad |= nonfinite4(cg);
          const float4 mn = mom4(cm, cg, mu);
          const float4 y = sgd4(cx, mn, lr);
          st_stream(a.m + off, mn, valid);
          if (e & kOrdStart) {
            yfirst = y;
          } else {
            const float4 xo = mean4(yprev, a.wire ? bf16r4(y) : y);
            st_stream(a.x + prev_off, xo, valid);
            if (DIAG) { cd.add(xo, rw[prev_row], first_diag, 1.0); first_diag = false; }
          }
          if (e & kOrdEnd) {
            const float4 xo = mean4(y, a.wire ? bf16r4(yfirst) : yfirst);
            st_stream(a.x + off, xo, valid);
            if (DIAG) { cd.add(xo, rw[row], first_diag, 1.0); first_diag = false; }
          }
          yprev = y;
          prev_off = off;
          prev_row = row;
        }
      }
    }
    if (DIAG) cd.finish(iws_all[s], (double)n, valid, dacc, zacc);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(a.err + kErrDiverged, 1);
  finish_step<DIAG, FUSED>(a, t, dacc, zacc);
}

// Hierarchical step with every worker co-resident (§3.3):
//   h1  gbar_G = fl(sum over members, ascending) * fp32(1/|G|)
//   h2  leader: m <- mu*m + gbar, y <- x - lr*m; then the cycle walk over the
//       leader topology mixes leaders' y (tag HIER); one leader: x' = y
//   h3  x' written to every member row of the group (bitwise identical)
template <bool DIAG, bool FUSED, bool LAYERS>
__global__ void __launch_bounds__(kThreads) k_hier_local(const LocalArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int L = a.n, gs = a.group_size;
  const int64_t ld = a.ld, d = a.d;
  const int64_t nvec = (d + 3) >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const float mu = a.mu, lr = a.lr, inv = a.inv_group;
  double dacc = 0.0, zacc = 0.0;
  bool bad = false;

  SmemTopo t = carve(smem_raw, L, a.k, DIAG && FUSED);
  if (FUSED) build_topology_smem<DIAG>(a, t);
  const uint32_t* ord_all = FUSED ? t.ord : a.ord;
  const double* rw_all = FUSED ? t.rw : a.rw;
  const double* iws_all = FUSED ? t.iws : a.inv_wsum;

  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += stride) {
    const int64_t j = v << 2;
    const int valid = (int)imin64(4, d - j);
    const int64_t q = j >> 5;
    int s = (int)imin64(a.k - 1, ((q + 1) * a.k - 1) / a.nq);
    if (LAYERS && a.seg_bounds) s = last_bound_le(a.seg_bounds, a.k, j);  // layer plan (C-19)
    const int layer = (LAYERS && a.lrs) ? last_bound_le(a.layer_bounds, a.n_layers, j) : 0;
    const uint32_t* ord = ord_all + (int64_t)s * L;
    const double* rw = DIAG ? rw_all + (int64_t)s * L : nullptr;
    float4 yfirst = make_float4(0.f, 0.f, 0.f, 0.f), yprev = yfirst;
    uint32_t prev_leader = 0;
    ColDiag cd;
    if (DIAG) cd.reset();
    bool first_diag = true;

    for (int p = 0; p < L; ++p) {
      const uint32_t e = ord[p];
      const uint32_t G = e & kOrdIdx;
      const int64_t lead_off = (int64_t)G * gs * ld + j;
      const float4 cx = ld_stream(a.x + lead_off);
      const float4 cm = ld_stream(a.m + lead_off);
      float4 gsum = ld_stream(a.g + lead_off);
      bad |= nonfinite4(gsum);
      // the members' rows are loaded 8 at a time (independent loads in flight), then added
      // in ascending member order (reading C-12), so the sum is the same bits
      int r = 1;
      for (; r + 8 <= gs; r += 8) {
        float4 gb[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) gb[u] = ld_stream(a.g + lead_off + (int64_t)(r + u) * ld);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          bad |= nonfinite4(gb[u]);
          gsum = make_float4(__fadd_rn(gsum.x, gb[u].x), __fadd_rn(gsum.y, gb[u].y),
                             __fadd_rn(gsum.z, gb[u].z), __fadd_rn(gsum.w, gb[u].w));
        }
      }
      for (; r < gs; ++r) {
        const float4 gr = ld_stream(a.g + lead_off + (int64_t)r * ld);
        bad |= nonfinite4(gr);
        gsum = make_float4(__fadd_rn(gsum.x, gr.x), __fadd_rn(gsum.y, gr.y),
                           __fadd_rn(gsum.z, gr.z), __fadd_rn(gsum.w, gr.w));
      }
      const float4 gbar = make_float4(__fmul_rn(gsum.x, inv), __fmul_rn(gsum.y, inv),
                                      __fmul_rn(gsum.z, inv), __fmul_rn(gsum.w, inv));
      // LARS on the group-reduced gradient (C-18): m' = mu*m + (gbar + wd*x)
      const bool lars = LAYERS && a.lrs;
      const float4 mn = mom4(cm, lars ? decay4(gbar, cx, a.wd) : gbar, mu);
      const float4 y = sgd4(cx, mn, lars ? __ldg(a.lrs + (int64_t)G * a.n_layers + layer) : lr);
      st_stream(a.m + lead_off, mn, valid);
      if (L == 1) {
        for (int r = 0; r < gs; ++r) st_stream(a.x + lead_off + (int64_t)r * ld, y, valid);
        if (DIAG) cd.add(y, rw[G], true, (double)gs);
        continue;
      }
      if (e & kOrdStart) {
        yfirst = y;
      } else {
        const float4 xo = mean4(yprev, y);
        const int64_t po = (int64_t)prev_leader * gs * ld + j;
        for (int r = 0; r < gs; ++r) st_stream(a.x + po + (int64_t)r * ld, xo, valid);
        if (DIAG) { cd.add(xo, rw[prev_leader], first_diag, (double)gs); first_diag = false; }
      }
      if (e & kOrdEnd) {
        const float4 xo = mean4(y, yfirst);
        for (int r = 0; r < gs; ++r) st_stream(a.x + lead_off + (int64_t)r * ld, xo, valid);
        if (DIAG) { cd.add(xo, rw[G], first_diag, (double)gs); first_diag = false; }
      }
      yprev = y;
      prev_leader = G;
    }
    if (DIAG) cd.finish(iws_all[s], (double)L * gs, valid, dacc, zacc);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(a.err + kErrDiverged, 1);
  finish_step<DIAG, FUSED>(a, t, dacc, zacc);
}

// ----------------------------------------------------------------------------
// Bulk-TMA variant of the flat single-GPU step (the default for n <= 64).
//
// Same column-owner cycle walk, but the rows of a column tile (up to 2048
// consecutive parameters of one segment) are staged in shared memory by 1-D
// bulk TMA copies (cp.async.bulk ... mbarrier::complete_tx), 8 KB per array per
// row, instead of per-thread 16-byte loads: every DRAM request is a long
// contiguous burst.  Warp-specialised: warp 8 (one elected lane) is the
// producer, walking the same (tile, cycle position) sequence as the consumers
// and refilling a kStages-deep ring of {x, m, g} row-tiles; warps 0-7 consume,
// each thread owning kVPT float4 columns of the tile, keeping y_first / y_prev
// of its columns in registers and storing x', m' straight to HBM.
// ----------------------------------------------------------------------------
namespace {

constexpr int kTmaConsumers = 256;
constexpr int kTmaThreads = kTmaConsumers + 32;
constexpr int kVPT = kTmaTileMax / (4 * kTmaConsumers);  // float4 columns per consumer thread
constexpr int kStages = 4;
constexpr size_t kStageBytes = 3ull * kTmaTileMax * sizeof(float);

using ptx::bulk_g2s;
using ptx::mbar_arrive;
using ptx::mbar_arrive_expect_tx;
using ptx::mbar_init;
using ptx::mbar_wait;
using ptx::smem_addr;


__host__ __device__ inline size_t tma_smem_bytes(int n, int k, bool diag) {
  return kStages * kStageBytes + 2 * kStages * sizeof(uint64_t) + kStages * (sizeof(float) + sizeof(int)) +
         sizeof(double) * (kTmaConsumers / 32) * (size_t)n +  // LARS: per-warp x'^2 sums per row
         fused_smem_bytes(n, k, kTmaThreads / 32, diag);
}

}  // namespace

// LARS (reading C-18): the producer stages the row's per-layer rate
// lrs[row][tile.layer] with each ring slot (st.shared before the release-arrive), and
// the update becomes m' = mu*m + (g + wd*x), y = x - rate*m'.
template <bool DIAG, bool LARS>
__global__ void __launch_bounds__(kTmaThreads) k_gossip_tma(const LocalArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stage_buf = reinterpret_cast<float*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  float* srate = reinterpret_cast<float*>(empty + kStages);  // [kStages]
  int* stile = reinterpret_cast<int*>(srate + kStages);       // [kStages] tile of a slot's first row; -1 ends
  double* wpart = reinterpret_cast<double*>(stile + kStages);  // [n][8] (LARS carry)
  SmemTopo t = carve(reinterpret_cast<unsigned char*>(wpart + (kTmaConsumers / 32) * a.n), a.n, a.k, DIAG);

  const int n = a.n;
  const int64_t ld = a.ld;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTmaConsumers / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  build_topology_smem<DIAG>(a, t);  // ends with __syncthreads (also publishes the barriers)

  double dacc = 0.0, zacc = 0.0;
  if (warp == kTmaConsumers / 32) {
    // ---------------- producer warp -------------------------------------------
    // tiles: claimed one at a time from the launch's counter (dynamic: CTAs that stream
    // faster take more; the table ends in small tiles so the last claims are short), or
    // round robin.  The tile index travels with the slot of its first row; -1 ends.
    uint32_t it = 0;
    auto next_tile = [&](int prev) {
      int u = prev < 0 ? (int)blockIdx.x : prev + (int)gridDim.x;
      if (a.claim) {
        if (lane == 0) u = (int)atomicAdd(a.claim, 1u);
        u = __shfl_sync(0xffffffffu, u, 0);
      }
      return u;
    };
    for (int u = next_tile(-1); u < a.n_tiles; u = next_tile(u)) {
      const TileDesc td = a.tiles[u];
      const uint32_t bytes = (uint32_t)(((td.len + 3) & ~3) * sizeof(float));
      const uint32_t* ord = t.ord + td.seg * n;
      for (int p = 0; p < n; ++p, ++it) {
        if (lane == 0) {
          const int st = (int)(it % kStages);
          mbar_wait(&empty[st], ((it / kStages) & 1u) ^ 1u);
          const int64_t off = (int64_t)(ord[p] & kOrdIdx) * ld + td.c0;
          float* buf = stage_buf + (size_t)st * 3 * kTmaTileMax;
          if (LARS) srate[st] = a.lrs[(int64_t)(ord[p] & kOrdIdx) * a.n_layers + td.layer];
          if (p == 0) stile[st] = u;
          mbar_arrive_expect_tx(&full[st], 3 * bytes);
          bulk_g2s(buf, a.x + off, bytes, &full[st]);
          bulk_g2s(buf + kTmaTileMax, a.m + off, bytes, &full[st]);
          bulk_g2s(buf + 2 * kTmaTileMax, a.g + off, bytes, &full[st]);
        }
        __syncwarp();
      }
    }
    if (lane == 0) {  // end marker
      const int st = (int)(it % kStages);
      mbar_wait(&empty[st], ((it / kStages) & 1u) ^ 1u);
      stile[st] = -1;
      mbar_arrive(&full[st]);
    }
  } else {
    // ---------------- consumer warps ------------------------------------------
    const float mu = a.mu, lr = a.lr;
    bool bad = false;
    uint32_t it = 0;
    for (;;) {
      mbar_wait(&full[it % kStages], (it / kStages) & 1u);  // the tile's first row (or the end)
      const int u = stile[it % kStages];
      if (u < 0) break;
      const TileDesc td = a.tiles[u];
      const uint32_t* ord = t.ord + td.seg * n;
      const double* rw = DIAG ? t.rw + td.seg * n : nullptr;
      float4 yfirst[kVPT], yprev[kVPT];
      ColDiag cd[kVPT];
      if (DIAG) {
#pragma unroll
        for (int c = 0; c < kVPT; ++c) cd[c].reset();
      }
      bool first_diag = true;
      uint32_t prev_row = 0;
      for (int p = 0; p < n; ++p, ++it) {
        const int st = (int)(it % kStages);
        if (p > 0) mbar_wait(&full[st], (it / kStages) & 1u);
        const float* buf = stage_buf + (size_t)st * 3 * kTmaTileMax;
        const uint32_t e = ord[p];
        const uint32_t row = e & kOrdIdx;
        const float rate = LARS ? srate[st] : lr;
        double qa = 0.0, qb = 0.0;  // LARS carry: this thread's sum of x'^2 for prev_row / row
#pragma unroll
        for (int c = 0; c < kVPT; ++c) {
          const int v = c * kTmaConsumers + threadIdx.x;       // float4 index in the tile
          const int valid = td.len - 4 * v;
          if (valid > 0) {
            const int vv = valid < 4 ? valid : 4;
            const float4 cx = reinterpret_cast<const float4*>(buf)[v];
            const float4 cm = reinterpret_cast<const float4*>(buf + kTmaTileMax)[v];
            const float4 cg = reinterpret_cast<const float4*>(buf + 2 * kTmaTileMax)[v];
            bad |= nonfinite4(cg);
            const float4 mn = mom4(cm, LARS ? decay4(cg, cx, a.wd) : cg, mu);
            const float4 y = sgd4(cx, mn, rate);
            const int64_t j = td.c0 + 4 * v;
            st_stream(a.m + (int64_t)row * ld + j, mn, vv);
            if (e & kOrdStart) {
              yfirst[c] = y;
            } else {
              const float4 xo = mean4(yprev[c], a.wire ? bf16r4(y) : y);
              st_stream(a.x + (int64_t)prev_row * ld + j, xo, vv);
              if (DIAG) cd[c].add(xo, rw[prev_row], first_diag, 1.0);
              if (LARS) qa = sumsq4(qa, xo, vv);
            }
            if (e & kOrdEnd) {
              const float4 xo = mean4(y, a.wire ? bf16r4(yfirst[c]) : yfirst[c]);
              st_stream(a.x + (int64_t)row * ld + j, xo, vv);
              if (DIAG) cd[c].add(xo, rw[row], first_diag && (e & kOrdStart), 1.0);
              if (LARS) qb = sumsq4(qb, xo, vv);
            }
            yprev[c] = y;
          }
        }
        if (DIAG && ((e & kOrdStart) == 0 || (e & kOrdEnd))) first_diag = false;
        if (LARS && a.xnorm_out) {  // per-warp sums (fixed shuffle order) of each row's x'^2
          if (!(e & kOrdStart)) {
            const double s = warp_sum(qa);
            if (lane == 0) wpart[prev_row * (kTmaConsumers / 32) + warp] = s;
          }
          if (e & kOrdEnd) {
            const double s = warp_sum(qb);
            if (lane == 0) wpart[row * (kTmaConsumers / 32) + warp] = s;
          }
        }
        prev_row = row;
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
      }
      if (LARS && a.xnorm_out) {  // the tile's x'^2 per row, warps in order -> .x of part[u][row]
        asm volatile("bar.sync 1, %0;" ::"n"(kTmaConsumers) : "memory");
        if (warp == 0)
          for (int r = lane; r < n; r += 32) {
            double s = 0.0;
            for (int w = 0; w < kTmaConsumers / 32; ++w) s = __dadd_rn(s, wpart[r * (kTmaConsumers / 32) + w]);
            a.xnorm_out[2 * ((int64_t)u * n + r)] = s;
          }
        asm volatile("bar.sync 1, %0;" ::"n"(kTmaConsumers) : "memory");
      }
      if (DIAG) {
#pragma unroll
        for (int c = 0; c < kVPT; ++c) {
          const int v = c * kTmaConsumers + threadIdx.x;
          const int valid = td.len - 4 * v;
          if (valid > 0) cd[c].finish(t.iws[td.seg], (double)n, valid < 4 ? valid : 4, dacc, zacc);
        }
      }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.err + kErrDiverged, 1);
  }
  finish_step<DIAG, true>(a, t, dacc, zacc);
}

int tma_grid(int n, int k, bool diag) {
  const size_t smem = tma_smem_bytes(n, k, diag);
  auto kern = diag ? k_gossip_tma<true, false> : k_gossip_tma<false, false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(diag ? k_gossip_tma<true, true> : k_gossip_tma<false, true>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kTmaThreads, smem);
  if (occ < 1) occ = 1;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms * occ;
}

// Tile length (multiple of 32, <= kTmaTileMax) chosen so the number of tiles is
// close to a multiple of the grid: the static round-robin schedule then leaves
// almost no tail imbalance.
int tma_tile_len(int64_t d, int grid) {
  const int64_t nq = (d + kQuantum - 1) / kQuantum;
  const int64_t per_wave = (int64_t)grid * (kTmaTileMax / kQuantum);   // quanta per full wave
  const int64_t waves = (nq + per_wave - 1) / per_wave;
  int64_t q = (nq + (int64_t)grid * waves - 1) / ((int64_t)grid * waves);
  if (q < 1) q = 1;
  if (q > kTmaTileMax / kQuantum) q = kTmaTileMax / kQuantum;
  return (int)(q * kQuantum);
}

cudaError_t launch_gossip_tma(const LocalArgs& a, bool diag, int grid, cudaStream_t st) {
  const size_t smem = tma_smem_bytes(a.n, a.k, diag);
  const bool lars = a.lrs != nullptr;
  if (diag && lars) k_gossip_tma<true, true><<<grid, kTmaThreads, smem, st>>>(a);
  else if (diag) k_gossip_tma<true, false><<<grid, kTmaThreads, smem, st>>>(a);
  else if (lars) k_gossip_tma<false, true><<<grid, kTmaThreads, smem, st>>>(a);
  else k_gossip_tma<false, false><<<grid, kTmaThreads, smem, st>>>(a);
  return cudaGetLastError();
}

// Test/bench input generator (NOT the method): SplitMix64 counter hash of
// synth/__init__.py, v = (z >> 40) * 2^-23 - 1, times `scale`.
__global__ void k_synth(float* out, int64_t rows, int64_t d, int64_t ld, uint64_t seed, int tag,
                        int64_t row0, float scale) {
  const int64_t total = rows * d;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / d, j = e - r * d;
    const uint64_t base = ((uint64_t)tag << 20) + (uint64_t)(row0 + r);
    const uint64_t c = base * (uint64_t)d + (uint64_t)j;
    uint64_t z = seed + (c + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    const float u = __fsub_rn(__fmul_rn((float)(uint32_t)(z >> 40), 1.1920928955078125e-07f), 1.0f);
    out[r * ld + j] = __fmul_rn(u, scale);
  }
}

// ------------------------------------------------------------------ launch ----

namespace {

int g_num_sms = 0;

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_num_sms;
}

// Register-pipeline depth of the flat kernel (rows in flight ahead of the one
// being computed).  CS_LOCAL_PF overrides it for tuning runs.
int pipeline_depth() {
  static int pf = 0;
  if (pf == 0) {
    const char* e = getenv("CS_LOCAL_PF");
    pf = e ? atoi(e) : 2;
    if (pf != 1 && pf != 2 && pf != 3 && pf != 4) pf = 2;
  }
  return pf;
}

template <typename K>
cudaError_t launch_persistent(K kernel, const LocalArgs& a, size_t smem, cudaStream_t st,
                              int* grid_out) {
  cudaError_t e = cudaSuccess;
  if (smem > 48 * 1024) {
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, smem);
  if (e != cudaSuccess) return e;
  if (occ < 1) occ = 1;
  const int64_t nvec = (a.d + 3) / 4;
  const int64_t need = (nvec + kThreads - 1) / kThreads;
  const int64_t cap = (int64_t)num_sms() * occ;
  const int grid = (int)(need < cap ? (need > 0 ? need : 1) : cap);
  kernel<<<grid, kThreads, smem, st>>>(a);
  if (grid_out) *grid_out = grid;
  return cudaGetLastError();
}

template <int PF>
cudaError_t launch_flat_pf(const LocalArgs& a, bool diag, bool fused, size_t smem, cudaStream_t st,
                           int* grid_out) {
  if (fused) {
    if (diag) return launch_persistent(k_gossip_local<PF, true, true>, a, smem, st, grid_out);
    return launch_persistent(k_gossip_local<PF, false, true>, a, smem, st, grid_out);
  }
  if (diag) return launch_persistent(k_gossip_local<PF, true, false>, a, 0, st, grid_out);
  return launch_persistent(k_gossip_local<PF, false, false>, a, 0, st, grid_out);
}

}  // namespace

bool fused_topology_ok(int n, int k) { return n <= kFusedMaxN && (int64_t)n * k <= kFusedMaxKN; }

int local_max_grid() { return num_sms() * 8; }

cudaError_t launch_gossip_local(const LocalArgs& a, bool diag, bool fused, cudaStream_t st,
                                int* grid_out) {
  const size_t smem = fused ? fused_smem_bytes(a.n, a.k, kThreads / 32, diag) : 0;
  switch (pipeline_depth()) {
    case 1: return launch_flat_pf<1>(a, diag, fused, smem, st, grid_out);
    case 3: return launch_flat_pf<3>(a, diag, fused, smem, st, grid_out);
    case 4: return launch_flat_pf<4>(a, diag, fused, smem, st, grid_out);
    default: return launch_flat_pf<2>(a, diag, fused, smem, st, grid_out);
  }
}

cudaError_t launch_hier_local(const LocalArgs& a, bool diag, bool fused, cudaStream_t st,
                              int* grid_out) {
  const bool layers = a.seg_bounds != nullptr || a.lrs != nullptr;  // layer-plan / LARS variant
  const size_t smem = fused ? fused_smem_bytes(a.n, a.k, kThreads / 32, diag) : 0;
  if (fused) {
    if (layers) {
      if (diag) return launch_persistent(k_hier_local<true, true, true>, a, smem, st, grid_out);
      return launch_persistent(k_hier_local<false, true, true>, a, smem, st, grid_out);
    }
    if (diag) return launch_persistent(k_hier_local<true, true, false>, a, smem, st, grid_out);
    return launch_persistent(k_hier_local<false, true, false>, a, smem, st, grid_out);
  }
  if (layers) {
    if (diag) return launch_persistent(k_hier_local<true, false, true>, a, 0, st, grid_out);
    return launch_persistent(k_hier_local<false, false, true>, a, 0, st, grid_out);
  }
  if (diag) return launch_persistent(k_hier_local<true, false, false>, a, 0, st, grid_out);
  return launch_persistent(k_hier_local<false, false, false>, a, 0, st, grid_out);
}

cudaError_t launch_synth(float* out, int64_t rows, int64_t d, int64_t ld, uint64_t seed, int tag,
                         int64_t row0, float scale, cudaStream_t st) {
  const int64_t total = rows * d;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  k_synth<<<(int)blocks, 256, 0, st>>>(out, rows, d, ld, seed, tag, row0, scale);
  return cudaGetLastError();
}

}  // namespace cs
