// Single-GPU hot path: every worker co-resident in this GPU's HBM (configs 1, 2;
// the paper itself ran "multiple processes for each GPU").
//
// k_gossip_local fuses, per float4 column (4 consecutive parameters), for all n
// workers:
//   a3  m_i <- fl(fl(mu*m_i) + g_i);  y_i <- fl(x_i - fl(lr*m_i))   (C-8, C-9)
//   a4  receive y_{src_s(i)} — here an HBM row already in flight in this thread
//   a5  x_i <- fl(fl(y_i + y_{src_s(i)}) * 0.5)                    (Alg.1 l.17)
//   a6  (DIAG) fp64 shifted sums of z = x'/w' per column -> per-block partials
//
// Column-owner cycle walk: the thread that owns column j visits the workers of
// segment s(j) in the cycle order of src_s (k_topology), so y_{c_p} and
// y_{c_{p+1}} = y_{src(c_p)} are both in registers when x'_{c_p} is written and
// each of x, m, g is read exactly once and x, m written exactly once: the
// algorithmic 20 B per parameter per worker, in place, with no ping-pong buffer
// (every element is read by its owner before its owner writes it).
// Loads of the next PF workers' rows are issued before the current row's
// arithmetic (explicit register pipeline) to keep enough bytes in flight.
//
// All fp32 arithmetic uses __fmul_rn/__fadd_rn/__fsub_rn: never contracted to
// FMA, so results are bit-identical to the oracle's separately rounded ops.
#include "common.cuh"

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

__device__ __forceinline__ float4 momentum_update(float4 m, float4 g, float mu) {
  return make_float4(__fadd_rn(__fmul_rn(mu, m.x), g.x), __fadd_rn(__fmul_rn(mu, m.y), g.y),
                     __fadd_rn(__fmul_rn(mu, m.z), g.z), __fadd_rn(__fmul_rn(mu, m.w), g.w));
}

__device__ __forceinline__ float4 sgd_apply(float4 x, float4 m, float lr) {
  return make_float4(__fsub_rn(x.x, __fmul_rn(lr, m.x)), __fsub_rn(x.y, __fmul_rn(lr, m.y)),
                     __fsub_rn(x.z, __fmul_rn(lr, m.z)), __fsub_rn(x.w, __fmul_rn(lr, m.w)));
}

__device__ __forceinline__ float4 pair_mean(float4 a, float4 b) {
  return make_float4(__fmul_rn(__fadd_rn(a.x, b.x), 0.5f), __fmul_rn(__fadd_rn(a.y, b.y), 0.5f),
                     __fmul_rn(__fadd_rn(a.z, b.z), 0.5f), __fmul_rn(__fadd_rn(a.w, b.w), 0.5f));
}

__device__ __forceinline__ bool nonfinite4(float4 g) {
  const uint32_t e = 0x7f800000u;
  return ((__float_as_uint(g.x) & e) == e) | ((__float_as_uint(g.y) & e) == e) |
         ((__float_as_uint(g.z) & e) == e) | ((__float_as_uint(g.w) & e) == e);
}

// Per-column fp64 accumulators for the consensus diagnostics: shifted by the
// first value c seen in the column so S2 - ... does not cancel near consensus.
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
  // column j's contribution: sum_i (z_ij - zbar_j)^2 and zbar_j
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

}  // namespace

constexpr int kThreads = 256;
constexpr int kPF = 2;  // rows in flight ahead of the one being computed

template <bool DIAG>
__global__ void __launch_bounds__(kThreads) k_gossip_local(const LocalArgs a) {
  const int n = a.n;
  const int64_t ld = a.ld, d = a.d;
  const int64_t nvec = (d + 3) >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const float mu = a.mu, lr = a.lr;
  double dacc = 0.0, zacc = 0.0;
  bool bad = false;

  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += stride) {
    const int64_t j = v << 2;
    const int valid = (int)imin64(4, d - j);
    // segment of column j (reading C-2): largest s with 32*floor(s*nq/k) <= j
    const int64_t q = j >> 5;
    const int s = (int)imin64(a.k - 1, ((q + 1) * a.k - 1) / a.nq);
    const uint32_t* ord = a.ord + (int64_t)s * n;
    const double* rw = DIAG ? a.rw + (int64_t)s * n : nullptr;

    float4 bx[kPF], bm[kPF], bg[kPF];
    uint32_t be[kPF];
#pragma unroll
    for (int t = 0; t < kPF; ++t) {
      if (t < n) {
        be[t] = __ldg(ord + t);
        const int64_t off = (int64_t)(be[t] & kOrdIdx) * ld + j;
        bx[t] = ld_stream(a.x + off);
        bm[t] = ld_stream(a.m + off);
        bg[t] = ld_stream(a.g + off);
      }
    }
    float4 yfirst = make_float4(0.f, 0.f, 0.f, 0.f), yprev = yfirst;
    int64_t prev_off = 0;
    uint32_t prev_row = 0;
    ColDiag cd;
    if (DIAG) cd.reset();
    bool first_diag = true;

    for (int p0 = 0; p0 < n; p0 += kPF) {
#pragma unroll
      for (int t = 0; t < kPF; ++t) {
        const int p = p0 + t;
        if (p < n) {
          const float4 cx = bx[t], cm = bm[t], cg = bg[t];
          const uint32_t e = be[t];
          if (p + kPF < n) {  // refill this slot with the row kPF ahead
            be[t] = __ldg(ord + p + kPF);
            const int64_t off2 = (int64_t)(be[t] & kOrdIdx) * ld + j;
            bx[t] = ld_stream(a.x + off2);
            bm[t] = ld_stream(a.m + off2);
            bg[t] = ld_stream(a.g + off2);
          }
          const uint32_t row = e & kOrdIdx;
          const int64_t off = (int64_t)row * ld + j;
          bad |= nonfinite4(cg);
          const float4 mn = momentum_update(cm, cg, mu);
          const float4 y = sgd_apply(cx, mn, lr);
          st_stream(a.m + off, mn, valid);
          if (e & kOrdStart) {
            yfirst = y;
          } else {
            const float4 xo = pair_mean(yprev, y);
            st_stream(a.x + prev_off, xo, valid);
            if (DIAG) { cd.add(xo, rw[prev_row], first_diag, 1.0); first_diag = false; }
          }
          if (e & kOrdEnd) {
            const float4 xo = pair_mean(y, yfirst);
            st_stream(a.x + off, xo, valid);
            if (DIAG) { cd.add(xo, rw[row], first_diag, 1.0); first_diag = false; }
          }
          yprev = y;
          prev_off = off;
          prev_row = row;
        }
      }
    }
    if (DIAG) cd.finish(a.inv_wsum[s], (double)n, valid, dacc, zacc);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(a.err + kErrDiverged, 1);
  if (DIAG) block_reduce_store(dacc, zacc, a.partials);
}

// Hierarchical step with every worker co-resident (§3.3):
//   h1  gbar_G = fl(sum over members, ascending) * fp32(1/|G|)
//   h2  leader: m <- mu*m + gbar, y <- x - lr*m; then the cycle walk over the
//       leader topology mixes leaders' y (tag HIER); one leader: x' = y
//   h3  x' written to every member row of the group (bitwise identical)
template <bool DIAG>
__global__ void __launch_bounds__(kThreads) k_hier_local(const LocalArgs a) {
  const int L = a.n, gs = a.group_size;
  const int64_t ld = a.ld, d = a.d;
  const int64_t nvec = (d + 3) >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const float mu = a.mu, lr = a.lr, inv = a.inv_group;
  double dacc = 0.0, zacc = 0.0;
  bool bad = false;

  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += stride) {
    const int64_t j = v << 2;
    const int valid = (int)imin64(4, d - j);
    const int64_t q = j >> 5;
    const int s = (int)imin64(a.k - 1, ((q + 1) * a.k - 1) / a.nq);
    const uint32_t* ord = a.ord + (int64_t)s * L;
    const double* rw = DIAG ? a.rw + (int64_t)s * L : nullptr;
    float4 yfirst = make_float4(0.f, 0.f, 0.f, 0.f), yprev = yfirst;
    uint32_t prev_leader = 0;
    ColDiag cd;
    if (DIAG) cd.reset();
    bool first_diag = true;

    for (int p = 0; p < L; ++p) {
      const uint32_t e = __ldg(ord + p);
      const uint32_t G = e & kOrdIdx;
      const int64_t lead_off = (int64_t)G * gs * ld + j;
      const float4 cx = ld_stream(a.x + lead_off);
      const float4 cm = ld_stream(a.m + lead_off);
      float4 gsum = ld_stream(a.g + lead_off);
      bad |= nonfinite4(gsum);
      for (int r = 1; r < gs; ++r) {
        const float4 gr = ld_stream(a.g + lead_off + (int64_t)r * ld);
        bad |= nonfinite4(gr);
        gsum = make_float4(__fadd_rn(gsum.x, gr.x), __fadd_rn(gsum.y, gr.y),
                           __fadd_rn(gsum.z, gr.z), __fadd_rn(gsum.w, gr.w));
      }
      const float4 gbar = make_float4(__fmul_rn(gsum.x, inv), __fmul_rn(gsum.y, inv),
                                      __fmul_rn(gsum.z, inv), __fmul_rn(gsum.w, inv));
      const float4 mn = momentum_update(cm, gbar, mu);
      const float4 y = sgd_apply(cx, mn, lr);
      st_stream(a.m + lead_off, mn, valid);
      if (L == 1) {
        for (int r = 0; r < gs; ++r) st_stream(a.x + lead_off + (int64_t)r * ld, y, valid);
        if (DIAG) { cd.add(y, rw[G], true, (double)gs); }
        continue;
      }
      if (e & kOrdStart) {
        yfirst = y;
      } else {
        const float4 xo = pair_mean(yprev, y);
        const int64_t po = (int64_t)prev_leader * gs * ld + j;
        for (int r = 0; r < gs; ++r) st_stream(a.x + po + (int64_t)r * ld, xo, valid);
        if (DIAG) { cd.add(xo, rw[prev_leader], first_diag, (double)gs); first_diag = false; }
      }
      if (e & kOrdEnd) {
        const float4 xo = pair_mean(y, yfirst);
        for (int r = 0; r < gs; ++r) st_stream(a.x + lead_off + (int64_t)r * ld, xo, valid);
        if (DIAG) { cd.add(xo, rw[G], first_diag, (double)gs); first_diag = false; }
      }
      yprev = y;
      prev_leader = G;
    }
    if (DIAG) cd.finish(a.inv_wsum[s], (double)L * gs, valid, dacc, zacc);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(a.err + kErrDiverged, 1);
  if (DIAG) block_reduce_store(dacc, zacc, a.partials);
}

// Fixed-order reduction of the per-block partials -> {CD, mean checksum}.
__global__ void __launch_bounds__(256) k_diag_finalize(const double* partials, int nparts, int n,
                                                       double* out) {
  __shared__ double sa[256], sb[256];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
    a += partials[2 * i];
    b += partials[2 * i + 1];
  }
  sa[threadIdx.x] = a;
  sb[threadIdx.x] = b;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      sa[threadIdx.x] += sa[threadIdx.x + w];
      sb[threadIdx.x] += sb[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = sqrt(fmax(sa[0], 0.0) / (double)n);
    out[1] = sb[0];
  }
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

static int g_num_sms = 0;
static int g_occ[2][2] = {{0, 0}, {0, 0}};

int local_grid_size(bool hier, bool diag, int64_t d) {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_occ[0][0], k_gossip_local<false>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_occ[0][1], k_gossip_local<true>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_occ[1][0], k_hier_local<false>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_occ[1][1], k_hier_local<true>, kThreads, 0);
  }
  const int64_t nvec = (d + 3) / 4;
  const int64_t need = (nvec + kThreads - 1) / kThreads;
  int64_t cap = (int64_t)g_num_sms * (g_occ[hier][diag] > 0 ? g_occ[hier][diag] : 1);
  return (int)(need < cap ? (need > 0 ? need : 1) : cap);
}

cudaError_t launch_gossip_local(const LocalArgs& a, bool diag, int grid, cudaStream_t st) {
  if (diag) k_gossip_local<true><<<grid, kThreads, 0, st>>>(a);
  else k_gossip_local<false><<<grid, kThreads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_hier_local(const LocalArgs& a, bool diag, int grid, cudaStream_t st) {
  if (diag) k_hier_local<true><<<grid, kThreads, 0, st>>>(a);
  else k_hier_local<false><<<grid, kThreads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_diag_finalize(const double* partials, int nparts, int n, double* out,
                                 cudaStream_t st) {
  k_diag_finalize<<<1, 256, 0, st>>>(partials, nparts, n, out);
  return cudaGetLastError();
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
