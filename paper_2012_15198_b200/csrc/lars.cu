// LARS per-layer rates.  PAPER.md:35: LARS "adapts the
// learning rate of each layer by the ratio of the weight norm to the gradient norm";
// Table 1: coefficient 0.0025, weight decay 5e-5
// lars_local_lr.  Readings C-18/C-19:
//   scale = eta*|x_l| / ((|g_l| + wd*|x_l|) + eps), 1 if |x_l| == 0 or |g_l| == 0   (fp64)
//   lrs   = fp32(lr * scale)
//
// Two launches before the step kernel:
//   k_lars_norms   one CTA per (tile, row) pair: fp64 sums of x^2 and g^2 over the tile
//                  (fixed warp-shuffle + CTA order) -> part[tile][row]    8 B/param HBM
//   k_lars_scale   one CTA per layer: for each row, folds the layer's tile partials in a
//                  fixed order, then the scale formula -> lrs[row][layer]
// The tiles are the step kernel's layer-split tiles, so a layer's tiles are the
// contiguous range [tile_first[l], tile_first[l+1]).
#include "common.cuh"
#include "ptx.cuh"

namespace cs {
namespace {

constexpr int kNormThreads = 256;

__device__ __forceinline__ double sq(float v) {
  const double d = (double)v;
  return __dmul_rn(d, d);  // exact: a 24-bit significand squared fits in 53 bits
}

// Fixed-order CTA sum of two doubles (warp xor-shuffle tree, then warps in order).
__device__ __forceinline__ double2 block_sum2(double a, double b, double2* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a = __dadd_rn(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = __dadd_rn(b, __shfl_xor_sync(0xffffffffu, b, o));
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = make_double2(a, b);
  __syncthreads();
  double2 r = make_double2(0.0, 0.0);
  if (threadIdx.x == 0) {
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      r.x = __dadd_rn(r.x, red[w].x);
      r.y = __dadd_rn(r.y, red[w].y);
    }
  }
  __syncthreads();
  return r;  // valid in thread 0
}

// DOX = false: the x sums were carried from the previous step (k_gossip_tma wrote the .x
// halves); only g is read and only the .y halves are written.
template <bool DOX>
__global__ void __launch_bounds__(kNormThreads)
    k_lars_norms(const float* __restrict__ x, const float* __restrict__ g, int64_t ld,
                 const TileDesc* __restrict__ tiles, int n_tiles, int rows, double2* __restrict__ part,
                 LarsWait w) {
  __shared__ double2 red[kNormThreads / 32];
  if (w.flags != nullptr) {
    // hierarchical: g is the group mean, complete once every member's all-gather arrived
    __shared__ int s_bad;
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    if ((int)threadIdx.x < w.count) {
      const uint32_t* f = w.flags + w.first + threadIdx.x;
      uint64_t t0 = 0;
      while ((int32_t)(ptx::ld_relaxed_sys(f) - w.epoch) < 0) {
        const uint64_t now = ptx::globaltimer();
        if (t0 == 0) t0 = now;
        if (now - t0 > 20000000000ull) { s_bad = 1; break; }
        __nanosleep(64);
      }
      ptx::fence_acq_rel_sys();
    }
    __syncthreads();
    if (s_bad) {
      if (threadIdx.x == 0) atomicOr(w.err + kErrTimeout, 1);
      return;
    }
  }
  const int64_t pairs = (int64_t)n_tiles * rows;
  for (int64_t p = blockIdx.x; p < pairs; p += gridDim.x) {
    const int u = (int)(p / rows), r = (int)(p % rows);
    const TileDesc td = tiles[u];
    const float* xr = x + (int64_t)r * ld + td.c0;
    const float* gr = g + (int64_t)r * ld + td.c0;
    double sx = 0.0, sg = 0.0;
    for (int v = threadIdx.x; 4 * v < td.len; v += kNormThreads) {
      const float4 a = DOX ? __ldcs(reinterpret_cast<const float4*>(xr) + v) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 b = __ldcs(reinterpret_cast<const float4*>(gr) + v);
      const int valid = td.len - 4 * v;  // the layer's ragged end (len % 4 != 0 only at d)
      sx = __dadd_rn(sx, sq(a.x));
      sg = __dadd_rn(sg, sq(b.x));
      if (valid > 1) { sx = __dadd_rn(sx, sq(a.y)); sg = __dadd_rn(sg, sq(b.y)); }
      if (valid > 2) { sx = __dadd_rn(sx, sq(a.z)); sg = __dadd_rn(sg, sq(b.z)); }
      if (valid > 3) { sx = __dadd_rn(sx, sq(a.w)); sg = __dadd_rn(sg, sq(b.w)); }
    }
    const double2 s = block_sum2(sx, sg, red);
    if (threadIdx.x == 0) {
      if (DOX) part[p] = s;
      else reinterpret_cast<double*>(part)[2 * p + 1] = s.y;  // keep the carried .x
    }
  }
}

__global__ void __launch_bounds__(kNormThreads)
    k_lars_scale(const double2* __restrict__ part, int rows, const int32_t* __restrict__ tile_first,
                 int n_layers, float lr, float eta, float wd, float eps, float* __restrict__ lrs) {
  __shared__ double2 red[kNormThreads / 32];
  const int l = blockIdx.x;
  if (l >= n_layers) return;
  const int t0 = tile_first[l], t1 = tile_first[l + 1];
  for (int r = 0; r < rows; ++r) {
    double sx = 0.0, sg = 0.0;
    for (int u = t0 + (int)threadIdx.x; u < t1; u += kNormThreads) {
      const double2 q = part[(int64_t)u * rows + r];
      sx = __dadd_rn(sx, q.x);
      sg = __dadd_rn(sg, q.y);
    }
    const double2 s = block_sum2(sx, sg, red);
    if (threadIdx.x == 0) {
      const double nw = __dsqrt_rn(s.x), ng = __dsqrt_rn(s.y);
      double scale = 1.0;
      if (nw != 0.0 && ng != 0.0)
        scale = __ddiv_rn(__dmul_rn((double)eta, nw),
                          __dadd_rn(__dadd_rn(ng, __dmul_rn((double)wd, nw)), (double)eps));
      lrs[(int64_t)r * n_layers + l] = __double2float_rn(__dmul_rn((double)lr, scale));
    }
  }
}

// Hierarchical (one GPU): pair p = (tile u, group G); sums of the leader's x^2 and of
// gbar^2 with gbar = fl(sum_{r ascending} g[G*gs + r]) * inv, as k_hier_local forms it.
__global__ void __launch_bounds__(kNormThreads)
    k_lars_norms_hier(const float* __restrict__ x, const float* __restrict__ g, int64_t ld,
                      const TileDesc* __restrict__ tiles, int n_tiles, int groups, int gs, float inv,
                      double2* __restrict__ part) {
  __shared__ double2 red[kNormThreads / 32];
  const int64_t pairs = (int64_t)n_tiles * groups;
  for (int64_t p = blockIdx.x; p < pairs; p += gridDim.x) {
    const int u = (int)(p / groups), G = (int)(p % groups);
    const TileDesc td = tiles[u];
    const float* xr = x + (int64_t)G * gs * ld + td.c0;
    const float* gr = g + (int64_t)G * gs * ld + td.c0;
    double sx = 0.0, sg = 0.0;
    for (int v = threadIdx.x; 4 * v < td.len; v += kNormThreads) {
      const float4 a = __ldcs(reinterpret_cast<const float4*>(xr) + v);
      float4 b = __ldcs(reinterpret_cast<const float4*>(gr) + v);
      for (int r = 1; r < gs; ++r) {
        const float4 c = __ldcs(reinterpret_cast<const float4*>(gr + (int64_t)r * ld) + v);
        b = make_float4(__fadd_rn(b.x, c.x), __fadd_rn(b.y, c.y), __fadd_rn(b.z, c.z), __fadd_rn(b.w, c.w));
      }
      b = make_float4(__fmul_rn(b.x, inv), __fmul_rn(b.y, inv), __fmul_rn(b.z, inv), __fmul_rn(b.w, inv));
      const int valid = td.len - 4 * v;
      sx = __dadd_rn(sx, sq(a.x));
      sg = __dadd_rn(sg, sq(b.x));
      if (valid > 1) { sx = __dadd_rn(sx, sq(a.y)); sg = __dadd_rn(sg, sq(b.y)); }
      if (valid > 2) { sx = __dadd_rn(sx, sq(a.z)); sg = __dadd_rn(sg, sq(b.z)); }
      if (valid > 3) { sx = __dadd_rn(sx, sq(a.w)); sg = __dadd_rn(sg, sq(b.w)); }
    }
    const double2 s = block_sum2(sx, sg, red);
    if (threadIdx.x == 0) part[p] = s;
  }
}

}  // namespace

cudaError_t launch_lars_rates_hier(const float* x, const float* g, int64_t ld, const TileDesc* tiles,
                                   int n_tiles, int groups, int gs, float inv, const int32_t* tile_first,
                                   int n_layers, double* part, float lr, float eta, float wd, float eps,
                                   float* lrs, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t pairs = (int64_t)n_tiles * groups;
  const int grid = (int)(pairs < (int64_t)sms * 8 ? pairs : (int64_t)sms * 8);
  k_lars_norms_hier<<<grid > 0 ? grid : 1, kNormThreads, 0, st>>>(x, g, ld, tiles, n_tiles, groups, gs, inv,
                                                                  reinterpret_cast<double2*>(part));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_lars_scale<<<n_layers, kNormThreads, 0, st>>>(reinterpret_cast<const double2*>(part), groups, tile_first,
                                                  n_layers, lr, eta, wd, eps, lrs);
  return cudaGetLastError();
}

cudaError_t launch_lars_rates(const float* x, const float* g, int64_t ld, const TileDesc* tiles,
                              int n_tiles, int rows, const int32_t* tile_first, int n_layers,
                              double* part, float lr, float eta, float wd, float eps, float* lrs,
                              cudaStream_t st, LarsWait w, bool x_from_carry) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t pairs = (int64_t)n_tiles * rows;
  const int grid = (int)(pairs < (int64_t)sms * 8 ? pairs : (int64_t)sms * 8);
  if (x_from_carry)
    k_lars_norms<false><<<grid > 0 ? grid : 1, kNormThreads, 0, st>>>(x, g, ld, tiles, n_tiles, rows,
                                                                      reinterpret_cast<double2*>(part), w);
  else
    k_lars_norms<true><<<grid > 0 ? grid : 1, kNormThreads, 0, st>>>(x, g, ld, tiles, n_tiles, rows,
                                                                     reinterpret_cast<double2*>(part), w);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_lars_scale<<<n_layers, kNormThreads, 0, st>>>(reinterpret_cast<const double2*>(part), rows,
                                                  tile_first, n_layers, lr, eta, wd, eps, lrs);
  return cudaGetLastError();
}

}  // namespace cs
