// LARS per-layer rates.  PAPER.md:35: LARS "adapts the
// learning rate of each layer by the ratio of the weight norm to the gradient norm";
// Table 1: coefficient 0.0025, weight decay 5e-5
// lars_local_lr.  Readings C-18/C-19:
//   scale = eta*|x_l| / ((|g_l| + wd*|x_l|) + eps), 1 if |x_l| == 0 or |g_l| == 0   (fp64)
//   lrs   = fp32(lr * scale)
//
// Two launches before the step kernel:
//   k_lars_norms   one warp per (tile, row) pair: fp64 sums of x^2 and g^2 over the tile
//                  (fixed lane + warp-shuffle order) -> part[tile][row]    8 B/param HBM
//                  (4 B/param when the step kernel carried the x sums)
//   k_lars_scale   one warp per (layer, row): folds the layer's tile partials in a
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

// One warp per (tile, row) pair: each lane keeps kNormVec float4 loads in flight (of g,
// or half of x and half of g), sums its squares in fp64 in a fixed order (its float4s in
// index order, then the x/y/z/w lanes), and the warp folds the 32 partials with a fixed
// xor-shuffle tree -- no CTA barrier per pair.  A tile is at most kTmaTileMax = 2048
// columns = 512 float4, so a pair is at most two rounds (four with x).
// DOX = false: the x sums were carried from the previous step (k_gossip_tma wrote the .x
// halves); only g is read and only the .y halves are written.
constexpr int kNormVec = 8;

template <bool DOX>
__global__ void __launch_bounds__(kNormThreads)
    k_lars_norms(const float* __restrict__ x, const float* __restrict__ g, int64_t ld,
                 const TileDesc* __restrict__ tiles, int n_tiles, int rows, double2* __restrict__ part,
                 LarsWait w) {
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
  const int lane = threadIdx.x & 31;
  const int64_t pairs = (int64_t)n_tiles * rows;
  const int64_t nwarps = (int64_t)gridDim.x * (kNormThreads / 32);
  for (int64_t p = (int64_t)blockIdx.x * (kNormThreads / 32) + (threadIdx.x >> 5); p < pairs; p += nwarps) {
    const int u = (int)(p / rows), r = (int)(p % rows);
    const TileDesc td = tiles[u];
    const float4* xr = reinterpret_cast<const float4*>(x + (int64_t)r * ld + td.c0);
    const float4* gr = reinterpret_cast<const float4*>(g + (int64_t)r * ld + td.c0);
    const int nv = (td.len + 3) >> 2;
    double sx = 0.0, sg = 0.0;
    constexpr int V = DOX ? kNormVec / 2 : kNormVec;
    for (int v0 = 0; v0 < nv; v0 += 32 * V) {
      float4 a[V], b[V];
#pragma unroll
      for (int c = 0; c < V; ++c) {
        const int v = v0 + c * 32 + lane;
        a[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        b[c] = a[c];
        if (v < nv) {
          if (DOX) a[c] = __ldcs(xr + v);
          b[c] = __ldcs(gr + v);
        }
      }
#pragma unroll
      for (int c = 0; c < V; ++c) {
        const int valid = td.len - 4 * (v0 + c * 32 + lane);  // ragged end only at d
        if (valid <= 0) continue;
        if (DOX) sx = __dadd_rn(sx, sq(a[c].x));
        sg = __dadd_rn(sg, sq(b[c].x));
        if (valid > 1) { if (DOX) sx = __dadd_rn(sx, sq(a[c].y)); sg = __dadd_rn(sg, sq(b[c].y)); }
        if (valid > 2) { if (DOX) sx = __dadd_rn(sx, sq(a[c].z)); sg = __dadd_rn(sg, sq(b[c].z)); }
        if (valid > 3) { if (DOX) sx = __dadd_rn(sx, sq(a[c].w)); sg = __dadd_rn(sg, sq(b[c].w)); }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      if (DOX) sx = __dadd_rn(sx, __shfl_xor_sync(0xffffffffu, sx, o));
      sg = __dadd_rn(sg, __shfl_xor_sync(0xffffffffu, sg, o));
    }
    if (lane == 0) {
      if (DOX) part[p] = make_double2(sx, sg);
      else reinterpret_cast<double*>(part)[2 * p + 1] = sg;  // keep the carried .x
    }
  }
}

// One warp per (layer, row): lane i folds tiles t0+i, t0+i+32, ... in that order, then a
// fixed xor-shuffle tree; lane 0 applies the scale formula.
__global__ void __launch_bounds__(kNormThreads)
    k_lars_scale(const double2* __restrict__ part, int rows, const int32_t* __restrict__ tile_first,
                 int n_layers, float lr, float eta, float wd, float eps, float* __restrict__ lrs) {
  const int lane = threadIdx.x & 31;
  const int64_t q = (int64_t)blockIdx.x * (kNormThreads / 32) + (threadIdx.x >> 5);
  if (q >= (int64_t)n_layers * rows) return;
  const int l = (int)(q / rows), r = (int)(q % rows);
  const int t0 = tile_first[l], t1 = tile_first[l + 1];
  double sx = 0.0, sg = 0.0;
  // the largest layer spans ~1200 tiles: issue 4 L2 loads before adding them (in order)
  for (int u0 = t0 + lane; u0 < t1; u0 += 4 * 32) {
    double2 v[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int u = u0 + 32 * c;
      v[c] = u < t1 ? part[(int64_t)u * rows + r] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (u0 + 32 * c >= t1) break;
      sx = __dadd_rn(sx, v[c].x);
      sg = __dadd_rn(sg, v[c].y);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sx = __dadd_rn(sx, __shfl_xor_sync(0xffffffffu, sx, o));
    sg = __dadd_rn(sg, __shfl_xor_sync(0xffffffffu, sg, o));
  }
  if (lane == 0) {
    const double nw = __dsqrt_rn(sx), ng = __dsqrt_rn(sg);
    double scale = 1.0;
    if (nw != 0.0 && ng != 0.0)
      scale = __ddiv_rn(__dmul_rn((double)eta, nw),
                        __dadd_rn(__dadd_rn(ng, __dmul_rn((double)wd, nw)), (double)eps));
    lrs[(int64_t)r * n_layers + l] = __double2float_rn(__dmul_rn((double)lr, scale));
  }
}

// Hierarchical (one GPU): pair p = (tile u, group G), one warp per pair as above; sums of
// the leader's x^2 and of gbar^2 with gbar = fl(sum_{r ascending} g[G*gs + r]) * inv, as
// k_hier_local forms it.
__global__ void __launch_bounds__(kNormThreads)
    k_lars_norms_hier(const float* __restrict__ x, const float* __restrict__ g, int64_t ld,
                      const TileDesc* __restrict__ tiles, int n_tiles, int groups, int gs, float inv,
                      double2* __restrict__ part) {
  constexpr int V = kNormVec / 2;
  const int lane = threadIdx.x & 31;
  const int64_t pairs = (int64_t)n_tiles * groups;
  const int64_t nwarps = (int64_t)gridDim.x * (kNormThreads / 32);
  for (int64_t p = (int64_t)blockIdx.x * (kNormThreads / 32) + (threadIdx.x >> 5); p < pairs; p += nwarps) {
    const int u = (int)(p / groups), G = (int)(p % groups);
    const TileDesc td = tiles[u];
    const float4* xr = reinterpret_cast<const float4*>(x + (int64_t)G * gs * ld + td.c0);
    const float* gr = g + (int64_t)G * gs * ld + td.c0;
    const int nv = (td.len + 3) >> 2;
    double sx = 0.0, sg = 0.0;
    for (int v0 = 0; v0 < nv; v0 += 32 * V) {
      float4 a[V], b[V];
#pragma unroll
      for (int c = 0; c < V; ++c) {
        const int v = v0 + c * 32 + lane;
        a[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        b[c] = a[c];
        if (v < nv) {
          a[c] = __ldcs(xr + v);
          b[c] = __ldcs(reinterpret_cast<const float4*>(gr) + v);
        }
      }
      for (int r = 1; r < gs; ++r) {
#pragma unroll
        for (int c = 0; c < V; ++c) {
          const int v = v0 + c * 32 + lane;
          if (v < nv) {
            const float4 e = __ldcs(reinterpret_cast<const float4*>(gr + (int64_t)r * ld) + v);
            b[c] = make_float4(__fadd_rn(b[c].x, e.x), __fadd_rn(b[c].y, e.y), __fadd_rn(b[c].z, e.z),
                               __fadd_rn(b[c].w, e.w));
          }
        }
      }
#pragma unroll
      for (int c = 0; c < V; ++c) {
        const int valid = td.len - 4 * (v0 + c * 32 + lane);
        if (valid <= 0) continue;
        const float4 m = make_float4(__fmul_rn(b[c].x, inv), __fmul_rn(b[c].y, inv), __fmul_rn(b[c].z, inv),
                                     __fmul_rn(b[c].w, inv));
        sx = __dadd_rn(sx, sq(a[c].x));
        sg = __dadd_rn(sg, sq(m.x));
        if (valid > 1) { sx = __dadd_rn(sx, sq(a[c].y)); sg = __dadd_rn(sg, sq(m.y)); }
        if (valid > 2) { sx = __dadd_rn(sx, sq(a[c].z)); sg = __dadd_rn(sg, sq(m.z)); }
        if (valid > 3) { sx = __dadd_rn(sx, sq(a[c].w)); sg = __dadd_rn(sg, sq(m.w)); }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sx = __dadd_rn(sx, __shfl_xor_sync(0xffffffffu, sx, o));
      sg = __dadd_rn(sg, __shfl_xor_sync(0xffffffffu, sg, o));
    }
    if (lane == 0) part[p] = make_double2(sx, sg);
  }
}

int scale_grid(int n_layers, int rows) {
  return (int)(((int64_t)n_layers * rows + kNormThreads / 32 - 1) / (kNormThreads / 32));
}

}  // namespace

cudaError_t launch_lars_rates_hier(const float* x, const float* g, int64_t ld, const TileDesc* tiles,
                                   int n_tiles, int groups, int gs, float inv, const int32_t* tile_first,
                                   int n_layers, double* part, float lr, float eta, float wd, float eps,
                                   float* lrs, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t pairs = (int64_t)n_tiles * groups;  // one warp per pair
  const int64_t ctas = (pairs + kNormThreads / 32 - 1) / (kNormThreads / 32);
  const int grid = (int)(ctas < (int64_t)sms * 8 ? ctas : (int64_t)sms * 8);
  k_lars_norms_hier<<<grid > 0 ? grid : 1, kNormThreads, 0, st>>>(x, g, ld, tiles, n_tiles, groups, gs, inv,
                                                                  reinterpret_cast<double2*>(part));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_lars_scale<<<scale_grid(n_layers, groups), kNormThreads, 0, st>>>(reinterpret_cast<const double2*>(part), groups, tile_first,
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
  const int64_t pairs = (int64_t)n_tiles * rows;  // one warp per pair
  const int64_t ctas = (pairs + kNormThreads / 32 - 1) / (kNormThreads / 32);
  const int grid = (int)(ctas < (int64_t)sms * 8 ? ctas : (int64_t)sms * 8);
  if (x_from_carry)
    k_lars_norms<false><<<grid > 0 ? grid : 1, kNormThreads, 0, st>>>(x, g, ld, tiles, n_tiles, rows,
                                                                      reinterpret_cast<double2*>(part), w);
  else
    k_lars_norms<true><<<grid > 0 ? grid : 1, kNormThreads, 0, st>>>(x, g, ld, tiles, n_tiles, rows,
                                                                     reinterpret_cast<double2*>(part), w);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_lars_scale<<<scale_grid(n_layers, rows), kNormThreads, 0, st>>>(reinterpret_cast<const double2*>(part), rows,
                                                  tile_first, n_layers, lr, eta, wd, eps, lrs);
  return cudaGetLastError();
}

}  // namespace cs
