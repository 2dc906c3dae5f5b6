// Communication-interval mode: the gradient accumulator that
// sits on the caller side of a3.  PAPER.md:209 (§4: "increase the communication
// interval and accumulate the loss during this interval"), Table 1 "Communication
// Interval 42"; the state machine is SPEC accumulate_and_flush:
// accumulator += grad, and at the I-th call emit accumulator / I and reset.
//
// One HBM-bound elementwise pass per micro-step over the bound [n_loc, ld] rows.
// count == 0 writes acc = 0 + g without reading acc (8 B/param); later micro-steps
// read acc and g and write acc (12 B/param).  The last micro-step of an interval
// divides by I in the same pass, so the flush costs no extra traffic and the next
// cs_gossip_step consumes acc unchanged.  Padding columns [d, ld) are never written.
#include "common.cuh"

namespace cs {
namespace {

constexpr int kAccThreads = 256;
constexpr int kAccUnroll = 4;  // float4 per thread in flight: 4 x 2 x 16 B

template <bool FIRST, bool LAST>
__device__ __forceinline__ float acc_one(float a, float g, float fI) {
  // 0 + g (not g): the accumulator starts at +0, so a -0 gradient becomes +0 as in
  // the definition; the division is IEEE round-to-nearest (-prec-div=true).
  float s = FIRST ? 0.0f + g : a + g;
  return LAST ? __fdiv_rn(s, fI) : s;
}

template <bool FIRST, bool LAST, bool PADDED>
__global__ void __launch_bounds__(kAccThreads)
    k_accumulate(float* __restrict__ acc, const float* __restrict__ g, int64_t rows, int64_t d,
                 int64_t ld, float fI) {
  const int64_t q = ld >> 2;
  const int64_t total = rows * q;
  float4* acc4 = reinterpret_cast<float4*>(acc);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  const int64_t stride = (int64_t)gridDim.x * kAccThreads * kAccUnroll;
  for (int64_t base = (int64_t)blockIdx.x * kAccThreads * kAccUnroll + threadIdx.x; base < total;
       base += stride) {
    float4 a[kAccUnroll], b[kAccUnroll];
#pragma unroll
    for (int u = 0; u < kAccUnroll; ++u) {
      const int64_t i = base + (int64_t)u * kAccThreads;
      if (i < total) {
        b[u] = __ldcs(g4 + i);
        if (!FIRST) a[u] = acc4[i];
      }
    }
#pragma unroll
    for (int u = 0; u < kAccUnroll; ++u) {
      const int64_t i = base + (int64_t)u * kAccThreads;
      if (i >= total) continue;
      float4 r;
      r.x = acc_one<FIRST, LAST>(FIRST ? 0.f : a[u].x, b[u].x, fI);
      r.y = acc_one<FIRST, LAST>(FIRST ? 0.f : a[u].y, b[u].y, fI);
      r.z = acc_one<FIRST, LAST>(FIRST ? 0.f : a[u].z, b[u].z, fI);
      r.w = acc_one<FIRST, LAST>(FIRST ? 0.f : a[u].w, b[u].w, fI);
      if (PADDED) {
        const int64_t col = (i % q) * 4;
        if (col + 4 > d) {  // the row's ragged tail: write only columns < d
          float* o = acc + (i / q) * ld + col;
          const float v[4] = {r.x, r.y, r.z, r.w};
          for (int e = 0; e < 4 && col + e < d; ++e) o[e] = v[e];
          continue;
        }
      }
      acc4[i] = r;
    }
  }
}

template <bool FIRST, bool LAST>
cudaError_t launch_acc2(float* acc, const float* g, int64_t rows, int64_t d, int64_t ld, float fI,
                        int grid, cudaStream_t st) {
  if (d == ld)
    k_accumulate<FIRST, LAST, false><<<grid, kAccThreads, 0, st>>>(acc, g, rows, d, ld, fI);
  else
    k_accumulate<FIRST, LAST, true><<<grid, kAccThreads, 0, st>>>(acc, g, rows, d, ld, fI);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_accumulate(float* acc, const float* g, int64_t rows, int64_t d, int64_t ld,
                              int count, int interval, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // 8 resident 256-thread CTAs per SM, fewer for small inputs
  const int64_t per_cta = (int64_t)kAccThreads * kAccUnroll;
  const int64_t need = (rows * (ld >> 2) + per_cta - 1) / per_cta;
  const int grid = (int)(need < (int64_t)sms * 8 ? (need > 0 ? need : 1) : (int64_t)sms * 8);
  const bool first = count == 0, last = count == interval - 1;
  const float fI = (float)interval;
  if (first && last) return launch_acc2<true, true>(acc, g, rows, d, ld, fI, grid, st);
  if (first) return launch_acc2<true, false>(acc, g, rows, d, ld, fI, grid, st);
  if (last) return launch_acc2<false, true>(acc, g, rows, d, ld, fI, grid, st);
  return launch_acc2<false, false>(acc, g, rows, d, ld, fI, grid, st);
}

}  // namespace cs
