// The method's fp32 arithmetic, one IEEE rounding per operation (no FMA: the library is
// also built with -fmad=false), shared by every kernel so each formula exists once.
//   a3  m' = fl(fl(mu*m) + g)           y = fl(x - fl(lr*m'))       (C-8, C-9)
//   a5  x' = fl(fl(y_i + y_src) * 0.5)                              (Alg.1 l.17; C-10)
//   LARS g + wd*x as fl(g + fl(wd*x))                               (C-18)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cs {

__device__ __forceinline__ float4 mom4(float4 m, float4 g, float mu) {
  return make_float4(__fadd_rn(__fmul_rn(mu, m.x), g.x), __fadd_rn(__fmul_rn(mu, m.y), g.y),
                     __fadd_rn(__fmul_rn(mu, m.z), g.z), __fadd_rn(__fmul_rn(mu, m.w), g.w));
}
__device__ __forceinline__ float4 sgd4(float4 x, float4 m, float lr) {
  return make_float4(__fsub_rn(x.x, __fmul_rn(lr, m.x)), __fsub_rn(x.y, __fmul_rn(lr, m.y)),
                     __fsub_rn(x.z, __fmul_rn(lr, m.z)), __fsub_rn(x.w, __fmul_rn(lr, m.w)));
}
__device__ __forceinline__ float4 decay4(float4 g, float4 x, float wd) {
  return make_float4(__fadd_rn(g.x, __fmul_rn(wd, x.x)), __fadd_rn(g.y, __fmul_rn(wd, x.y)),
                     __fadd_rn(g.z, __fmul_rn(wd, x.z)), __fadd_rn(g.w, __fmul_rn(wd, x.w)));
}
__device__ __forceinline__ float4 mean4(float4 a, float4 b) {
  return make_float4(__fmul_rn(__fadd_rn(a.x, b.x), 0.5f), __fmul_rn(__fadd_rn(a.y, b.y), 0.5f),
                     __fmul_rn(__fadd_rn(a.z, b.z), 0.5f), __fmul_rn(__fadd_rn(a.w, b.w), 0.5f));
}
__device__ __forceinline__ float pair_mean1(float a, float b) { return __fmul_rn(__fadd_rn(a, b), 0.5f); }
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float4 scale4(float4 a, float s) {
  return make_float4(__fmul_rn(a.x, s), __fmul_rn(a.y, s), __fmul_rn(a.z, s), __fmul_rn(a.w, s));
}
// any of the four is Inf or NaN (SPEC.md:382 divergence check)
__device__ __forceinline__ bool nonfinite4(float4 g) {
  const uint32_t e = 0x7f800000u;
  return ((__float_as_uint(g.x) & e) == e) | ((__float_as_uint(g.y) & e) == e) |
         ((__float_as_uint(g.z) & e) == e) | ((__float_as_uint(g.w) & e) == e);
}

}  // namespace cs
