// Hierarchical h1 through the NVSwitch (NVLS multicast): the intra-group gradient average
// of PAPER.md:197 (§3.3: "reduce the gradients in each group"; reading C-12) as an in-switch
// reduction, the route north_star names for the intra-group average ("NCCL over NVLink ...
// for the intra-group average"; NVLS / multimem).
//
// One worker per GPU, groups of gs GPUs, each group bound to one multicast object (caller-
// provided symmetric memory, cs_set_multicast).  Member c of a group owns the column chunk
// [c*chunk, (c+1)*chunk):
//   B1  every member has its gradient in the multicast-bound buffer (staged by this kernel
//       unless the caller's gradient already lives in a registered multicast region)
//   A   for its chunk: sum = multimem.ld_reduce.add (the switch reads the gs members' words
//       and returns their fp32 sum), gbar = fl(sum * fp32(1/|G|)), multimem.st gbar to every
//       member's gbar (one NVLink write, replicated by the switch)
//   B2  every member finished A: gbar is whole on every member, and no member reads any
//       member's gradient any more (the caller may overwrite it once the step completes)
// The update / leader exchange that follows reads gbar from local HBM.
//
// Per GPU and step: NVLink out d*4 B (its gradient, pulled by the switch, one chunk per
// reducing member) + d/gs*4 B (its mean chunk); NVLink in d/gs*4 B (reduced chunk) + d*4 B
// (every member's mean chunk).  gs = 4, d = 25,557,032: 128 MB each way, against 153 MB each
// way for a reduce-scatter + all-gather over point-to-point links.
//
// Summation order: the switch's, not the oracle's ascending order, so for gs >= 3 results
// match the oracle within the hierarchical tolerance (norm-wise <= 1e-6);
// for gs = 2 the sum of two values is order-free and results stay bitwise.  All members
// receive the same gbar, so the intra-group bitwise equality (P12) is unaffected.
//
// Barriers: each CTA releases its work (fence.acq_rel.sys) and adds to a local arrival
// counter; the CTA completing the count adds 1 to the barrier word of every member with
// one multimem.red.release.sys; every CTA waits (bounded) for gs * epoch.  Words are
// never reset (epoch-tagged, modular comparison).
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "peer.cuh"
#include "ptx.cuh"

namespace cs {

namespace {

constexpr int kNvlsThreads = 512;
constexpr int kNvlsUnroll = 2;   // float4 reductions in flight per thread (4 spilled at 64 registers)

__device__ __forceinline__ float4 mm_ld_reduce4(const float* mc) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(mc)
               : "memory");
  return v;
}
__device__ __forceinline__ float mm_ld_reduce1(const float* mc) {
  float v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(mc) : "memory");
  return v;
}
__device__ __forceinline__ void mm_st4(float* mc, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void mm_st1(float* mc, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mc), "f"(v) : "memory");
}
__device__ __forceinline__ void mm_red_release_add(uint32_t* mc, uint32_t v) {
  asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(mc), "r"(v) : "memory");
}

struct NvlsArgs {
  const float* g;        // this member's gradient (unicast); staged into `stage` if stage != nullptr
  float* stage;          // staging row in the multicast workspace (unicast), or nullptr
  const float* g_mc;     // multicast address of the gradient row every member reduces
  float* gbar_mc;        // multicast address of the group-mean row
  uint32_t* bar_uc;      // barrier words [2] at 64-byte stride (this GPU)
  uint32_t* bar_mc;      // the same words, multicast
  uint32_t* count;       // local arrival counters [2] at 64-byte stride
  int64_t d, chunk;      // columns; columns per member (multiple of 4)
  int member, gs;
  float inv_gs;
  uint32_t epoch;        // barrier b of step e completes at gs * e
  uint32_t target[2];    // running totals of CTAs launched against each counter
  int* err;
  int probe;             // measurement only (CS_NVLS_PROBE): 1 = reduce, plain local store;
                         // 2 = plain local load, multicast store (results not the method's)
};

// grid barrier across the group's GPUs: returns false on timeout
__device__ bool group_barrier(const NvlsArgs& a, int b, int& s_ok) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ptx::fence_acq_rel_sys();
    uint32_t* cnt = a.count + 16 * b;
    const uint32_t prev = atomicAdd(cnt, 1u);
    if (prev + 1 == a.target[b]) {
      ptx::fence_acq_rel_sys();
      mm_red_release_add(a.bar_mc + 16 * b, 1u);
    }
    s_ok = ptx::wait_geq_sys(a.bar_uc + 16 * b, a.epoch * (uint32_t)a.gs) ? 1 : 0;
  }
  __syncthreads();
  return s_ok != 0;
}

__global__ void __launch_bounds__(kNvlsThreads, 2) k_hier_nvls(const NvlsArgs a) {
  __shared__ int s_ok;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a.stage) {  // own gradient into the multicast-bound row
    const int64_t nv = a.d / 4;
    for (int64_t v = tid; v < nv; v += stride)
      __stcg(reinterpret_cast<float4*>(a.stage) + v, __ldcs(reinterpret_cast<const float4*>(a.g) + v));
    for (int64_t j = nv * 4 + tid; j < a.d; j += stride) a.stage[j] = a.g[j];
  }
  bool ok = group_barrier(a, 0, s_ok);
  if (ok) {
    const int64_t c0 = (int64_t)a.member * a.chunk;
    const int64_t c1 = c0 + a.chunk < a.d ? c0 + a.chunk : a.d;
    if (c1 > c0) {
      const int64_t nv = (c1 - c0) / 4;  // whole float4s (c0 is a multiple of 4)
      const float* gp = a.g_mc + c0;
      float* op = a.gbar_mc + c0;
      int64_t v = tid;
      if (a.probe) {  // CS_NVLS_PROBE: time one half of the exchange
        float* lp = a.stage ? a.stage : const_cast<float*>(a.g);
        for (; v < nv; v += stride) {
          const float4 s = a.probe == 1 ? mm_ld_reduce4(gp + 4 * v) : *reinterpret_cast<const float4*>(lp + c0 + 4 * v);
          if (a.probe == 1) *reinterpret_cast<float4*>(lp + c0 + 4 * v) = s;
          else mm_st4(op + 4 * v, s);
        }
        v = nv;
      }
      for (; v + (kNvlsUnroll - 1) * stride < nv; v += kNvlsUnroll * stride) {
        float4 s[kNvlsUnroll];
#pragma unroll
        for (int u = 0; u < kNvlsUnroll; ++u) s[u] = mm_ld_reduce4(gp + 4 * (v + u * stride));
#pragma unroll
        for (int u = 0; u < kNvlsUnroll; ++u) {
          const float4 m = make_float4(__fmul_rn(s[u].x, a.inv_gs), __fmul_rn(s[u].y, a.inv_gs),
                                       __fmul_rn(s[u].z, a.inv_gs), __fmul_rn(s[u].w, a.inv_gs));
          mm_st4(op + 4 * (v + u * stride), m);
        }
      }
      for (; v < nv; v += stride) {
        const float4 s = mm_ld_reduce4(gp + 4 * v);
        mm_st4(op + 4 * v, make_float4(__fmul_rn(s.x, a.inv_gs), __fmul_rn(s.y, a.inv_gs),
                                       __fmul_rn(s.z, a.inv_gs), __fmul_rn(s.w, a.inv_gs)));
      }
      for (int64_t j = c0 + nv * 4 + tid; j < c1; j += stride)  // ragged end of the vector
        mm_st1(a.gbar_mc + j, __fmul_rn(mm_ld_reduce1(a.g_mc + j), a.inv_gs));
    }
  }
  ok = group_barrier(a, 1, s_ok) && ok;
  if (!ok && threadIdx.x == 0) atomicOr(a.err + kErrTimeout, 1);
}

}  // namespace

int nvls_grid() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return 2 * sms;  // 2 x 512 threads per SM: every CTA co-resident (the barriers need it)
}

// Layout of the caller's multicast workspace (cs_multicast_bytes): barrier words and
// arrival counters, then the group-mean row and the staging row, 16-byte aligned.
size_t nvls_off_gbar() { return 4096; }
size_t nvls_off_stage(int64_t ld) { return 4096 + ((size_t)ld * sizeof(float) + 255) / 256 * 256; }
size_t nvls_bytes(int64_t ld) { return nvls_off_stage(ld) + ((size_t)ld * sizeof(float) + 255) / 256 * 256; }

int nvls_h1(PeerState& p, const float* g, const float* g_mc, int member, float inv_gs, int* err, cudaStream_t st) {
  NvlsArgs a;
  char* uc = p.mc_uc;
  char* mc = p.mc_mc;
  a.g = g;
  a.stage = g_mc ? nullptr : reinterpret_cast<float*>(uc + nvls_off_stage(p.ld));
  a.g_mc = g_mc ? g_mc : reinterpret_cast<const float*>(mc + nvls_off_stage(p.ld));
  a.gbar_mc = reinterpret_cast<float*>(mc + nvls_off_gbar());
  a.bar_uc = reinterpret_cast<uint32_t*>(uc);
  a.bar_mc = reinterpret_cast<uint32_t*>(mc);
  a.count = p.d_nvls_count;
  a.d = p.d;
  a.chunk = ((p.d + p.gs - 1) / p.gs + 3) / 4 * 4;
  a.member = member;
  a.gs = p.gs;
  a.inv_gs = inv_gs;
  a.epoch = ++p.nvls_epoch;
  const int grid = nvls_grid();
  a.target[0] = (p.nvls_tot[0] += (uint32_t)grid);
  a.target[1] = (p.nvls_tot[1] += (uint32_t)grid);
  a.err = err;
  static const int probe = getenv("CS_NVLS_PROBE") ? atoi(getenv("CS_NVLS_PROBE")) : 0;
  a.probe = probe;
  ++g_peer_launches;
  k_hier_nvls<<<grid, kNvlsThreads, 0, st>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace cs
