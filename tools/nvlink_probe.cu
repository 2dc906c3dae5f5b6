// NVLink peer-bandwidth probe (tuning tool, not part of the library).
// One process drives GPUs 0 and 1 with peer access enabled and measures, for a
// 256 MiB buffer, the bandwidth of: 128-bit stores into the peer (push),
// 128-bit loads from the peer (pull), 1-D bulk-TMA copies shared->peer and
// peer->shared, each one-way (GPU0 only) and two-way (both GPUs at once), plus
// cudaMemcpyPeerAsync.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvlink_probe nvlink_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                \
    }                                                                          \
  } while (0)

__global__ void k_store(float4* __restrict__ dst, int64_t n4, int unroll) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) dst[i] = v;
}

__global__ void k_load(const float4* __restrict__ src, int64_t n4, float* sink) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  float acc = 0.f;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {
    float4 a = __ldcg(src + i), b = __ldcg(src + i + stride), c = __ldcg(src + i + 2 * stride),
           d = __ldcg(src + i + 3 * stride);
    acc += a.x + b.y + c.z + d.w;
  }
  for (; i < n4; i += stride) acc += __ldcg(src + i).x;
  if (acc == 123.456f) *sink = acc;
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// each CTA moves chunks of `chunk` bytes with bulk copies (one elected thread), double-buffered
__global__ void k_bulk_s2g(char* dst, int64_t bytes, int chunk) {
  extern __shared__ __align__(128) char sm[];
  if (threadIdx.x != 0) return;
  const int64_t nch = bytes / chunk;
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * chunk), "r"(sa(sm)),
                 "r"(chunk)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void k_bulk_g2s(const char* src, int64_t bytes, int chunk, int stages) {
  extern __shared__ __align__(128) char sm[];
  __shared__ uint64_t bar[8];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t nch = bytes / chunk;
  int64_t it = 0;
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x, ++it) {
    const int s = (int)(it % stages);
    if (it >= stages) {  // wait for the previous use of this stage
      const uint32_t par = (uint32_t)(((it / stages) - 1) & 1);
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                     : "=r"(done)
                     : "r"(sa(&bar[s])), "r"(par)
                     : "memory");
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sa(sm + (size_t)s * chunk)),
                 "l"(src + c * chunk), "r"(chunk), "r"(sa(&bar[s]))
                 : "memory");
  }
  for (int64_t k = it > stages ? it - stages : 0; k < it; ++k) {
    const int s = (int)(k % stages);
    const uint32_t par = (uint32_t)((k / stages) & 1);
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                   : "=r"(done)
                   : "r"(sa(&bar[s])), "r"(par)
                   : "memory");
  }
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    printf("need 2 GPUs\n");
    return 0;
  }
  const int64_t bytes = 256ll << 20;
  const int64_t n4 = bytes / 16;
  float4* buf[2];
  float* sink[2];
  cudaStream_t st[2];
  cudaEvent_t e0[2], e1[2];
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceEnablePeerAccess(1 - g, 0));
    CK(cudaMalloc(&buf[g], bytes));
    CK(cudaMalloc(&sink[g], 4));
    CK(cudaMemset(buf[g], 0, bytes));
    CK(cudaStreamCreate(&st[g]));
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
    CK(cudaFuncSetAttribute(k_bulk_s2g, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_bulk_g2s, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  }
  auto run = [&](const char* name, int kind, int two_way, int grid_mult, int block, int chunk) -> int {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      for (int g = 0; g < (two_way ? 2 : 1); ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventRecord(e0[g], st[g]));
        float4* peer = buf[1 - g];
        float4* own = buf[g];
        (void)own;
        const int grid = sms * grid_mult;
        if (kind == 0) k_store<<<grid, block, 0, st[g]>>>(peer, n4, 1);
        if (kind == 1) k_load<<<grid, block, 0, st[g]>>>(peer, n4, sink[g]);
        if (kind == 2) k_bulk_s2g<<<grid, 32, chunk, st[g]>>>((char*)peer, bytes, chunk);
        if (kind == 3) k_bulk_g2s<<<grid, 32, chunk * 4, st[g]>>>((const char*)peer, bytes, chunk, 4);
        if (kind == 4) CK(cudaMemcpyPeerAsync(own, g, peer, 1 - g, bytes, st[g]));
        CK(cudaEventRecord(e1[g], st[g]));
      }
      float worst = 0.f;
      for (int g = 0; g < (two_way ? 2 : 1); ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventSynchronize(e1[g]));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
        if (ms > worst) worst = ms;
      }
      if (rep > 0 && worst < best) best = worst;
    }
    printf("%-40s %s  grid=%3dx%d block=%4d chunk=%6d : %8.1f GB/s per direction\n", name, two_way ? "2-way" : "1-way",
           sms, grid_mult, block, chunk, bytes / (best * 1e-3) / 1e9);
    return 0;
  };
  for (int tw = 0; tw < 2; ++tw) {
    run("st.v4 push to peer", 0, tw, 8, 256, 0);
    run("st.v4 push to peer", 0, tw, 2, 512, 0);
    run("ld.v4 pull from peer", 1, tw, 8, 256, 0);
    run("ld.v4 pull from peer", 1, tw, 4, 512, 0);
    run("bulk s2g push to peer", 2, tw, 1, 32, 16384);
    run("bulk s2g push to peer", 2, tw, 4, 32, 16384);
    run("bulk s2g push to peer", 2, tw, 4, 32, 65536);
    run("bulk g2s pull from peer", 3, tw, 1, 32, 16384);
    run("bulk g2s pull from peer", 3, tw, 2, 32, 32768);
    run("cudaMemcpyPeerAsync", 4, tw, 1, 0, 0);
  }
  return 0;
}
