// Internal declarations shared by the library's translation units.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace cs {

constexpr int kMaxWorld = 1024;          // == CS_MAX_WORLD
constexpr int kMaxAttempts = 10000;      // Alg. 2 restart cap (reading C-6)
constexpr int kQuantum = 32;             // segment quantum (reading C-2)

// Cycle-order table entries: worker index | flags.  For segment s the table
// lists every worker once, cycle by cycle, each cycle in the order
// c0, c1 = src(c0), c2 = src(c1), ...; so x'_{c_p} = (y_{c_p} + y_{c_{p+1}})/2 and
// the last member of a cycle closes with its first.
constexpr uint32_t kOrdStart = 1u << 30;
constexpr uint32_t kOrdEnd = 1u << 31;
constexpr uint32_t kOrdIdx = (1u << 30) - 1;

// Device error flags (int[3]): [0] topology restart cap hit, [1] non-finite gradient,
// [2] a cross-GPU wait timed out.
enum { kErrTopology = 0, kErrDiverged = 1, kErrTimeout = 2, kNumErr = 3 };

struct TopoArgs {
  uint64_t seed;
  uint32_t step;
  int n;               // ranks in this topology (world, or #leaders)
  int k;
  int tag;
  const int32_t* given;  // device [k][n] injected topology, or nullptr
  int32_t* src;        // out [k][n]   receiver -> sender
  int32_t* dst;        // out [k][n]   sender -> receiver (inverse)
  uint32_t* ord;       // out [k][n]   cycle order (kOrd* flags)
  float* psw;          // in/out [rows][k] push-sum weights (nullptr: skip)
  int group_size;      // rows per topology rank (1 flat, |G| hierarchical)
  double* rw;          // out [k][n] 1 / w'_{rank,s} in fp64 (diagnostics)
  double* inv_wsum;    // out [k] 1 / sum over all rows of w'_{.,s}
  int* err;
};

struct TileDesc;

struct LocalArgs {
  float* x;            // [rows][ld]
  float* m;            // [rows][ld]
  const float* g;      // [rows][ld]
  int64_t ld;
  int64_t d;
  int n;               // ranks of the topology (world, or #leaders when hierarchical)
  int group_size;      // rows per rank: 1 flat, |G| hierarchical
  int k;
  int64_t nq;          // ceil(d / 32)
  // fused topology (prologue builds the tables in shared memory)
  uint64_t seed;
  uint32_t step;
  int tag;
  const int32_t* given;  // injected [k][n] topology (tests) or nullptr
  // precomputed tables (fallback when n > 64 or k*n is large; built by k_topology)
  const uint32_t* ord;
  const double* rw;
  const double* inv_wsum;
  float* psw;          // [rows][k]; fused path mixes it (last CTA), fallback: k_topology did
  float lr, mu, inv_group;
  double* partials;    // [gridDim.x][2]
  double* diag_out;    // [2] {CD, mean checksum}
  unsigned* counter;   // CTA arrival counter (0 between launches)
  int* err;
  // bulk-TMA kernel: segment-aligned column tiles
  const TileDesc* tiles;
  int n_tiles;
  // LARS (k_gossip_tma<., true>): per-(row, layer) rates of this step and the weight decay
  const float* lrs;    // [rows][n_layers]
  int n_layers;
  float wd;
  int wire;            // CS_WIRE_BF16: the received y is rounded to bf16 (reading C-20)
  // k_hier_local with a layer table: the segment plan and the layer bounds (device), or nullptr
  const int64_t* seg_bounds;    // [k+1]
  const int64_t* layer_bounds;  // [n_layers+1]
  // LARS on k_gossip_tma: the step writes sum_j x'^2 per (tile, row) into the .x halves of
  // this double2 [n_tiles][rows] buffer, so the next step's norm pass reads only g
  double* xnorm_out;
  // k_gossip_tma over a piece of the tiles (cs_gossip_step_io): only the step's last piece
  // writes the mixed push-sum weights
  int skip_psw;
  // k_gossip_tma dynamic tile claims (nullptr: static round robin): this launch's counter,
  // 0 at launch; the launch's last CTA zeroes claim_next, the next launch's counter
  unsigned* claim;
  unsigned* claim_next;
};

// bf16 wire format (reading C-20): round to the nearest bf16 (ties to even), widen back.
__device__ __forceinline__ float bf16r(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }
__device__ __forceinline__ float4 bf16r4(float4 v) {
  return make_float4(bf16r(v.x), bf16r(v.y), bf16r(v.z), bf16r(v.w));
}
// 4 values packed as 4 bf16 (8 bytes) and back
__device__ __forceinline__ uint2 pack_bf16x4(float4 v) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
  return make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
}
__device__ __forceinline__ float4 unpack_bf16x4(uint2 u) {
  // a bf16 is the top half of the fp32 with the same value: widening is exact
  return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u),
                     __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xFFFF0000u));
}

// A column tile [c0, c0 + len) inside segment seg and layer `layer` (len <= kTmaTileMax,
// c0 % 4 == 0; c0 % 32 == 0 under the equal split without a layer table).
struct TileDesc {
  int64_t c0;
  int32_t seg;
  int32_t len;
  int32_t layer;
  int32_t pad_;
};

constexpr int kTmaTileMax = 2048;   // elements per row-tile (8 KB per array)

constexpr int kFusedMaxN = 64;      // fused prologue: u64 availability mask
constexpr int kFusedMaxKN = 2048;   // fused prologue: k*n table entries in shared memory

cudaError_t launch_topology(const TopoArgs& a, cudaStream_t st);
int host_alg2(uint64_t seed, uint32_t step, uint32_t seg, int n, int tag, int32_t* src);

bool fused_topology_ok(int n, int k);
cudaError_t launch_gossip_local(const LocalArgs& a, bool diag, bool fused, cudaStream_t st,
                                int* grid_out);
cudaError_t launch_hier_local(const LocalArgs& a, bool diag, bool fused, cudaStream_t st,
                              int* grid_out);
int local_max_grid();
// bulk-TMA single-GPU kernel: grid size, and the balanced tile length for (d, grid)
int tma_grid(int n, int k, bool diag);
int tma_tile_len(int64_t d, int grid);
cudaError_t launch_gossip_tma(const LocalArgs& a, bool diag, int grid, cudaStream_t st);
cudaError_t launch_synth(float* out, int64_t rows, int64_t d, int64_t ld, uint64_t seed,
                         int tag, int64_t row0, float scale, cudaStream_t st);
// LARS (lars.cu): per-(tile, row) fp64 partial sums of x^2, g^2, then per-(row, layer)
// rates lrs = fp32(lr * scale).  tile_first: [n_layers + 1] tile ranges of the layers.
// Optional wait before the norms (hierarchical: the group mean is complete when every
// member's flag flags[first .. first+count) reaches epoch).
struct LarsWait {
  const uint32_t* flags = nullptr;
  int first = 0, count = 0;
  uint32_t epoch = 0;
  int* err = nullptr;
};
cudaError_t launch_lars_rates(const float* x, const float* g, int64_t ld, const TileDesc* tiles,
                              int n_tiles, int rows, const int32_t* tile_first, int n_layers,
                              double* part, float lr, float eta, float wd, float eps, float* lrs,
                              cudaStream_t st, LarsWait w = LarsWait(), bool x_from_carry = false);
// Hierarchical LARS on one GPU: rates per (group, layer) from the leader's x and the group
// mean gbar, formed exactly as k_hier_local forms it (ascending sum, then * inv).
cudaError_t launch_lars_rates_hier(const float* x, const float* g, int64_t ld, const TileDesc* tiles,
                                   int n_tiles, int groups, int gs, float inv, const int32_t* tile_first,
                                   int n_layers, double* part, float lr, float eta, float wd, float eps,
                                   float* lrs, cudaStream_t st);
cudaError_t launch_accumulate(float* acc, const float* g, int64_t rows, int64_t d, int64_t ld,
                              int count, int interval, cudaStream_t st);

}  // namespace cs

namespace cs {
__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
}  // namespace cs
