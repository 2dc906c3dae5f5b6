// C ABI (include/crossover_sgd.h): process-wide context, argument validation,
// device tables and kernel launches.  No compute happens on the host except the
// (pure, cheap) host topology of cs_topology / byte accounting.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/crossover_sgd.h"
#include "common.cuh"
#include "peer.cuh"

using namespace cs;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(CS_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CS_CUDA(call)                                  \
  do {                                                 \
    cudaError_t _e = (call);                           \
    if (_e != cudaSuccess) return cuda_fail(_e, #call); \
  } while (0)

struct Ctx {
  bool inited = false;
  int world = 0, groups = 0, k = 0;
  uint64_t seed = 0;

  bool bound = false;
  int64_t d = 0, ld = 0, nq = 0;
  int rank = 0, nprocs = 1, n_loc = 0, first = 0;
  float* mom = nullptr;
  cudaStream_t stream = nullptr;
  int device = 0;

  int64_t step = 0;
  int diag = 0;
  bool diag_valid = false;

  // device tables
  int64_t* d_bounds = nullptr;
  int32_t* d_src = nullptr;
  int32_t* d_dst = nullptr;
  uint32_t* d_ord = nullptr;
  int32_t* d_given = nullptr;
  double* d_rw = nullptr;
  double* d_inv_wsum = nullptr;
  int* d_err = nullptr;
  double* d_partials = nullptr;   // [local_max_grid()][2]
  double* d_diag = nullptr;
  unsigned* d_counter = nullptr;  // CTA arrival counter of the fused kernels
  int launches_per_step = 0;
  const char* hot_kernel = "";

  // bulk-TMA single-GPU kernel (n <= 64): balanced segment-aligned tiles
  int path = CS_PATH_AUTO;     // requested by cs_set_path (applies at the next cs_bind)
  bool use_tma = false;
  bool use_peer = false;
  TileDesc* d_tiles = nullptr;
  int n_tiles = 0;
  int tma_grid_plain = 0, tma_grid_diag = 0;
  // k_gossip_tma claims tiles dynamically (CS_TMA_DYNAMIC=0: static round robin); the
  // launch sequence number picks the claim counter (two, alternating by launch)
  bool tma_dynamic = true;
  unsigned claim_seq = 0;
  bool has_override = false;

  float* d_stage = nullptr;   // cs_gossip_step_host staging buffer
  size_t stage_bytes = 0;
  // cs_gossip_step_io: host copies of the bulk-TMA tiles' columns, copy streams and events
  std::vector<int64_t> h_tile_c0, h_tile_end;
  cudaStream_t io_h2d = nullptr, io_d2h = nullptr;
  std::vector<cudaEvent_t> io_ev;

  PeerState peer;             // multi-GPU exchange region (nprocs > 1)

  // layer table (cs_set_layers) and LARS (cs_set_lars); the layer table is per cs_bind
  std::vector<int64_t> layer_bounds;  // [n_layers + 1]; empty: no table
  std::vector<int64_t> plan;          // segment bounds in use [k + 1]
  int n_layers = 0;
  int32_t* d_tile_first = nullptr;    // [n_layers + 1] tile range of each layer
  float* d_lrs = nullptr;             // [n_loc][n_layers] rates of the last LARS step
  int64_t* d_layer_bounds = nullptr;  // [n_layers + 1] (single-GPU hierarchical kernel)
  double* d_lars_part = nullptr;      // [n_tiles][n_loc][2]
  bool lars = false;
  float lars_eta = 0.f, lars_wd = 0.f, lars_eps = 0.f;
  bool lars_valid = false;
  // LARS carry: the .x halves of d_lars_part hold sum x'^2 of the last TMA LARS step on xnorm_x
  bool xnorm_valid = false;
  bool lars_carry = false;    // cs_set_lars_carry: the caller promises cs_params_modified
  const float* xnorm_x = nullptr;

  // topology kind (cs_set_topology_kind): SGP's exponential graph as [H][k][world] tables
  int topo_kind = CS_TOPO_CROSSOVER;
  int wire = CS_WIRE_FP32;   // cs_set_wire
  int32_t* d_exp = nullptr;
  int exp_h = 0;

  // multi-GPU schedule (cs_set_schedule) and the single-GPU emulation of V ranks
  // (cs_test_emulate_ranks): both apply from the next cs_bind
  int sched = CS_SCHED_INSTEP;
  int vranks = 1;

  // hot-kernel timing (cs_set_timing): event pairs recorded around each launch
  bool timing = false;
  std::vector<cudaEvent_t> events;
  size_t events_used = 0;
};

Ctx g;

void free_events() {
  for (cudaEvent_t e : g.events) cudaEventDestroy(e);
  g.events.clear();
  g.events_used = 0;
}

// Two events bracketing the next hot-kernel launch (nullptr pair when timing is off).
int next_event_pair(cudaEvent_t* ev) {
  ev[0] = ev[1] = nullptr;
  if (!g.timing) return CS_OK;
  while (g.events.size() < g.events_used + 2) {
    cudaEvent_t e;
    CS_CUDA(cudaEventCreate(&e));
    g.events.push_back(e);
  }
  ev[0] = g.events[g.events_used];
  ev[1] = g.events[g.events_used + 1];
  g.events_used += 2;
  return CS_OK;
}

// Completes a deferred merge of the multi-GPU push/mix schedule (see cs_flush).
int flush_pending() {
  if (!g.bound || !g.use_peer) return CS_OK;
  const int rc = peer_flush(g.peer, g.stream);
  return rc ? fail(rc, "%s", peer_error()) : CS_OK;
}

void free_device() {
  auto f = [](void* p) { if (p) cudaFree(p); };
  f(g.d_bounds); f(g.d_src); f(g.d_dst); f(g.d_ord); f(g.d_given); f(g.d_rw);
  f(g.d_inv_wsum); f(g.d_err); f(g.d_partials); f(g.d_diag); f(g.d_stage); f(g.d_counter); f(g.d_tiles);
  f(g.d_tile_first); f(g.d_lrs); f(g.d_lars_part); f(g.d_exp); f(g.d_layer_bounds);
  g.d_exp = nullptr;
  g.d_layer_bounds = nullptr;
  g.d_tile_first = nullptr; g.d_lrs = nullptr; g.d_lars_part = nullptr;
  g.layer_bounds.clear(); g.plan.clear(); g.n_layers = 0; g.lars_valid = false;
  g.d_bounds = nullptr; g.d_src = nullptr; g.d_dst = nullptr; g.d_ord = nullptr;
  g.d_given = nullptr; g.d_rw = nullptr; g.d_inv_wsum = nullptr; g.d_err = nullptr;
  g.d_partials = nullptr; g.d_diag = nullptr; g.d_stage = nullptr; g.d_counter = nullptr;
  g.d_tiles = nullptr; g.n_tiles = 0; g.use_tma = false;
  g.stage_bytes = 0;
  g.has_override = false;  // the injected topology lived in d_given
  if (g.io_h2d) cudaStreamDestroy(g.io_h2d);
  if (g.io_d2h) cudaStreamDestroy(g.io_d2h);
  for (cudaEvent_t e : g.io_ev) cudaEventDestroy(e);
  g.io_h2d = g.io_d2h = nullptr;
  g.io_ev.clear();
  peer_release(g.peer);
}

std::vector<int64_t> host_bounds(int64_t d, int k) {
  const int64_t nq = (d + kQuantum - 1) / kQuantum;
  std::vector<int64_t> b(k + 1);
  for (int s = 0; s < k; ++s) {
    int64_t v = kQuantum * ((s * nq) / k);
    b[s] = v < d ? v : d;
  }
  b[k] = d;
  return b;
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// SGP's directed exponential graph: worker i sends to
// (i + 2^(t mod log2 n)) mod n, so it receives from (i - 2^(t mod log2 n)) mod n, in
// every segment.  n is a power of two.
int log2_exact(int n) {
  int h = 0;
  while ((1 << h) < n) ++h;
  return h;
}

void exponential_rows(int64_t step, int n, int k, int32_t* src) {
  const int off = 1 << (int)(step % log2_exact(n));
  for (int s = 0; s < k; ++s)
    for (int i = 0; i < n; ++i) src[(int64_t)s * n + i] = (i - off + n) % n;
}

// The flat step's injected topology: the test override, else the exponential table
// row of this step, else nullptr (Alg. 2 drawn on the device).
const int32_t* flat_given() {
  if (g.has_override) return g.d_given;
  if (g.topo_kind == CS_TOPO_EXPONENTIAL && g.d_exp)
    return g.d_exp + (g.step % g.exp_h) * (int64_t)g.k * g.world;
  return nullptr;
}

int upload_exponential() {
  if (g.d_exp) cudaFree(g.d_exp);
  g.d_exp = nullptr;
  g.exp_h = log2_exact(g.world);
  const size_t kn = (size_t)g.k * g.world;
  std::vector<int32_t> tab(kn * g.exp_h);
  for (int h = 0; h < g.exp_h; ++h) exponential_rows(h, g.world, g.k, tab.data() + h * kn);
  CS_CUDA(cudaMalloc(&g.d_exp, sizeof(int32_t) * tab.size()));
  CS_CUDA(cudaMemcpy(g.d_exp, tab.data(), sizeof(int32_t) * tab.size(), cudaMemcpyHostToDevice));
  return CS_OK;
}

// Dynamic tile claims of the next k_gossip_tma launch (consecutive launches on the bound
// stream alternate between two counters; each launch's last CTA zeroes the other one).
void tma_claims(LocalArgs& a) {
  if (!g.tma_dynamic) return;
  const unsigned q = g.claim_seq++ & 1u;
  a.claim = g.d_counter + 1 + q;
  a.claim_next = g.d_counter + 1 + (q ^ 1u);
}

// Bulk-TMA tiles: every (segment, layer) intersection in column order, cut into pieces
// of at most T columns, so each tile lies in one segment and one layer and the tiles of
// a layer are a contiguous range.  Without a layer table the whole vector is layer 0.
int build_tma_tiles() {
  const std::vector<int64_t>& b = g.plan;
  std::vector<int64_t> lb = g.layer_bounds.empty() ? std::vector<int64_t>{0, g.d} : g.layer_bounds;
  const int L = (int)lb.size() - 1;
  // static schedule: a tile length giving a whole number of waves; dynamic claims: full
  // tiles, then small ones over the last columns so the final claims are short
  const int T = g.tma_dynamic ? kTmaTileMax : tma_tile_len(g.d, g.tma_grid_plain);
  const int T_tail = 512;
  const int64_t tail_start =
      g.tma_dynamic ? std::max<int64_t>(0, (g.d - (int64_t)2 * g.tma_grid_plain * T_tail) / 32 * 32) : g.d;
  std::vector<TileDesc> tiles;
  std::vector<int32_t> first(L + 1, 0);
  int l = 0;
  for (int s = 0; s < g.k; ++s) {
    int64_t c = b[s];
    while (c < b[s + 1]) {
      while (lb[l + 1] <= c) first[++l] = (int32_t)tiles.size();
      const int64_t end = std::min(std::min(b[s + 1], lb[l + 1]), c + (c >= tail_start ? T_tail : T));
      TileDesc td;
      td.c0 = c;
      td.seg = s;
      td.len = (int32_t)(end - c);
      td.layer = l;
      td.pad_ = 0;
      tiles.push_back(td);
      c = end;
    }
  }
  while (l < L) first[++l] = (int32_t)tiles.size();
  if (g.d_tiles) cudaFree(g.d_tiles);
  if (g.d_tile_first) cudaFree(g.d_tile_first);
  g.d_tiles = nullptr;
  g.d_tile_first = nullptr;
  g.n_tiles = (int)tiles.size();
  g.h_tile_c0.resize(tiles.size());
  g.h_tile_end.resize(tiles.size());
  for (size_t i = 0; i < tiles.size(); ++i) {
    g.h_tile_c0[i] = tiles[i].c0;
    g.h_tile_end[i] = tiles[i].c0 + tiles[i].len;
  }
  CS_CUDA(cudaMalloc(&g.d_tiles, sizeof(TileDesc) * tiles.size()));
  CS_CUDA(cudaMemcpy(g.d_tiles, tiles.data(), sizeof(TileDesc) * tiles.size(), cudaMemcpyHostToDevice));
  CS_CUDA(cudaMalloc(&g.d_tile_first, sizeof(int32_t) * first.size()));
  CS_CUDA(cudaMemcpy(g.d_tile_first, first.data(), sizeof(int32_t) * first.size(), cudaMemcpyHostToDevice));
  return CS_OK;
}

int check_bound() {
  if (!g.inited) return fail(CS_ENOTINIT, "cs_init has not been called");
  if (!g.bound) return fail(CS_ENOTBOUND, "cs_bind has not been called");
  return CS_OK;
}

int check_step_args(const float* params, const float* grads, const float* psw) {
  if (!params || !grads || !psw) return fail(CS_EINVAL, "NULL params/grads/psw");
  if (!aligned16(params) || !aligned16(grads))
    return fail(CS_ELAYOUT, "params and grads must be 16-byte aligned");
  if (((uintptr_t)psw & 3u) != 0) return fail(CS_ELAYOUT, "psw must be 4-byte aligned");
  if (g.step < 0 || g.step >= (int64_t(1) << 32))
    return fail(CS_EINVAL, "step %lld outside [0, 2^32)", (long long)g.step);
  return CS_OK;
}

// Deferred device errors (topology restart cap, non-finite gradient).
int poll_device_errors() {
  int h[kNumErr] = {0, 0, 0};
  CS_CUDA(cudaMemcpy(h, g.d_err, sizeof(h), cudaMemcpyDeviceToHost));
  if (h[kErrTopology] || h[kErrDiverged] || h[kErrTimeout]) {
    int z[kNumErr] = {0, 0, 0};
    CS_CUDA(cudaMemcpy(g.d_err, z, sizeof(z), cudaMemcpyHostToDevice));
  }
  if (h[kErrTimeout]) return fail(CS_ETIMEOUT, "a cross-GPU wait exceeded its bound");
  if (h[kErrTopology]) return fail(CS_ETOPOLOGY, "Alg.2 restart limit (10,000) exceeded");
  if (h[kErrDiverged]) return fail(CS_EDIVERGED, "non-finite gradient seen in a step");
  return CS_OK;
}

TopoArgs topo_args(int n, int tag, float* psw, int group_size) {
  TopoArgs t;
  t.seed = g.seed;
  t.step = (uint32_t)g.step;
  t.n = n;
  t.k = g.k;
  t.tag = tag;
  t.given = nullptr;
  t.src = g.d_src;
  t.dst = g.d_dst;
  t.ord = g.d_ord;
  t.psw = psw;
  t.group_size = group_size;
  t.rw = g.d_rw;
  t.inv_wsum = g.d_inv_wsum;
  t.err = g.d_err;
  return t;
}

LocalArgs local_args(float* params, const float* grads, float* psw, int n, int gs, int tag,
                     float lr, float mu) {
  LocalArgs a;
  a.x = params;
  a.m = g.mom;
  a.g = grads;
  a.ld = g.ld;
  a.d = g.d;
  a.n = n;
  a.group_size = gs;
  a.k = g.k;
  a.nq = g.nq;
  a.seed = g.seed;
  a.step = (uint32_t)g.step;
  a.tag = tag;
  a.given = nullptr;
  a.ord = g.d_ord;
  a.rw = g.d_rw;
  a.inv_wsum = g.d_inv_wsum;
  a.psw = psw;
  a.lr = lr;
  a.mu = mu;
  a.inv_group = 1.0f / (float)gs;
  a.partials = g.d_partials;
  a.diag_out = g.d_diag;
  a.counter = g.d_counter;
  a.err = g.d_err;
  a.tiles = g.d_tiles;
  a.n_tiles = g.n_tiles;
  a.lrs = nullptr;
  a.n_layers = 0;
  a.wd = 0.f;
  a.wire = g.wire == CS_WIRE_BF16 ? 1 : 0;
  a.seg_bounds = nullptr;
  a.layer_bounds = nullptr;
  a.xnorm_out = nullptr;
  a.skip_psw = 0;
  a.claim = nullptr;
  a.claim_next = nullptr;
  return a;
}

PeerStepArgs peer_args(float* params, const float* grads, float* psw, float lr, float mu) {
  PeerStepArgs pa;
  pa.x = params;
  pa.m = g.mom;
  pa.g = grads;
  pa.psw = psw;
  pa.ld = g.ld;
  pa.d = g.d;
  pa.nq = g.nq;
  pa.k = g.k;
  pa.world = g.world;
  pa.n_loc = g.n_loc;
  pa.first = g.first;
  pa.rank = g.rank;
  pa.nprocs = g.nprocs;
  pa.step = (uint32_t)g.step;
  pa.seed = g.seed;
  pa.lr = lr;
  pa.mu = mu;
  pa.given = nullptr;
  pa.src = g.d_src;
  pa.dst = g.d_dst;
  pa.err = g.d_err;
  pa.groups = g.groups;
  pa.gs = 0;
  pa.inv_gs = 1.0f / (float)(g.world / g.groups);
  pa.wire = g.wire == CS_WIRE_BF16 ? 1 : 0;
  pa.lrs = nullptr;
  pa.n_layers = 0;
  pa.wd = 0.f;
  pa.lrs_out = nullptr;
  pa.eta = 0.f;
  pa.eps = 0.f;
  pa.tile_first = nullptr;
  pa.lars_part = nullptr;
  pa.g_off = 0;
  pa.gbar_local = 0;
  pa.gpull_chunk = 0;
  pa.g_scale = 1.f;
  if (g.vranks > 1) {  // emulated ranks: rank 0's view; each CTA shifts to its own rank
    pa.n_loc = g.world / g.vranks;
    pa.nprocs = g.vranks;
    pa.rank = 0;
    pa.first = 0;
  }
  return pa;
}

int validate_derangements(const int32_t* src, int n, int k) {
  std::vector<int> seen(n);
  for (int s = 0; s < k; ++s) {
    std::fill(seen.begin(), seen.end(), 0);
    for (int i = 0; i < n; ++i) {
      int r = src[(int64_t)s * n + i];
      if (r < 0 || r >= n || r == i || seen[r])
        return fail(CS_EINVAL_TOPOLOGY, "row %d is not a derangement (entry %d -> %d)", s, i, r);
      seen[r] = 1;
    }
  }
  return CS_OK;
}

// One flat step on one GPU.  Small topologies (n <= 64, k*n <= 2048) are built by
// every CTA of the fused kernel itself (one launch per step); larger ones by
// k_topology into global tables first.
int enqueue_flat_step(float* params, const float* grads, float* psw, float lr, float mu,
                      bool diag) {
  const int n = g.world;
  const bool fused = fused_topology_ok(n, g.k);
  LocalArgs a = local_args(params, grads, psw, n, 1, CS_TAG_FLAT, lr, mu);
  if (g.lars && g.n_layers == 0) return fail(CS_EINVAL, "LARS needs a layer table (cs_set_layers)");
  if (g.lars && !(fused && g.use_tma))
    return fail(CS_EUNSUPPORTED, "LARS runs on the bulk-TMA path (world <= 64, k*world <= 2048)");
  if (fused && g.use_tma) {
    a.given = flat_given();
    cudaEvent_t ev[2];
    int rc = next_event_pair(ev);
    if (rc) return rc;
    if (ev[0]) CS_CUDA(cudaEventRecord(ev[0], g.stream));
    if (g.lars) {
      // per-(worker, layer) rates from this step's x and g, then the LARS step kernel.  The
      // x sums come from the previous LARS step's kernel when nothing else touched params
      // (the norm pass then reads only g: 24 instead of 28 B/param)
      const bool carry = g.lars_carry && g.xnorm_valid && g.xnorm_x == params;
      CS_CUDA(launch_lars_rates(params, grads, g.ld, g.d_tiles, g.n_tiles, g.n_loc, g.d_tile_first,
                                g.n_layers, g.d_lars_part, lr, g.lars_eta, g.lars_wd, g.lars_eps,
                                g.d_lrs, g.stream, LarsWait(), carry));
      a.lrs = g.d_lrs;
      a.n_layers = g.n_layers;
      a.wd = g.lars_wd;
      a.xnorm_out = g.d_lars_part;
      g.xnorm_valid = true;
      g.xnorm_x = params;
    } else {
      g.xnorm_valid = false;
    }
    if (!diag) tma_claims(a);  // diagnostics: round-robin tiles, so each CTA's fp64 partials
                               // (summed in CTA order by the last CTA) are the same every run
    CS_CUDA(launch_gossip_tma(a, diag, diag ? g.tma_grid_diag : g.tma_grid_plain, g.stream));
    if (ev[1]) CS_CUDA(cudaEventRecord(ev[1], g.stream));
    g.launches_per_step = g.lars ? 3 : 1;
    g.hot_kernel = g.lars ? "k_lars_norms+k_lars_scale+k_gossip_tma" : "k_gossip_tma";
    if (g.lars) g.lars_valid = true;
    return CS_OK;
  }
  if (fused) {
    a.given = flat_given();
  } else {
    TopoArgs t = topo_args(n, CS_TAG_FLAT, psw, 1);
    t.given = flat_given();
    CS_CUDA(launch_topology(t, g.stream));
  }
  cudaEvent_t ev[2];
  int rc = next_event_pair(ev);
  if (rc) return rc;
  if (ev[0]) CS_CUDA(cudaEventRecord(ev[0], g.stream));
  CS_CUDA(launch_gossip_local(a, diag, fused, g.stream, nullptr));
  if (ev[1]) CS_CUDA(cudaEventRecord(ev[1], g.stream));
  g.launches_per_step = fused ? 1 : 2;
  g.hot_kernel = "k_gossip_local";
  return CS_OK;
}

}  // namespace

extern "C" {

int cs_version(void) { return 300; }  // 0.3.0: in-step merge schedule, emulated ranks, build id

#ifndef CS_BUILD_ID
#define CS_BUILD_ID "unknown-build-id"
#endif
// The marker lets __graft_entry__.build() read the id from the file without loading it.
static const char kBuildIdMarker[] = "CSBUILDID:" CS_BUILD_ID;
const char* cs_build_id(void) { return kBuildIdMarker + 10; }

const char* cs_last_error(void) { return g_err.c_str(); }

int cs_init(int world, int groups, int k_segments, uint64_t seed) {
  g_err.clear();
  if (g.inited) cs_finalize();
  if (world < 2 || world > CS_MAX_WORLD)
    return fail(CS_EINVAL_WORLD, "world %d outside [2, %d]", world, CS_MAX_WORLD);
  if (groups < 1 || world % groups != 0)
    return fail(CS_EINVAL_GROUPS, "groups %d must be >= 1 and divide world %d", groups, world);
  if (k_segments < 1 || k_segments > CS_MAX_SEGMENTS)
    return fail(CS_EINVAL_SEGMENTS, "k %d outside [1, %d]", k_segments, CS_MAX_SEGMENTS);
  g = Ctx();
  g.world = world;
  g.groups = groups;
  g.k = k_segments;
  g.seed = seed;
  g.inited = true;
  return CS_OK;
}

void cs_finalize(void) {
  if (g.bound) {
    flush_pending();
    cudaStreamSynchronize(g.stream);
    free_device();
  }
  free_events();
  g = Ctx();
}

int cs_segment_bounds(int64_t d, int64_t* bounds_out) {
  if (!g.inited) return fail(CS_ENOTINIT, "cs_init has not been called");
  if (!bounds_out) return fail(CS_EINVAL, "NULL bounds_out");
  if (d < 1) return fail(CS_ELAYOUT, "d must be >= 1");
  if ((d + kQuantum - 1) / kQuantum < g.k)
    return fail(CS_EINVAL_SEGMENTS, "k %d > ceil(d/32) = %lld", g.k, (long long)((d + 31) / 32));
  std::vector<int64_t> b = host_bounds(d, g.k);
  memcpy(bounds_out, b.data(), sizeof(int64_t) * b.size());
  return CS_OK;
}

static int topology_common(int64_t step, int n, int tag, int32_t* src_out) {
  if (!g.inited) return fail(CS_ENOTINIT, "cs_init has not been called");
  if (!src_out) return fail(CS_EINVAL, "NULL src_out");
  if (step < 0 || step >= (int64_t(1) << 32))
    return fail(CS_EINVAL, "step %lld outside [0, 2^32)", (long long)step);
  if (tag == CS_TAG_FLAT && g.topo_kind == CS_TOPO_EXPONENTIAL) {
    exponential_rows(step, n, g.k, src_out);
    return CS_OK;
  }
  for (int s = 0; s < g.k; ++s) {
    if (host_alg2(g.seed, (uint32_t)step, (uint32_t)s, n, tag, src_out + (int64_t)s * n) < 0)
      return fail(CS_ETOPOLOGY, "Alg.2 restart limit (10,000) exceeded");
  }
  return CS_OK;
}

int cs_topology(int64_t step, int32_t* src_out) {
  return topology_common(step, g.world, CS_TAG_FLAT, src_out);
}

int cs_topology_hier(int64_t step, int32_t* src_out) {
  if (g.inited && g.groups < 2)
    return fail(CS_EINVAL_GROUPS, "leader topology needs groups >= 2 (have %d)", g.groups);
  return topology_common(step, g.groups, CS_TAG_HIER, src_out);
}

int cs_bind(float* momentum, int64_t d, int64_t ld, int proc_rank, int nprocs, void* stream) {
  if (!g.inited) return fail(CS_ENOTINIT, "cs_init has not been called");
  if (nprocs < 1 || proc_rank < 0 || proc_rank >= nprocs)
    return fail(CS_EINVAL, "proc_rank %d / nprocs %d invalid", proc_rank, nprocs);
  if (g.world % nprocs != 0)
    return fail(CS_EINVAL_WORLD, "world %d not divisible by nprocs %d", g.world, nprocs);
  if (!momentum) return fail(CS_EINVAL, "NULL momentum");
  if (d < 1 || ld < d || (ld & 3) != 0)
    return fail(CS_ELAYOUT, "need d >= 1, ld >= d, ld %% 4 == 0 (d=%lld ld=%lld)", (long long)d,
                (long long)ld);
  if (!aligned16(momentum)) return fail(CS_ELAYOUT, "momentum must be 16-byte aligned");
  if ((d + kQuantum - 1) / kQuantum < g.k)
    return fail(CS_EINVAL_SEGMENTS, "k %d > ceil(d/32) = %lld", g.k, (long long)((d + 31) / 32));
  if (g.bound) {
    flush_pending();
    cudaStreamSynchronize(g.stream);
    free_device();
    g.bound = false;
  }
  g.d = d;
  g.ld = ld;
  g.nq = (d + kQuantum - 1) / kQuantum;
  g.xnorm_valid = false;
  g.rank = proc_rank;
  g.nprocs = nprocs;
  g.n_loc = g.world / nprocs;
  g.first = proc_rank * g.n_loc;
  g.mom = momentum;
  g.stream = (cudaStream_t)stream;
  CS_CUDA(cudaGetDevice(&g.device));
  const size_t kn = (size_t)g.k * g.world;
  std::vector<int64_t> b = host_bounds(d, g.k);
  g.plan = b;
  CS_CUDA(cudaMalloc(&g.d_bounds, sizeof(int64_t) * b.size()));
  CS_CUDA(cudaMemcpy(g.d_bounds, b.data(), sizeof(int64_t) * b.size(), cudaMemcpyHostToDevice));
  CS_CUDA(cudaMalloc(&g.d_src, sizeof(int32_t) * kn));
  CS_CUDA(cudaMalloc(&g.d_dst, sizeof(int32_t) * kn));
  CS_CUDA(cudaMalloc(&g.d_ord, sizeof(uint32_t) * kn));
  CS_CUDA(cudaMalloc(&g.d_given, sizeof(int32_t) * kn));
  CS_CUDA(cudaMalloc(&g.d_rw, sizeof(double) * kn));
  CS_CUDA(cudaMalloc(&g.d_inv_wsum, sizeof(double) * g.k));
  CS_CUDA(cudaMalloc(&g.d_err, sizeof(int) * kNumErr));
  CS_CUDA(cudaMemset(g.d_err, 0, sizeof(int) * kNumErr));
  CS_CUDA(cudaMalloc(&g.d_diag, sizeof(double) * 2));
  CS_CUDA(cudaMalloc(&g.d_partials, sizeof(double) * 2 * (size_t)local_max_grid()));
  CS_CUDA(cudaMalloc(&g.d_counter, 4 * sizeof(unsigned)));  // arrival counter, 2 tile-claim counters
  CS_CUDA(cudaMemset(g.d_counter, 0, 4 * sizeof(unsigned)));
  g.claim_seq = 0;
  g.tma_dynamic = !(getenv("CS_TMA_DYNAMIC") && getenv("CS_TMA_DYNAMIC")[0] == '0');
  if (g.vranks > 1 && (nprocs != 1 || g.world % g.vranks != 0))
    return fail(CS_EINVAL, "emulated ranks need nprocs == 1 and vranks dividing world");
  g.use_peer = nprocs > 1 || g.path == CS_PATH_PEER || g.vranks > 1;
  if (g.path == CS_PATH_TMA && !fused_topology_ok(g.world, g.k))
    return fail(CS_EUNSUPPORTED, "CS_PATH_TMA needs world <= 64 and k*world <= 2048");
  g.use_tma = !g.use_peer && g.path != CS_PATH_REG && fused_topology_ok(g.world, g.k);
  if (g.use_tma) {
    g.tma_grid_plain = tma_grid(g.world, g.k, false);
    g.tma_grid_diag = tma_grid(g.world, g.k, true);
    CS_CUDA(cudaGetLastError());
    int rc = build_tma_tiles();
    if (rc) return rc;
  }
  if (g.use_peer) {
    // hierarchical steps over the peer path: one worker per GPU, groups of world/groups GPUs
    const int ranks = g.vranks > 1 ? g.vranks : nprocs;
    const int n_loc_rank = g.world / ranks;
    const int hier_gs = (ranks > 1 && n_loc_rank == 1) ? g.world / g.groups : 0;
    int rc = peer_alloc(g.peer, n_loc_rank, d, ld, g.k, ranks, g.vranks > 1 ? 0 : proc_rank, hier_gs, g.vranks);
    if (rc) return fail(rc, "%s", peer_error());
    rc = peer_set_schedule(g.peer, g.sched, g.stream);
    if (rc) return fail(rc, "%s", peer_error());
    if (nprocs == 1) {  // single-GPU emulation: every rank's region is on this GPU
      rc = peer_import_self(g.peer);
      if (rc) return fail(rc, "%s", peer_error());
    }
  }
  if (g.topo_kind == CS_TOPO_EXPONENTIAL) {
    int rc = upload_exponential();
    if (rc) return rc;
  }
  g.bound = true;
  g.diag_valid = false;
  return CS_OK;
}

int cs_set_wire(int format) {
  if (!g.inited) return fail(CS_ENOTINIT, "cs_init has not been called");
  if (int rc = flush_pending()) return rc;  // a pending merge reads the inbox in the current format
  if (format != CS_WIRE_FP32 && format != CS_WIRE_BF16) return fail(CS_EINVAL, "unknown wire format %d", format);
  g.wire = format;
  return CS_OK;
}

int cs_set_topology_kind(int kind) {
  if (!g.inited) return fail(CS_ENOTINIT, "cs_init has not been called");
  if (kind != CS_TOPO_CROSSOVER && kind != CS_TOPO_EXPONENTIAL)
    return fail(CS_EINVAL, "unknown topology kind %d", kind);
  if (kind == CS_TOPO_EXPONENTIAL && (g.world & (g.world - 1)) != 0)
    return fail(CS_EUNSUPPORTED, "the exponential graph needs a power-of-two world (have %d)", g.world);
  g.topo_kind = kind;
  if (g.bound && kind == CS_TOPO_EXPONENTIAL) return upload_exponential();
  return CS_OK;
}

int cs_set_path(int path) {
  if (!g.inited) return fail(CS_ENOTINIT, "cs_init has not been called");
  if (path < CS_PATH_AUTO || path > CS_PATH_PEER) return fail(CS_EINVAL, "unknown path %d", path);
  g.path = path;
  return CS_OK;
}

int cs_set_schedule(int schedule) {
  if (!g.inited) return fail(CS_ENOTINIT, "cs_init has not been called");
  if (schedule < CS_SCHED_INSTEP || schedule > CS_SCHED_SPLIT) return fail(CS_EINVAL, "unknown schedule %d", schedule);
  g.sched = schedule;
  if (g.bound && g.use_peer) {
    const int rc = peer_set_schedule(g.peer, schedule, g.stream);
    if (rc) return fail(rc, "%s", peer_error());
  }
  return CS_OK;
}

int cs_test_emulate_ranks(int vranks) {
  if (!g.inited) return fail(CS_ENOTINIT, "cs_init has not been called");
  if (vranks < 1 || vranks > g.world || g.world % vranks != 0)
    return fail(CS_EINVAL, "vranks %d must divide world %d", vranks, g.world);
  g.vranks = vranks;
  return CS_OK;
}

int cs_set_stream(void* stream) {
  int rc = check_bound();
  if (rc) return rc;
  // the library's scratch (arrival counters, partials, a pending deferred merge) is shared by
  // work on both streams: the new stream starts after everything queued on the old one
  if ((cudaStream_t)stream != g.stream) {
    cudaEvent_t ev;
    CS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    cudaError_t e = cudaEventRecord(ev, g.stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent((cudaStream_t)stream, ev, 0);
    cudaEventDestroy(ev);
    if (e != cudaSuccess) return cuda_fail(e, "cs_set_stream ordering");
  }
  g.stream = (cudaStream_t)stream;
  return CS_OK;
}

int cs_ipc_export(char* handle_out) {
  int rc = check_bound();
  if (rc) return rc;
  if (!handle_out) return fail(CS_EINVAL, "NULL handle_out");
  if (g.nprocs < 2) return fail(CS_EINVAL, "cs_ipc_export needs nprocs > 1");
  rc = peer_export(g.peer, handle_out);
  return rc ? fail(rc, "%s", peer_error()) : CS_OK;
}

int cs_ipc_import(const char* all_handles) {
  int rc = check_bound();
  if (rc) return rc;
  if (!all_handles) return fail(CS_EINVAL, "NULL all_handles");
  if (g.nprocs < 2) return fail(CS_EINVAL, "cs_ipc_import needs nprocs > 1");
  rc = peer_import(g.peer, all_handles);
  return rc ? fail(rc, "%s", peer_error()) : CS_OK;
}

int cs_multicast_bytes(int64_t* bytes_out) {
  int rc = check_bound();
  if (rc) return rc;
  if (!bytes_out) return fail(CS_EINVAL, "NULL bytes_out");
  *bytes_out = (int64_t)nvls_bytes(g.ld);
  return CS_OK;
}

int cs_set_multicast(void* uc_base, void* mc_base, int64_t bytes) {
  int rc = check_bound();
  if (rc) return rc;
  PeerState& p = g.peer;
  if (uc_base == nullptr) {  // back to the point-to-point reduce-scatter
    if ((rc = flush_pending()) != CS_OK) return rc;
    CS_CUDA(cudaStreamSynchronize(g.stream));
    p.mc_uc = p.mc_mc = nullptr;
    p.mc_bytes = 0;
    p.mc_grads.clear();
    return CS_OK;
  }
  if (!mc_base) return fail(CS_EINVAL, "NULL mc_base");
  if (g.nprocs < 2 || g.vranks > 1 || !p.imported)
    return fail(CS_EUNSUPPORTED, "multicast h1 needs one process per GPU with the peers imported");
  if (p.gs < 2) return fail(CS_EUNSUPPORTED, "multicast h1 needs hierarchical groups of >= 2 GPUs");
  if (bytes < (int64_t)nvls_bytes(g.ld))
    return fail(CS_EINVAL, "multicast workspace of %lld bytes < cs_multicast_bytes() = %lld", (long long)bytes,
                (long long)nvls_bytes(g.ld));
  if (((uintptr_t)uc_base | (uintptr_t)mc_base) % 256 != 0) return fail(CS_ELAYOUT, "multicast workspace not 256-B aligned");
  CS_CUDA(cudaStreamSynchronize(g.stream));
  if (!p.d_nvls_count) CS_CUDA(cudaMalloc(&p.d_nvls_count, 128));
  CS_CUDA(cudaMemset(p.d_nvls_count, 0, 128));
  CS_CUDA(cudaMemset(uc_base, 0, nvls_off_gbar()));  // barrier words (callers barrier before stepping)
  CS_CUDA(cudaDeviceSynchronize());
  nccl_group_release(p);  // one h1 route at a time
  p.mc_uc = static_cast<char*>(uc_base);
  p.mc_mc = static_cast<char*>(mc_base);
  p.mc_bytes = (size_t)bytes;
  p.nvls_epoch = 0;
  p.nvls_tot[0] = p.nvls_tot[1] = 0;
  return CS_OK;
}

int cs_nccl_unique_id(char* id_out) {
  if (!id_out) return fail(CS_EINVAL, "NULL id_out");
  if (nccl_unique_id(id_out)) return fail(CS_EUNSUPPORTED, "%s", nccl_error());
  return CS_OK;
}

int cs_set_hier_nccl(const char* group_id) {
  int rc = check_bound();
  if (rc) return rc;
  PeerState& p = g.peer;
  if (group_id && (g.nprocs < 2 || g.vranks > 1 || !p.imported))
    return fail(CS_EUNSUPPORTED, "NCCL h1 needs one process per GPU with the peers imported");
  if (group_id && p.gs < 2) return fail(CS_EUNSUPPORTED, "NCCL h1 needs hierarchical groups of >= 2 GPUs");
  if ((rc = flush_pending()) != CS_OK) return rc;
  CS_CUDA(cudaStreamSynchronize(g.stream));
  if (group_id && p.mc_uc) {  // one h1 route at a time
    p.mc_uc = p.mc_mc = nullptr;
    p.mc_grads.clear();
  }
  if (nccl_group_init(p, group_id, p.gs > 0 ? g.rank % p.gs : 0))
    return fail(CS_ECUDA, "%s", nccl_error());
  return CS_OK;
}

int cs_add_multicast_grads(void* uc_base, void* mc_base, int64_t bytes) {
  int rc = check_bound();
  if (rc) return rc;
  if (!g.peer.mc_uc) return fail(CS_ENOTBOUND, "cs_set_multicast has not been called");
  if (!uc_base || !mc_base || bytes <= 0) return fail(CS_EINVAL, "NULL region or bytes <= 0");
  if (((uintptr_t)uc_base | (uintptr_t)mc_base) % 16 != 0) return fail(CS_ELAYOUT, "region not 16-B aligned");
  if (g.peer.mc_grads.size() >= 8) return fail(CS_EINVAL, "at most 8 multicast gradient regions");
  g.peer.mc_grads.push_back({static_cast<char*>(uc_base), static_cast<char*>(mc_base), (size_t)bytes});
  return CS_OK;
}

int cs_gossip_step(float* params, const float* grads, float* psw, float lr, float momentum) {
  int rc = check_bound();
  if (rc) return rc;
  rc = check_step_args(params, grads, psw);
  if (rc) return rc;
  const bool diag = g.diag != 0;
  if (!g.use_peer) {
    rc = enqueue_flat_step(params, grads, psw, lr, momentum, diag);
  } else {
    if (!g.peer.imported) return fail(CS_ENOTBOUND, "multi-GPU: cs_ipc_import has not been called");
    if (g.lars && g.n_layers == 0) return fail(CS_EINVAL, "LARS needs a layer table (cs_set_layers)");
    if (g.n_layers > 0 && g.wire != CS_WIRE_FP32)
      return fail(CS_EUNSUPPORTED, "bf16 wire with a layer table is not implemented on the multi-GPU path");
    PeerStepArgs pa = peer_args(params, grads, psw, lr, momentum);
    pa.given = flat_given();
    cudaEvent_t ev[2];
    rc = next_event_pair(ev);
    if (rc) return rc;
    if (g.lars) {  // per-(worker, layer) rates from this step's x and g, over the peer tiles
      if (ev[0]) CS_CUDA(cudaEventRecord(ev[0], g.stream));  // the timed pair covers the rates
      if ((rc = flush_pending()) != CS_OK) return rc;        // the norms need the merged x
      ev[0] = nullptr;
      CS_CUDA(launch_lars_rates(params, grads, g.ld, peer_tiles(g.peer), peer_tile_count(g.peer), g.n_loc,
                                g.d_tile_first, g.n_layers, g.d_lars_part, lr, g.lars_eta, g.lars_wd,
                                g.lars_eps, g.d_lrs, g.stream));
      pa.lrs = g.d_lrs;
      pa.n_layers = g.n_layers;
      pa.wd = g.lars_wd;
      g.lars_valid = true;
    }
    rc = peer_flat_step(g.peer, pa, g.stream, ev[0], ev[1]);
    if (rc) return fail(rc, "%s", peer_error());
    if (diag) {
      if ((rc = flush_pending()) != CS_OK) return rc;  // diagnostics of the merged x'
      rc = peer_diag(g.peer, pa, g.d_partials, local_max_grid(), g.d_diag, g.stream);
      if (rc) return fail(rc, "%s", peer_error());
    }
    const bool fused_topo = g.world <= 64;  // the topology is drawn inside the first kernel
    const bool merge = peer_merge_ok(g.peer, pa);
    // in-step merge: one launch; deferred merge: one push launch per step (its merge runs in
    // the next push / cs_flush); split: push + mix
    g.launches_per_step = ((merge || g.peer.last_fused) ? 1 : 2) + (fused_topo ? 0 : 1) + (g.lars ? 2 : 0);
    g.hot_kernel = merge               ? (g.lars ? "k_lars_norms+k_lars_scale+k_push_merge" : "k_push_merge")
                   : g.peer.use_hybrid ? (g.peer.last_fused ? "k_hyb_walk(fused tail merge)" : "k_hyb_walk+k_hyb_tail")
                   : g.lars           ? "k_lars_norms+k_lars_scale+k_peer_push+k_peer_mix"
                   : g.peer.last_fused ? "k_peer_push(fused merge)"
                                       : "k_peer_push+k_peer_mix";
  }
  if (rc) return rc;
  if (diag) g.diag_valid = true;
  g.step += 1;
  return CS_OK;
}

int cs_gossip_step_host(float* params, const float* grads_host, float* psw, float lr,
                        float momentum, double* diag_out) {
  int rc = check_bound();
  if (rc) return rc;
  if (!grads_host || !diag_out) return fail(CS_EINVAL, "NULL grads_host/diag_out");
  if (g.use_peer) return fail(CS_EUNSUPPORTED, "cs_gossip_step_host is single-GPU (local paths)");
  const size_t bytes = sizeof(float) * (size_t)g.n_loc * (size_t)g.ld;
  if (g.stage_bytes < bytes) {
    if (g.d_stage) cudaFree(g.d_stage);
    g.d_stage = nullptr;
    CS_CUDA(cudaMalloc(&g.d_stage, bytes));
    g.stage_bytes = bytes;
  }
  CS_CUDA(cudaMemcpyAsync(g.d_stage, grads_host, bytes, cudaMemcpyHostToDevice, g.stream));
  rc = check_step_args(params, g.d_stage, psw);
  if (rc) return rc;
  rc = enqueue_flat_step(params, g.d_stage, psw, lr, momentum, true);
  if (rc) return rc;
  g.diag_valid = true;
  g.step += 1;
  CS_CUDA(cudaMemcpyAsync(diag_out, g.d_diag, 2 * sizeof(double), cudaMemcpyDeviceToHost, g.stream));
  CS_CUDA(cudaStreamSynchronize(g.stream));
  return poll_device_errors();
}

int cs_gossip_step_io(float* params, const float* grads_host, float* psw, float lr, float momentum,
                      float* params_host_out, float* psw_host_out) {
  int rc = check_bound();
  if (rc) return rc;
  if (!grads_host || !params_host_out || !psw_host_out) return fail(CS_EINVAL, "NULL host buffer");
  if (g.use_peer || !g.use_tma || g.lars || !fused_topology_ok(g.world, g.k))
    return fail(CS_EUNSUPPORTED, "cs_gossip_step_io runs on the single-GPU bulk-TMA path without LARS");
  const size_t bytes = sizeof(float) * (size_t)g.n_loc * (size_t)g.ld;
  if (g.stage_bytes < bytes) {
    if (g.d_stage) cudaFree(g.d_stage);
    g.d_stage = nullptr;
    CS_CUDA(cudaMalloc(&g.d_stage, bytes));
    g.stage_bytes = bytes;
  }
  rc = check_step_args(params, g.d_stage, psw);
  if (rc) return rc;
  constexpr int P = 8;  // column pieces: H2D of piece q+1 and D2H of piece q-1 overlap step piece q
  if (!g.io_h2d) {
    CS_CUDA(cudaStreamCreateWithFlags(&g.io_h2d, cudaStreamNonBlocking));
    CS_CUDA(cudaStreamCreateWithFlags(&g.io_d2h, cudaStreamNonBlocking));
    g.io_ev.resize(2 * P + 1);
    for (auto& e : g.io_ev) CS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  // the previous io step's reads of the staging buffer (its pieces) precede this step's copies
  CS_CUDA(cudaEventRecord(g.io_ev[2 * P], g.stream));
  CS_CUDA(cudaStreamWaitEvent(g.io_h2d, g.io_ev[2 * P], 0));
  cudaEvent_t ev[2];
  rc = next_event_pair(ev);
  if (rc) return rc;
  if (ev[0]) CS_CUDA(cudaEventRecord(ev[0], g.stream));
  const int nt = g.n_tiles;
  const size_t pitch = sizeof(float) * (size_t)g.ld;
  for (int q = 0; q < P; ++q) {
    const int t_lo = (int)((int64_t)q * nt / P), t_hi = (int)((int64_t)(q + 1) * nt / P);
    if (t_hi <= t_lo) continue;
    const int64_t c_lo = g.h_tile_c0[t_lo], c_hi = g.h_tile_end[t_hi - 1];
    const size_t width = sizeof(float) * (size_t)(c_hi - c_lo);
    CS_CUDA(cudaMemcpy2DAsync(g.d_stage + c_lo, pitch, grads_host + c_lo, pitch, width, g.n_loc,
                              cudaMemcpyHostToDevice, g.io_h2d));
    CS_CUDA(cudaEventRecord(g.io_ev[q], g.io_h2d));
    CS_CUDA(cudaStreamWaitEvent(g.stream, g.io_ev[q], 0));
    LocalArgs a = local_args(params, g.d_stage, psw, g.world, 1, CS_TAG_FLAT, lr, momentum);
    a.given = flat_given();
    a.tiles = g.d_tiles + t_lo;  // this piece's tiles; the last piece also mixes psw
    a.n_tiles = t_hi - t_lo;
    a.skip_psw = t_hi < nt ? 1 : 0;
    tma_claims(a);
    CS_CUDA(launch_gossip_tma(a, false, g.tma_grid_plain, g.stream));
    CS_CUDA(cudaEventRecord(g.io_ev[P + q], g.stream));
    CS_CUDA(cudaStreamWaitEvent(g.io_d2h, g.io_ev[P + q], 0));
    CS_CUDA(cudaMemcpy2DAsync(params_host_out + c_lo, pitch, params + c_lo, pitch, width, g.n_loc,
                              cudaMemcpyDeviceToHost, g.io_d2h));
  }
  CS_CUDA(cudaMemcpyAsync(psw_host_out, psw, sizeof(float) * (size_t)g.n_loc * g.k, cudaMemcpyDeviceToHost,
                          g.io_d2h));
  CS_CUDA(cudaEventRecord(g.io_ev[2 * P], g.io_d2h));
  CS_CUDA(cudaStreamWaitEvent(g.stream, g.io_ev[2 * P], 0));
  if (ev[1]) CS_CUDA(cudaEventRecord(ev[1], g.stream));
  g.launches_per_step = P;
  g.hot_kernel = "k_gossip_tma";
  g.xnorm_valid = false;
  g.step += 1;
  CS_CUDA(cudaStreamSynchronize(g.io_d2h));
  return poll_device_errors();
}

int cs_hier_step(float* params, float* grads, float* psw, float lr, float momentum) {
  int rc = check_bound();
  if (rc) return rc;
  g.xnorm_valid = false;
  if ((g.lars || g.n_layers > 0) && g.nprocs == 1 && g.vranks <= 1 && (g.use_peer || !g.use_tma))
    return fail(CS_EUNSUPPORTED, "LARS / layer tables in the single-GPU hierarchical step need the bulk-TMA tiles");
  if (g.lars && g.n_layers == 0) return fail(CS_EINVAL, "LARS needs a layer table (cs_set_layers)");
  if (g.wire != CS_WIRE_FP32)
    return fail(CS_EUNSUPPORTED, "the bf16 wire format is implemented for the flat step only");
  rc = check_step_args(params, grads, psw);
  if (rc) return rc;
  const bool diag = g.diag != 0;
  if (g.nprocs > 1 || g.vranks > 1) {  // across GPUs, or their single-GPU emulation
    if ((g.vranks > 1 ? g.world / g.vranks : g.n_loc) != 1)
      return fail(CS_EUNSUPPORTED, "multi-GPU hierarchical step needs one worker per GPU (world == nprocs)");
    if (!g.peer.imported) return fail(CS_ENOTBOUND, "multi-GPU: cs_ipc_import has not been called");
    PeerStepArgs pa = peer_args(params, grads, psw, lr, momentum);
    if (g.lars) {  // rates from the leader replica's x and the group mean
      pa.lrs_out = g.d_lrs;
      pa.n_layers = g.n_layers;
      pa.wd = g.lars_wd;
      pa.eta = g.lars_eta;
      pa.eps = g.lars_eps;
      pa.tile_first = g.d_tile_first;
      pa.lars_part = g.d_lars_part;
      g.lars_valid = true;
    }
    cudaEvent_t ev[2];
    rc = next_event_pair(ev);
    if (rc) return rc;
    const long launches0 = g_peer_launches;
    rc = peer_hier_step(g.peer, pa, g.stream, ev[0], ev[1]);
    if (rc) return fail(rc, "%s", peer_error());
    if (diag) {
      if ((rc = flush_pending()) != CS_OK) return rc;  // diagnostics of the merged x'
      rc = peer_diag(g.peer, pa, g.d_partials, local_max_grid(), g.d_diag, g.stream);
      if (rc) return fail(rc, "%s", peer_error());
      g.diag_valid = true;
    }
    // (topology,) scatter, reduce, push (, mix unless the leader exchange's merge is deferred)
    g.launches_per_step = (int)(g_peer_launches - launches0) + (g.lars ? 2 : 0);
    g.hot_kernel = g.lars ? "k_hier_scatter+k_hier_reduce+k_lars_norms+k_lars_scale+k_peer_push+k_peer_mix"
                   : g.peer.last_nvls ? (g.groups >= 2 ? "k_hier_nvls+k_push_merge" : "k_hier_nvls+k_peer_push")
                   : g.peer.last_nccl ? (g.groups >= 2 ? "ncclAllReduce+k_push_merge" : "ncclAllReduce+k_peer_push")
                                      : "k_hier_scatter+k_hier_reduce+k_peer_push+k_peer_mix";
    g.step += 1;
    return CS_OK;
  }
  const int L = g.groups, gs = g.world / g.groups;
  const bool fused = fused_topology_ok(L, g.k);
  LocalArgs a = local_args(params, grads, psw, L, gs, CS_TAG_HIER, lr, momentum);
  if (g.n_layers > 0) {  // layer plan (C-19) and layer lookups for LARS
    a.seg_bounds = g.d_bounds;
    a.layer_bounds = g.d_layer_bounds;
    a.n_layers = g.n_layers;
  }
  if (!fused) {
    TopoArgs t = topo_args(L, CS_TAG_HIER, psw, gs);
    CS_CUDA(launch_topology(t, g.stream));
  }
  cudaEvent_t ev[2];
  rc = next_event_pair(ev);
  if (rc) return rc;
  if (ev[0]) CS_CUDA(cudaEventRecord(ev[0], g.stream));
  if (g.lars) {  // rates per (group, layer) from the leader's x and the group mean
    CS_CUDA(launch_lars_rates_hier(params, grads, g.ld, g.d_tiles, g.n_tiles, L, gs, a.inv_group, g.d_tile_first,
                                   g.n_layers, g.d_lars_part, lr, g.lars_eta, g.lars_wd, g.lars_eps, g.d_lrs,
                                   g.stream));
    a.lrs = g.d_lrs;
    a.wd = g.lars_wd;
    g.lars_valid = true;
  }
  CS_CUDA(launch_hier_local(a, diag, fused, g.stream, nullptr));
  if (ev[1]) CS_CUDA(cudaEventRecord(ev[1], g.stream));
  if (diag) g.diag_valid = true;
  g.launches_per_step = (fused ? 1 : 2) + (g.lars ? 2 : 0);
  g.hot_kernel = g.lars ? "k_lars_norms_hier+k_lars_scale+k_hier_local" : "k_hier_local";
  g.step += 1;
  return CS_OK;
}

int cs_segment_plan(const int64_t* layer_sizes, int n_layers, int k, int32_t* seg_of_layer_out) {
  if (!layer_sizes || !seg_of_layer_out) return fail(CS_EINVAL, "NULL layer_sizes/seg_of_layer_out");
  if (n_layers < 1 || n_layers > CS_MAX_LAYERS)
    return fail(CS_EINVAL, "n_layers %d outside [1, %d]", n_layers, CS_MAX_LAYERS);
  if (k < 1 || k > n_layers) return fail(CS_EINVAL_SEGMENTS, "k %d outside [1, n_layers=%d]", k, n_layers);
  std::vector<int64_t> pre(n_layers + 1, 0);
  int64_t mx = 0;
  for (int i = 0; i < n_layers; ++i) {
    if (layer_sizes[i] < 1) return fail(CS_EINVAL, "layer %d has size %lld", i, (long long)layer_sizes[i]);
    pre[i + 1] = pre[i] + layer_sizes[i];
    mx = std::max(mx, layer_sizes[i]);
  }
  // can layers [i, n) be cut into at most `pieces` contiguous runs of <= cap?
  auto feasible = [&](int i, int pieces, int64_t cap) {
    int used = (i < n_layers) ? 1 : 0;
    int64_t cur = 0;
    for (int j = i; j < n_layers; ++j) {
      if (cur + layer_sizes[j] > cap) { ++used; cur = layer_sizes[j]; }
      else cur += layer_sizes[j];
    }
    return used <= pieces;
  };
  // smallest cap (a contiguous sum) admitting k pieces: binary search on integers
  int64_t lo = mx, hi = pre[n_layers];
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (feasible(0, k, mid)) hi = mid; else lo = mid + 1;
  }
  const int64_t cap = lo;
  // each segment, left to right, takes as many layers as the cap and the rest allow
  int start = 0;
  for (int s = 0; s < k; ++s) {
    const int left = k - s - 1;
    int end = n_layers;
    if (left > 0) {
      int e1 = start + 1;  // largest end with sum(start, e1) <= cap
      while (e1 + 1 <= n_layers - left && pre[e1 + 1] - pre[start] <= cap) ++e1;
      end = e1;
      while (end > start + 1 && !feasible(end, left, cap)) --end;
    }
    for (int i = start; i < end; ++i) seg_of_layer_out[i] = s;
    start = end;
  }
  return CS_OK;
}

int cs_set_layers(const int64_t* layer_bounds, int n_layers, const int32_t* seg_of_layer) {
  int rc = check_bound();
  if (rc) return rc;
  if ((rc = flush_pending()) != CS_OK) return rc;  // the tiles change
  g.xnorm_valid = false;
  if (!layer_bounds || n_layers == 0) {  // clear: back to the equal split, no layers
    g.layer_bounds.clear();
    g.n_layers = 0;
    g.plan = host_bounds(g.d, g.k);
    CS_CUDA(cudaMemcpy(g.d_bounds, g.plan.data(), sizeof(int64_t) * g.plan.size(), cudaMemcpyHostToDevice));
    if (g.use_peer) {
      std::vector<int32_t> first;
      rc = peer_set_layers(g.peer, g.plan, g.layer_bounds, first);
      return rc ? fail(rc, "%s", peer_error()) : CS_OK;
    }
    return g.use_tma ? build_tma_tiles() : CS_OK;
  }
  if (n_layers < 1 || n_layers > CS_MAX_LAYERS)
    return fail(CS_EINVAL, "n_layers %d outside [1, %d]", n_layers, CS_MAX_LAYERS);
  if (g.use_peer ? false : !g.use_tma)
    return fail(CS_EUNSUPPORTED, "layer tables run on the single-GPU bulk-TMA path and the multi-GPU paths");
  if (layer_bounds[0] != 0 || layer_bounds[n_layers] != g.d)
    return fail(CS_ELAYOUT, "layer bounds must run from 0 to d = %lld", (long long)g.d);
  for (int i = 0; i < n_layers; ++i) {
    if (layer_bounds[i + 1] <= layer_bounds[i])
      return fail(CS_ELAYOUT, "layer %d is empty or the bounds decrease", i);
    if (layer_bounds[i] % 4 != 0)
      return fail(CS_ELAYOUT, "layer bound %lld is not a multiple of 4 elements", (long long)layer_bounds[i]);
  }
  std::vector<int64_t> plan;
  if (seg_of_layer) {
    if (seg_of_layer[0] != 0 || seg_of_layer[n_layers - 1] != g.k - 1)
      return fail(CS_EINVAL_SEGMENTS, "seg_of_layer must run from 0 to k-1 = %d", g.k - 1);
    plan.push_back(0);
    for (int i = 1; i < n_layers; ++i) {
      const int step = seg_of_layer[i] - seg_of_layer[i - 1];
      if (step != 0 && step != 1)
        return fail(CS_EINVAL_SEGMENTS, "seg_of_layer must be contiguous (layer %d)", i);
      if (step == 1) plan.push_back(layer_bounds[i]);
    }
    plan.push_back(g.d);
  } else {
    plan = host_bounds(g.d, g.k);
  }
  g.layer_bounds.assign(layer_bounds, layer_bounds + n_layers + 1);
  g.n_layers = n_layers;
  g.plan = plan;
  int tiles_for_norms = 0;
  if (g.use_peer) {  // every process sets the same table (collective by convention)
    CS_CUDA(cudaStreamSynchronize(g.stream));
    std::vector<int32_t> first;
    rc = peer_set_layers(g.peer, g.plan, g.layer_bounds, first);
    if (rc) return fail(rc, "%s", peer_error());
    if (g.d_tile_first) cudaFree(g.d_tile_first);
    g.d_tile_first = nullptr;
    CS_CUDA(cudaMalloc(&g.d_tile_first, sizeof(int32_t) * first.size()));
    CS_CUDA(cudaMemcpy(g.d_tile_first, first.data(), sizeof(int32_t) * first.size(), cudaMemcpyHostToDevice));
    tiles_for_norms = peer_tile_count(g.peer);
  } else {
    rc = build_tma_tiles();
    if (rc) return rc;
    tiles_for_norms = g.n_tiles;
  }
  if (g.d_lrs) cudaFree(g.d_lrs);
  if (g.d_lars_part) cudaFree(g.d_lars_part);
  g.d_lrs = nullptr;
  g.d_lars_part = nullptr;
  CS_CUDA(cudaMalloc(&g.d_lrs, sizeof(float) * (size_t)g.n_loc * n_layers));
  CS_CUDA(cudaMalloc(&g.d_lars_part, sizeof(double) * 2 * (size_t)tiles_for_norms * g.n_loc));
  // the plan and the layer bounds on the device (the single-GPU hierarchical kernel looks them up)
  if (g.d_layer_bounds) cudaFree(g.d_layer_bounds);
  g.d_layer_bounds = nullptr;
  CS_CUDA(cudaMalloc(&g.d_layer_bounds, sizeof(int64_t) * (size_t)(n_layers + 1)));
  CS_CUDA(cudaMemcpy(g.d_layer_bounds, layer_bounds, sizeof(int64_t) * (size_t)(n_layers + 1), cudaMemcpyHostToDevice));
  CS_CUDA(cudaMemcpy(g.d_bounds, g.plan.data(), sizeof(int64_t) * g.plan.size(), cudaMemcpyHostToDevice));
  g.lars_valid = false;
  return CS_OK;
}

int cs_set_lars(float eta, float weight_decay, float eps) {
  if (!g.inited) return fail(CS_ENOTINIT, "cs_init has not been called");
  if (!(eta >= 0.f) || !(weight_decay >= 0.f) || !(eps >= 0.f) || !std::isfinite(eta) ||
      !std::isfinite(weight_decay) || !std::isfinite(eps))
    return fail(CS_EINVAL, "LARS eta, weight_decay, eps must be finite and >= 0");
  g.lars = eta > 0.f;
  g.lars_eta = eta;
  g.lars_wd = weight_decay;
  g.lars_eps = eps;
  return CS_OK;
}

int cs_set_lars_carry(int enable) {
  if (!g.inited) return fail(CS_ENOTINIT, "cs_init has not been called");
  g.lars_carry = enable != 0;
  g.xnorm_valid = false;
  return CS_OK;
}

int cs_params_modified(void) {
  if (!g.inited) return fail(CS_ENOTINIT, "cs_init has not been called");
  g.xnorm_valid = false;
  return CS_OK;
}

int cs_get_lars_rates(float* rates_out) {
  int rc = check_bound();
  if (rc) return rc;
  if (!rates_out) return fail(CS_EINVAL, "NULL rates_out");
  if (!g.lars_valid || !g.d_lrs) return fail(CS_EINVAL, "no LARS step since the layer table was set");
  CS_CUDA(cudaStreamSynchronize(g.stream));
  CS_CUDA(cudaMemcpy(rates_out, g.d_lrs, sizeof(float) * (size_t)g.n_loc * g.n_layers,
                     cudaMemcpyDeviceToHost));
  return poll_device_errors();
}

int cs_accumulate(float* acc, const float* grads, int count, int interval) {
  int rc = check_bound();
  if (rc) return rc;
  if (!acc || !grads) return fail(CS_EINVAL, "NULL acc/grads");
  if (interval < 1 || interval >= (1 << 24))
    return fail(CS_EINVAL, "interval %d outside [1, 2^24)", interval);
  if (count < 0 || count >= interval)
    return fail(CS_EINVAL, "count %d outside [0, interval=%d)", count, interval);
  if (!aligned16(acc) || !aligned16(grads)) return fail(CS_ELAYOUT, "acc and grads must be 16-byte aligned");
  CS_CUDA(launch_accumulate(acc, grads, g.n_loc, g.d, g.ld, count, interval, g.stream));
  return CS_OK;
}

int cs_flush(void) {
  int rc = check_bound();
  if (rc) return rc;
  return flush_pending();
}

int cs_set_step(int64_t step) {
  if (!g.inited) return fail(CS_ENOTINIT, "cs_init has not been called");
  if (step < 0 || step >= (int64_t(1) << 32)) return fail(CS_EINVAL, "step outside [0, 2^32)");
  int rc = flush_pending();
  if (rc) return rc;
  g.xnorm_valid = false;  // resumed parameters: the next LARS step recomputes the x norms
  g.step = step;
  g.peer.need_sync = true;  // resumed state: re-replicate leaders to members on the next hier step
  return CS_OK;
}

int cs_get_step(int64_t* step_out) {
  if (!g.inited) return fail(CS_ENOTINIT, "cs_init has not been called");
  if (!step_out) return fail(CS_EINVAL, "NULL step_out");
  *step_out = g.step;
  return CS_OK;
}

int cs_set_diag(int enable) {
  if (!g.inited) return fail(CS_ENOTINIT, "cs_init has not been called");
  g.diag = enable ? 1 : 0;
  return CS_OK;
}

int cs_get_diag(double* cd_out, double* mean_out) {
  int rc = check_bound();
  if (rc) return rc;
  if (!cd_out || !mean_out) return fail(CS_EINVAL, "NULL output");
  if (!g.diag_valid) return fail(CS_EINVAL, "no step with diagnostics enabled yet");
  double h[2];
  CS_CUDA(cudaMemcpyAsync(h, g.d_diag, sizeof(h), cudaMemcpyDeviceToHost, g.stream));
  CS_CUDA(cudaStreamSynchronize(g.stream));
  rc = poll_device_errors();
  if (rc) return rc;
  *cd_out = h[0];
  *mean_out = h[1];
  return CS_OK;
}

int cs_sync(void) {
  int rc = check_bound();
  if (rc) return rc;
  if ((rc = flush_pending()) != CS_OK) return rc;
  CS_CUDA(cudaStreamSynchronize(g.stream));
  CS_CUDA(cudaGetLastError());
  return poll_device_errors();
}

int cs_test_set_topology(const int32_t* src) {
  int rc = check_bound();
  if (rc) return rc;
  if (src == nullptr) {
    g.has_override = false;
    return CS_OK;
  }
  rc = validate_derangements(src, g.world, g.k);
  if (rc) return rc;
  CS_CUDA(cudaStreamSynchronize(g.stream));
  CS_CUDA(cudaMemcpy(g.d_given, src, sizeof(int32_t) * (size_t)g.k * g.world,
                     cudaMemcpyHostToDevice));
  g.has_override = true;
  return CS_OK;
}

int cs_test_device_topology(int64_t step, int tag, int32_t* src_out) {
  int rc = check_bound();
  if (rc) return rc;
  if (!src_out) return fail(CS_EINVAL, "NULL src_out");
  if (step < 0 || step >= (int64_t(1) << 32)) return fail(CS_EINVAL, "step outside [0, 2^32)");
  const int n = tag == CS_TAG_HIER ? g.groups : g.world;
  TopoArgs t = topo_args(n, tag, nullptr, 1);
  t.step = (uint32_t)step;
  t.rw = nullptr;
  t.inv_wsum = nullptr;
  CS_CUDA(launch_topology(t, g.stream));
  CS_CUDA(cudaMemcpyAsync(src_out, g.d_src, sizeof(int32_t) * (size_t)g.k * n,
                          cudaMemcpyDeviceToHost, g.stream));
  CS_CUDA(cudaStreamSynchronize(g.stream));
  return poll_device_errors();
}

int cs_synth_fill(float* out, int64_t rows, int64_t d, int64_t ld, uint64_t seed, int tag,
                  int64_t row0, float scale) {
  if (!out) return fail(CS_EINVAL, "NULL out");
  if (rows < 0 || d < 0 || ld < d || row0 < 0 || tag < 0)
    return fail(CS_EINVAL, "bad synth shape");
  if (rows == 0 || d == 0) return CS_OK;
  CS_CUDA(launch_synth(out, rows, d, ld, seed, tag, row0, scale, g.bound ? g.stream : nullptr));
  return CS_OK;
}

int cs_step_bytes(int64_t step, int hier, double* out) {
  if (!g.inited) return fail(CS_ENOTINIT, "cs_init has not been called");
  if (!g.bound) return fail(CS_ENOTBOUND, "cs_bind has not been called");
  if (!out) return fail(CS_EINVAL, "NULL out");
  const double d = (double)g.d;
  std::vector<int64_t> b = host_bounds(g.d, g.k);
  if (!hier) {
    // read x, m, g; write x', m'; + LARS norms: x and g (28), or g alone when the previous
    // single-GPU LARS step carried the x norms (24)
    out[0] = (g.lars ? ((g.lars_carry && g.xnorm_valid && !g.use_peer) ? 24.0 : 28.0) : 20.0) * g.n_loc * d;
    std::vector<int32_t> src((size_t)g.k * g.world);
    int rc = cs_topology(step, src.data());
    if (rc) return rc;
    double nvl = 0.0;
    for (int s = 0; s < g.k; ++s)
      for (int i = g.first; i < g.first + g.n_loc; ++i)
        if (src[(size_t)s * g.world + i] / g.n_loc != g.rank)
          nvl += (g.wire == CS_WIRE_BF16 ? 2.0 : 4.0) * (double)(b[s + 1] - b[s]);
    out[1] = nvl;
  } else if (g.nprocs == 1) {
    const int gs = g.world / g.groups;
    const int L_loc = g.n_loc / gs > 0 ? g.n_loc / gs : 1;
    // read members' g, leaders' x and m; write leaders' m and every member's x
    out[0] = (4.0 * g.n_loc + 12.0 * L_loc + 4.0 * g.n_loc) * d;
    out[1] = 0.0;
  } else {
    // one worker per GPU: the group mean needs every member's g (reduce-scatter +
    // all-gather, (gs-1)/gs of 4 B each way), then the leader exchange (4 B per
    // parameter when there are >= 2 groups); HBM as a flat step on the group mean
    // Through the NVSwitch (cs_set_multicast) a GPU takes in its reduced chunk (d/gs) and the
    // other members' mean chunks ((gs-1)/gs of d): 4 B per parameter
    const int gs = g.world / g.groups;
    const double frac = (double)(gs - 1) / (double)gs;
    const bool nvls = g.peer.mc_uc != nullptr && gs > 1 && !g.lars;
    out[0] = 20.0 * d;
    out[1] = (nvls ? 4.0 * d : 2.0 * 4.0 * frac * d) + (g.groups >= 2 ? 4.0 * d : 0.0);
  }
  return CS_OK;
}

int cs_set_timing(int enable) {
  if (!g.inited) return fail(CS_ENOTINIT, "cs_init has not been called");
  if (g.bound) CS_CUDA(cudaStreamSynchronize(g.stream));
  g.timing = enable != 0;
  g.events_used = 0;
  return CS_OK;
}

int cs_get_timing(double* total_ms_out, int64_t* launches_out) {
  if (!g.inited) return fail(CS_ENOTINIT, "cs_init has not been called");
  if (!total_ms_out || !launches_out) return fail(CS_EINVAL, "NULL output");
  double total = 0.0;
  for (size_t i = 0; i + 1 < g.events_used; i += 2) {
    CS_CUDA(cudaEventSynchronize(g.events[i + 1]));
    float ms = 0.f;
    CS_CUDA(cudaEventElapsedTime(&ms, g.events[i], g.events[i + 1]));
    total += ms;
  }
  *total_ms_out = total;
  *launches_out = (int64_t)(g.events_used / 2);
  return CS_OK;
}

const char* cs_kernel_info(int* launches_per_step_out) {
  if (launches_per_step_out) *launches_per_step_out = g.launches_per_step;
  return g.hot_kernel;
}

}  // extern "C"
