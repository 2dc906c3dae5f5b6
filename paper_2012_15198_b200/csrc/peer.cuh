// Multi-GPU steps: one process per GPU, workers partitioned contiguously
// (worker w on GPU w / n_loc), segments exchanged through NVLink peer memory.
// See peer.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace cs {

constexpr int kPeerTile = 2048;   // columns per push unit: 8 KB of one worker's row

// Step schedules of the multi-GPU flat step (cs_set_schedule).
enum { kSchedInStep = 0, kSchedDeferred = 1, kSchedSplit = 2 };

struct PeerStepArgs {
  float* x;
  float* m;
  const float* g;
  float* psw;
  int64_t ld, d, nq;
  int k, world, n_loc, first, rank, nprocs;
  uint32_t step;
  uint64_t seed;
  float lr, mu;
  const int32_t* given;
  int32_t* src;
  int32_t* dst;
  int* err;
  // hierarchical step: groups of gs GPUs (one worker per GPU)
  int groups;     // G; the topology is over the G groups
  int gs;         // GPUs (= workers) per group; 0 for the flat step
  float inv_gs;   // fp32(1/|G|)
  // bf16 wire format (reading C-20): inbox rows hold bf16 with stride (ld + 7) & ~7
  int wire;
  // LARS (reading C-18): per-(local worker, layer) rates of this step, weight decay
  const float* lrs;
  int n_layers;
  float wd;
  // hierarchical LARS: the rates are computed inside peer_hier_step from x and the group
  // mean into lrs_out
  float* lrs_out;
  float eta, eps;
  const int32_t* tile_first;
  double* lars_part;
  // nonzero: g is the rank's own exchange region + g_off (the hierarchical group mean)
  size_t g_off;
  // 1: the hierarchical group mean g is complete on this GPU before the kernel starts
  // (NVLS h1, hier_nvls.cu), so the update does not wait for the reduce flags
  int gbar_local;
  // > 0: pulled group mean (hierarchical h1 without the all-gather): the mean of column c
  // lives only in the gbar row of member c / gpull_chunk of this GPU's group (region + g_off);
  // the update bulk-loads it from there over NVLink
  int64_t gpull_chunk;
  // != 1: g holds the group's gradient SUM (NCCL h1); the update multiplies it by g_scale
  // (fp32(1/|G|), the oracle's final operation of the mean) as it loads it
  float g_scale;
};

struct PeerState {
  bool allocated = false;
  bool imported = false;
  int nprocs = 0, rank = 0, n_loc = 0, k = 0;
  int64_t d = 0, ld = 0;
  int n_tiles = 0;
  int grid_push = 0, grid_mix = 0, grid_hier = 0;
  // single-GPU emulation of the protocol over vranks ranks (one cooperative launch per
  // kernel, CTAs split among the ranks; 1 = a real process per GPU).  nprocs == vranks then.
  int vranks = 1;
  // in-step merge schedule (k_push_merge, one worker per GPU): CTAs per rank and smem
  int sched = kSchedInStep;
  int grid_merge = 0;
  size_t off_mflag = 0, off_hdr = 0;  // per-tile trailers uint4 [2][mflag_cap]; layout header
  unsigned int* d_stats = nullptr;     // [0]: merge tiles re-read after a failed verification
  size_t off_claim = 0;                // chunk claim counters [2] (by epoch parity)
  int mflag_cap = 0;                   // trailer slots per parity (tiles x n_loc)
  int32_t* d_chunk_t0 = nullptr;       // [n_chunks + 1] first tile of each chunk
  int n_chunks = 0;
  int gs = 0;              // hierarchical group size in GPUs (0: flat only)
  int64_t chunk = 0;       // hierarchical reduce-scatter chunk (elements, multiple of 4)
  size_t bytes = 0;
  size_t off_inbox = 0, off_wbox = 0, off_done = 0, off_count = 0;
  size_t off_pdone = 0, off_pcount = 0;                  // push-complete epochs, push arrivals
  size_t off_gbox = 0, off_gbar = 0;                     // hierarchical gradient buffers
  size_t off_d1 = 0, off_c1 = 0, off_d2 = 0, off_c2 = 0; // hierarchical phase epochs / arrivals
  size_t off_xsync = 0, off_msync = 0, off_wsync = 0;    // leader -> member replica sync buffers
  size_t off_d3 = 0, off_c3 = 0;
  bool need_sync = true;   // next hierarchical step first copies each leader's state to its members
  char* base = nullptr;                 // this GPU's region
  std::vector<char*> peer_base;         // mapped regions of every rank (own at [rank])
  char** d_peer_base = nullptr;         // device copy
  int64_t* d_bounds = nullptr;          // [k+1] segment bounds
  int32_t* d_seg_t0 = nullptr;          // [k+1] first tile index of each segment
  uint32_t epoch = 0;                   // multi-GPU steps issued since bind
  // The tiles of a step are cut into `pieces` contiguous ranges; push(p + 1) on the
  // caller's stream overlaps mix(p) on `aux`.  Each piece has its own done / push-done
  // flags ([nprocs] words at off_done / off_pdone + p * flag_stride) and arrival
  // counters (off_count / off_pcount + 64 p).
  static constexpr int kMaxPieces = 8;
  int pieces = 1;
  std::vector<int> piece_tile;          // [pieces + 1] tile boundaries
  std::vector<int64_t> h_bounds;        // host copies of the segment bounds / first tiles
  std::vector<int32_t> h_seg_t0;
  size_t flag_stride = 0;
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_push[kMaxPieces] = {};
  cudaEvent_t ev_mix = nullptr;
  // running totals of CTAs launched against each arrival counter (kernel targets)
  uint32_t tot_count[kMaxPieces] = {}, tot_pcount[kMaxPieces] = {};
  uint32_t tot_c1[kMaxPieces] = {}, tot_c2[kMaxPieces] = {}, tot_c3 = 0;
  int hier_pieces = 1;
  // multi-GPU diagnostics: every GPU owns a column chunk of diag_chunk columns and
  // receives all workers' x' (off_dx, [world][diag_chunk]) and psw (off_dw, [world][k])
  // for it; per-GPU partials (off_dpart, [nprocs][2] fp64) are combined in rank order
  int64_t diag_chunk = 0;
  size_t off_dx = 0, off_dw = 0, off_dpart = 0, off_dd1 = 0, off_dd2 = 0, off_dc1 = 0, off_dc2 = 0;
  uint32_t tot_dc1 = 0, tot_dc2 = 0, diag_epoch = 0;
  // hybrid flat step (several workers per GPU): local cycle walk + NVLink chain heads
  bool use_hybrid = false;
  // deferred merge (CS_PEER_FUSE, default on; push/mix schedule): the merge of step `pending`
  // runs inside the next step's push kernel, or in peer_flush
  bool fuse = false;
  uint32_t pending = 0;
  bool last_fused = false;   // the last flat step ran as one fused push launch
  PeerStepArgs pending_args{};
  // layer table (cs_set_layers, one worker per GPU): explicit tiles split at segment and
  // layer bounds; nullptr = the closed-form equal split of kPeerTile tiles
  struct TileDesc* d_ptiles = nullptr;
  std::vector<int64_t> h_tile_c0;     // [n_tiles + 1] first column of each tile (d at the end)
  int grid_push_max = 0;
  struct TileDesc* d_htiles = nullptr;
  int n_htiles = 0, grid_hyb = 0, grid_tail = 0;
  uint8_t* d_tail_tbl = nullptr;
  // NVLS h1 (hier_nvls.cu): the caller's multicast workspace of this GPU's group (unicast and
  // multicast views, cs_set_multicast) and multicast-bound gradient regions it registered
  char* mc_uc = nullptr;
  char* mc_mc = nullptr;
  size_t mc_bytes = 0;
  struct McRegion { char* uc; char* mc; size_t bytes; };
  std::vector<McRegion> mc_grads;
  uint32_t* d_nvls_count = nullptr;   // local arrival counters [2] at 64-byte stride
  uint32_t nvls_epoch = 0;
  uint32_t nvls_tot[2] = {0, 0};
  bool last_nvls = false;   // the last hierarchical step's h1 ran through NVLS
  // NCCL h1 (hier_nccl.cu): a communicator over this GPU's hierarchical group (cs_set_hier_nccl)
  void* nccl_comm = nullptr;
  bool last_nccl = false;
};

// NCCL h1 (hier_nccl.cu; NCCL loaded at run time)
int nccl_unique_id(char* out /* 128 bytes */);
int nccl_group_init(PeerState& p, const char* id_bytes /* nullptr: release */, int member);
void nccl_group_release(PeerState& p);
int nccl_h1(PeerState& p, const float* g, float* gsum, int64_t d, cudaStream_t st);
const char* nccl_error();

// kernels the multi-GPU steps launched (plaunch / peer_launch / topology / NVLS): the
// bench's launch count is the difference across a step
extern long g_peer_launches;

// NVLS h1 (hier_nvls.cu)
size_t nvls_off_gbar();
size_t nvls_bytes(int64_t ld);
// g_mc: multicast address of g when g lies in a registered multicast region, else nullptr
// (the kernel stages g into the workspace first)
int nvls_h1(PeerState& p, const float* g, const float* g_mc, int member, float inv_gs, int* err, cudaStream_t st);

// gs: GPUs per hierarchical group when a hierarchical step is possible (one worker
// per GPU and groups < world), else 0.
int peer_alloc(PeerState& p, int n_loc, int64_t d, int64_t ld, int k, int nprocs, int rank, int gs, int vranks = 1);
void peer_release(PeerState& p);
int peer_export(PeerState& p, char* handle_out);
int peer_import(PeerState& p, const char* all_handles);
int peer_import_self(PeerState& p);  // nprocs == 1: the only peer is this GPU
int peer_flat_step(PeerState& p, const PeerStepArgs& a, cudaStream_t st, cudaEvent_t ev0,
                   cudaEvent_t ev1);
// Layer table on the push/mix path: tiles split at the plan's segment bounds and the layer
// bounds.  Returns the tile range of each layer in tile_first [n_layers + 1].  Empty
// layer_bounds restores the equal split.
int peer_set_layers(PeerState& p, const std::vector<int64_t>& plan, const std::vector<int64_t>& layer_bounds,
                    std::vector<int32_t>& tile_first);
const struct TileDesc* peer_tiles(const PeerState& p);
int peer_tile_count(const PeerState& p);
// Completes a deferred merge (no-op if none is pending).
int peer_flush(PeerState& p, cudaStream_t st);
// Schedule of later flat steps (cs_set_schedule); completes a pending deferred merge first.
int peer_set_schedule(PeerState& p, int sched, cudaStream_t st);
// One flat step whose merge completes inside the step's own kernel (k_push_merge; one
// worker per GPU).  hier: the leader exchange of a hierarchical step (g = group mean).
int peer_merge_launch(PeerState& p, const PeerStepArgs& a, uint32_t epoch, cudaStream_t st);
bool peer_merge_ok(const PeerState& p, const PeerStepArgs& a);
size_t peer_merge_smem(int k, int n_loc);
std::vector<int32_t> peer_merge_chunks(const std::vector<int32_t>& seg_t0, int chunk, int grid);
constexpr int kMergeChunk = 4;    // tiles per claimed chunk (one landed flag and release each)
int peer_merge_capacity(int k);   // co-resident k_push_merge CTAs on this GPU
// launch helper: plain launch, or a cooperative one over all emulated ranks
cudaError_t peer_launch(const PeerState& p, const void* fn, int grid_per_rank, int threads, size_t smem,
                        cudaStream_t st, void** args);
int peer_hier_step(PeerState& p, const PeerStepArgs& a, cudaStream_t st, cudaEvent_t ev0,
                   cudaEvent_t ev1);
// diagnostics of the current state (after a step), all GPUs; out: device double[2]
int peer_diag(PeerState& p, const PeerStepArgs& a, double* partials, int partials_cap, double* out,
              cudaStream_t st);
const char* peer_error();

}  // namespace cs
