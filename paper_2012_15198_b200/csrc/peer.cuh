// Multi-GPU flat step: one process per GPU, workers partitioned contiguously
// (worker w on GPU w / n_loc).  See peer.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace cs {

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
  uint32_t* ord;
  int* err;
};

struct PeerState {
  bool allocated = false;
  bool imported = false;
  int nprocs = 0, rank = 0, n_loc = 0, k = 0;
  int64_t ld = 0;
  int tile = 0;          // elements per tile (multiple of 32)
  int mode = 0;          // CS_PEER_MODE diagnostics: 0 normal, 1 local-only, 2 no waits
  int waves = 0;         // push/mix waves per step
  int per_wave = 0;      // units per CTA per wave
  int algo = 0;          // 0: fused wave kernel; 2: push kernel + mix kernel
  int grid_push = 0, grid_mix = 0;
  size_t off_pdone = 0;  // [nprocs] push-complete epochs (two-kernel schedule)
  size_t off_pcount = 0; // push-kernel CTA arrival counter
  size_t off_wave = 0;   // per-wave arrival counters [waves]
  int n_tiles = 0;
  int grid = 0;
  size_t bytes = 0;
  size_t off_inbox = 0, off_wbox = 0, off_flags = 0, off_done = 0, off_count = 0;
  char* base = nullptr;                 // this GPU's region
  std::vector<char*> peer_base;         // mapped regions of every rank (own at [rank])
  char** d_peer_base = nullptr;         // device copy
  int64_t* d_tiles = nullptr;           // [n_tiles][2]: (segment, start column), end implied
  int64_t* d_tile_end = nullptr;        // [n_tiles]
  int64_t* d_bounds = nullptr;          // [k+1] segment bounds
  int32_t* d_seg_t0 = nullptr;          // [k+1] first tile index of each segment
  uint32_t epoch = 0;                   // multi-GPU steps issued since bind
};

int peer_alloc(PeerState& p, int n_loc, int64_t d, int64_t ld, int k, int nprocs, int rank);
void peer_release(PeerState& p);
int peer_export(PeerState& p, char* handle_out);
int peer_import(PeerState& p, const char* all_handles);
int peer_import_self(PeerState& p);  // nprocs == 1: the only peer is this GPU
int peer_flat_step(PeerState& p, const PeerStepArgs& a, cudaStream_t st, cudaEvent_t ev0,
                   cudaEvent_t ev1);
const char* peer_error();

}  // namespace cs
