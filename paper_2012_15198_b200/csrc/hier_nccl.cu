// Hierarchical h1 through NCCL: the intra-group gradient sum of PAPER.md:197 (§3.3 "reduce
// the gradients in each group"; reading C-12) as ncclAllReduce over a communicator of the
// group's GPUs -- the library north_star names for the intra-group average ("NCCL over
// NVLink is used only for the intra-group average of hierarchical mode").  The update
// kernels then scale the sum by fp32(1/|G|) as they load it (the oracle's final operation);
// NCCL's summation order differs from the oracle's ascending order, so groups of >= 3 GPUs
// match within the hierarchical tolerance, groups of 2 bitwise.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2"): in a PyTorch process that is the NCCL
// torch already loaded; otherwise the system's.  Only the five entry points below are used.
#include <dlfcn.h>
#include <nccl.h>
#include <stdio.h>
#include <string.h>

#include "peer.cuh"

namespace cs {

namespace {

struct NcclApi {
  bool loaded = false;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) =
      nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi g_nccl;
char g_nccl_err[256] = {0};

bool load_nccl() {
  if (g_nccl.loaded) return true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    snprintf(g_nccl_err, sizeof(g_nccl_err), "dlopen libnccl.so.2: %s", dlerror());
    return false;
  }
  g_nccl.get_unique_id = reinterpret_cast<decltype(g_nccl.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
  g_nccl.comm_init_rank = reinterpret_cast<decltype(g_nccl.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
  g_nccl.comm_destroy = reinterpret_cast<decltype(g_nccl.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
  g_nccl.all_reduce = reinterpret_cast<decltype(g_nccl.all_reduce)>(dlsym(h, "ncclAllReduce"));
  g_nccl.error_string = reinterpret_cast<decltype(g_nccl.error_string)>(dlsym(h, "ncclGetErrorString"));
  if (!g_nccl.get_unique_id || !g_nccl.comm_init_rank || !g_nccl.comm_destroy || !g_nccl.all_reduce ||
      !g_nccl.error_string) {
    snprintf(g_nccl_err, sizeof(g_nccl_err), "libnccl.so.2 lacks an entry point");
    return false;
  }
  g_nccl.loaded = true;
  return true;
}

const char* nccl_msg(ncclResult_t r) { return g_nccl.error_string ? g_nccl.error_string(r) : "?"; }

}  // namespace

const char* nccl_error() { return g_nccl_err; }

int nccl_unique_id(char* out) {
  if (!load_nccl()) return -1;
  ncclUniqueId id;
  const ncclResult_t r = g_nccl.get_unique_id(&id);
  if (r != ncclSuccess) {
    snprintf(g_nccl_err, sizeof(g_nccl_err), "ncclGetUniqueId: %s", nccl_msg(r));
    return -1;
  }
  memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return 0;
}

int nccl_group_init(PeerState& p, const char* id_bytes, int member) {
  nccl_group_release(p);
  if (!id_bytes) return 0;  // disable
  if (!load_nccl()) return -1;
  ncclUniqueId id;
  memcpy(id.internal, id_bytes, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t comm = nullptr;
  const ncclResult_t r = g_nccl.comm_init_rank(&comm, p.gs, id, member);
  if (r != ncclSuccess) {
    snprintf(g_nccl_err, sizeof(g_nccl_err), "ncclCommInitRank(%d of %d): %s", member, p.gs, nccl_msg(r));
    return -1;
  }
  p.nccl_comm = comm;
  return 0;
}

void nccl_group_release(PeerState& p) {
  if (p.nccl_comm && g_nccl.loaded) g_nccl.comm_destroy(static_cast<ncclComm_t>(p.nccl_comm));
  p.nccl_comm = nullptr;
}

int nccl_h1(PeerState& p, const float* g, float* gsum, int64_t d, cudaStream_t st) {
  const ncclResult_t r = g_nccl.all_reduce(g, gsum, (size_t)d, ncclFloat32, ncclSum,
                                           static_cast<ncclComm_t>(p.nccl_comm), st);
  if (r != ncclSuccess) {
    snprintf(g_nccl_err, sizeof(g_nccl_err), "ncclAllReduce: %s", nccl_msg(r));
    return -1;
  }
  return 0;
}

}  // namespace cs
