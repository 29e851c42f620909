// Multi-GPU collectives of the sharded operator.
//
// One process per GPU.  The library owns an NCCL communicator per sharded handle, created from a
// unique id the caller distributes (torch.distributed is plumbing only), and enqueues the two
// collectives of an operator application -- the reduce-scatter of the symmetric K1 partial sums
// and the all-gather of the owned rows -- on the handle's stream: no host synchronisation, no
// callback.  NCCL is resolved at run time with dlopen (the copy torch already loaded when there
// is one), so libbpqn has no link-time NCCL dependency and a missing NCCL is an error only for
// the calls that need it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "bpqn_internal.h"

namespace bpqn {

struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*reduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
  std::string why;
};

static NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's NCCL (torch's), if loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("NCCL not found: ") + (dlerror() ? dlerror() : "");
      return;
    }
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(h, "ncclAllGather"));
    api.reduceScatter = reinterpret_cast<decltype(api.reduceScatter)>(dlsym(h, "ncclReduceScatter"));
    api.errorString = reinterpret_cast<decltype(api.errorString)>(dlsym(h, "ncclGetErrorString"));
    if (!api.getUniqueId || !api.commInitRank || !api.commDestroy || !api.allGather || !api.reduceScatter)
      api.why = "NCCL library lacks a required symbol";
  });
  if (!api.why.empty()) throw Error{BPQN_ERR_CUDA, api.why};
  return api;
}

#define BPQN_NCCL(call)                                                                             \
  do {                                                                                              \
    ncclResult_t r_ = (call);                                                                       \
    if (r_ != ncclSuccess)                                                                          \
      throw ::bpqn::Error{BPQN_ERR_CUDA, std::string(#call) + ": " +                                \
                                             (nccl().errorString ? nccl().errorString(r_) : "error")}; \
  } while (0)

void comm_unique_id(void* out128) {
  ncclUniqueId id;
  BPQN_NCCL(nccl().getUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
}

void comm_destroy(Geom& g) {
  if (!g.nccl_comm) return;
  nccl().commDestroy(static_cast<ncclComm_t>(g.nccl_comm));
  g.nccl_comm = nullptr;
}

// Create this rank's communicator (collective over the `world` ranks that call it with the same id)
// and the library-owned exchange buffers: all-gather [world][rows][3], reduce-scatter send
// [world][rows][3] and receive [rows][3].
void comm_init(Geom& g, int rank, int world, const void* uid128) {
  comm_destroy(g);
  ncclUniqueId id;
  std::memcpy(&id, uid128, sizeof(id));
  ncclComm_t c = nullptr;
  BPQN_NCCL(nccl().commInitRank(&c, world, id, rank));
  g.nccl_comm = c;
  const size_t rows = (size_t)((g.np + world - 1) / world) * g.nq;
  g.sh_own_send.ensure(3 * rows);
  g.sh_own_recv.ensure(3 * rows * world);
  g.sh_own_rs_send.ensure(3 * rows * world);
  g.sh_own_rs_recv.ensure(3 * rows);
}

void comm_allgather(Geom& g, const double* send, double* recv, size_t count, cudaStream_t st) {
  BPQN_NCCL(nccl().allGather(send, recv, count, ncclFloat64, static_cast<ncclComm_t>(g.nccl_comm), st));
}

void comm_reduce_scatter(Geom& g, const double* send, double* recv, size_t count, cudaStream_t st) {
  BPQN_NCCL(nccl().reduceScatter(send, recv, count, ncclFloat64, ncclSum, static_cast<ncclComm_t>(g.nccl_comm), st));
}

}  // namespace bpqn
