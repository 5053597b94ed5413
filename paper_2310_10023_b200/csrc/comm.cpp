// comm.cpp — NCCL communicator of a sharded search.
//
// The multi-GPU exchanges of a sharded search (incumbent max-all-reduce every
// epoch; in the batch-split exact mode also the root scores once and every
// flush's scores) are enqueued on the search stream as ncclAllReduce(MAX)
// calls over NVLink / NVSwitch: no host round-trip per epoch, and the epochs
// stay capturable into the batch CUDA graph.
//
// NCCL is dlopen'ed ("libnccl.so.2") on first use instead of linked: inside a
// torch process this resolves to the NCCL torch already loaded (one NCCL per
// process), and the library still loads on machines without NCCL (only
// bbs_comm_* then fail, with BBS_ERR_CUDA).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "bbs_comm.h"
#include "bbs_internal.h"

namespace bbs {
namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
  bool ok = false;
  std::string why;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.why = std::string("NCCL not found: ") + (e ? e : "dlopen failed");
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.get_version = reinterpret_cast<decltype(api.get_version)>(dlsym(h, "ncclGetVersion"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce &&
             api.error_string;
    if (!api.ok) api.why = "NCCL library lacks a required symbol";
  });
  return api;
}

const NcclApi& require() {
  const NcclApi& a = nccl();
  if (!a.ok) throw Error(BBS_ERR_CUDA, a.why);
  return a;
}

void check(const NcclApi& a, ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(BBS_ERR_CUDA, std::string(what) + ": " + (a.error_string ? a.error_string(r) : "nccl error"));
}

}  // namespace

void comm_unique_id(uint8_t out[128]) {
  const NcclApi& a = require();
  ncclUniqueId id;
  check(a, a.get_unique_id(&id), "ncclGetUniqueId");
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out, &id, sizeof(id));
}

Comm* comm_create(int device, int rank, int world, const uint8_t id[128]) {
  const NcclApi& a = require();
  if (world < 1 || rank < 0 || rank >= world) throw Error(BBS_ERR_CONFIG, "comm: rank out of range");
  int prev = 0;
  BBS_CUDA(cudaGetDevice(&prev));
  BBS_CUDA(cudaSetDevice(device));
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  const ncclResult_t r = a.comm_init_rank(&c, world, uid, rank);
  cudaSetDevice(prev);
  check(a, r, "ncclCommInitRank");
  Comm* out = new Comm;
  out->nccl = c;
  out->device = device;
  out->rank = rank;
  out->world = world;
  return out;
}

void comm_destroy(Comm* c) {
  if (!c) return;
  const NcclApi& a = nccl();
  if (a.ok && c->nccl) a.comm_destroy(static_cast<ncclComm_t>(c->nccl));
  delete c;
}

void comm_allreduce_max_i32(Comm* c, int32_t* d, size_t n, cudaStream_t s) {
  if (n == 0) return;
  const NcclApi& a = require();
  check(a, a.all_reduce(d, d, n, ncclInt32, ncclMax, static_cast<ncclComm_t>(c->nccl), s),
        "ncclAllReduce");
}

int comm_nccl_version() {
  const NcclApi& a = nccl();
  int v = 0;
  if (a.ok && a.get_version) a.get_version(&v);
  return v;
}

}  // namespace bbs
