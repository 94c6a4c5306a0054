// Stage-replica gradient aggregation (SURVEY.md §8(a) a20, §8(b) spx_comm_*): NCCL communicators
// owned by libspx, one per replicated stage, and an all-reduce that sums a stage's flat fp32
// gradient over the GPUs holding that stage.  NCCL is resolved at run time
// (dlopen, reusing the libnccl.so.2 the process already loaded, e.g. PyTorch's), so libspx still
// loads on a box without NCCL and never links a second copy.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>
#include <mutex>

#include "spx_internal.h"

namespace spx {
namespace {

struct Nccl {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    n.init_rank = reinterpret_cast<decltype(n.init_rank)>(dlsym(h, "ncclCommInitRank"));
    n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(h, "ncclAllReduce"));
    n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(h, "ncclCommDestroy"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
    n.ok = n.get_unique_id && n.init_rank && n.all_reduce && n.destroy && n.error_string;
  });
  return n;
}

int nccl_error(ncclResult_t r, const char* where) {
  char buf[256];
  snprintf(buf, sizeof buf, "%s: %s", where, nccl().error_string ? nccl().error_string(r) : "nccl error");
  return set_error(SPX_ERR_NCCL, buf);
}

}  // namespace
}  // namespace spx

using namespace spx;

extern "C" int spx_comm_unique_id(void* id_out) {
  if (!id_out) return set_error(SPX_ERR_ARG, "comm_unique_id: null output");
  if (!nccl().ok) return set_error(SPX_ERR_NCCL, "comm_unique_id: libnccl.so.2 not found");
  ncclUniqueId id;
  ncclResult_t r = nccl().get_unique_id(&id);
  if (r != ncclSuccess) return nccl_error(r, "ncclGetUniqueId");
  memcpy(id_out, &id, sizeof id);
  return SPX_OK;
}

extern "C" int spx_comm_init(const void* id, int32_t nranks, int32_t rank, void** comm_out) {
  if (!id || !comm_out) return set_error(SPX_ERR_ARG, "comm_init: null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return set_error(SPX_ERR_ARG, "comm_init: need 0 <= rank < nranks");
  if (!nccl().ok) return set_error(SPX_ERR_NCCL, "comm_init: libnccl.so.2 not found");
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof uid);
  ncclComm_t c = nullptr;
  ncclResult_t r = nccl().init_rank(&c, nranks, uid, rank);
  if (r != ncclSuccess) return nccl_error(r, "ncclCommInitRank");
  *comm_out = c;
  return SPX_OK;
}

extern "C" int spx_allreduce(void* comm, void* buf, int64_t count, int32_t dtype, void* stream) {
  if (!comm || (!buf && count > 0)) return set_error(SPX_ERR_ARG, "allreduce: null communicator or buffer");
  if (count < 0) return set_error(SPX_ERR_ARG, "allreduce: negative count");
  ncclDataType_t t;
  if (dtype == SPX_DTYPE_F32) t = ncclFloat32;
  else if (dtype == SPX_DTYPE_BF16) t = ncclBfloat16;
  else return set_error(SPX_ERR_ARG, "allreduce: dtype must be SPX_DTYPE_F32 or SPX_DTYPE_BF16");
  if (!nccl().ok) return set_error(SPX_ERR_NCCL, "allreduce: libnccl.so.2 not found");
  ncclResult_t r = nccl().all_reduce(buf, buf, (size_t)count, t, ncclSum, reinterpret_cast<ncclComm_t>(comm),
                                     reinterpret_cast<cudaStream_t>(stream));
  if (r != ncclSuccess) return nccl_error(r, "ncclAllReduce");
  return SPX_OK;
}

extern "C" int spx_comm_destroy(void* comm) {
  if (!comm) return set_error(SPX_ERR_ARG, "comm_destroy: null communicator");
  if (!nccl().ok) return set_error(SPX_ERR_NCCL, "comm_destroy: libnccl.so.2 not found");
  ncclResult_t r = nccl().destroy(reinterpret_cast<ncclComm_t>(comm));
  if (r != ncclSuccess) return nccl_error(r, "ncclCommDestroy");
  return SPX_OK;
}
