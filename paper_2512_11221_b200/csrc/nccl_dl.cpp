// paper_2512_11221_b200/csrc/nccl_dl.cpp — NCCL for the head-sharded mode, loaded with dlopen so
// that libasr.so has no link-time dependency on it (the torch wheel ships libnccl.so.2).
#include <dlfcn.h>
#include <nccl.h>

#include "asr_internal.h"

namespace asr {
namespace {

decltype(&ncclGetUniqueId) p_uid = nullptr;
decltype(&ncclCommInitRank) p_init = nullptr;
decltype(&ncclAllReduce) p_allreduce = nullptr;
decltype(&ncclCommDestroy) p_destroy = nullptr;
decltype(&ncclGetErrorString) p_err = nullptr;

int w_uid(void* out) { return (int)p_uid(reinterpret_cast<ncclUniqueId*>(out)); }
int w_init(void** comm, int nranks, const void* id, int rank) {
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  return (int)p_init(reinterpret_cast<ncclComm_t*>(comm), nranks, u, rank);
}
int w_allreduce(const void* send, void* recv, size_t count, int dtype, int op, void* comm, cudaStream_t st) {
  return (int)p_allreduce(send, recv, count, (ncclDataType_t)dtype, (ncclRedOp_t)op, (ncclComm_t)comm, st);
}
int w_destroy(void* comm) { return (int)p_destroy((ncclComm_t)comm); }
const char* w_err(int rc) { return p_err((ncclResult_t)rc); }

NcclApi load() {
  NcclApi a;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return a;
  p_uid = (decltype(p_uid))dlsym(h, "ncclGetUniqueId");
  p_init = (decltype(p_init))dlsym(h, "ncclCommInitRank");
  p_allreduce = (decltype(p_allreduce))dlsym(h, "ncclAllReduce");
  p_destroy = (decltype(p_destroy))dlsym(h, "ncclCommDestroy");
  p_err = (decltype(p_err))dlsym(h, "ncclGetErrorString");
  if (!p_uid || !p_init || !p_allreduce || !p_destroy || !p_err) return a;
  a.ok = true;
  a.get_unique_id = w_uid;
  a.comm_init_rank = w_init;
  a.all_reduce = w_allreduce;
  a.comm_destroy = w_destroy;
  a.get_error = w_err;
  return a;
}

}  // namespace

NcclApi& nccl_api() {
  static NcclApi api = load();
  return api;
}

}  // namespace asr
