// comm.cpp — NCCL over NVLink / NVSwitch for the multi-GPU distribution:
// one process per GPU, blocks of the P x P temporal structure owned by the cyclic K_P plan,
// partial matrix-vector products summed with one NCCL all-reduce (= reduce-scatter of the
// partial products + all-gather of the result) per product.
// NCCL is loaded at run time (dlopen of the libnccl.so.2 that torch already mapped), so the
// library loads on machines without NCCL and links no second copy.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "internal.h"

namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};
NcclApi g_nccl;
std::once_flag g_nccl_once;
void load_nccl() {
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* n : names) {
    g_nccl.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    if (g_nccl.h) break;
  }
  if (!g_nccl.h) return;
  g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(g_nccl.h, "ncclGetUniqueId");
  g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(g_nccl.h, "ncclCommInitRank");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(g_nccl.h, "ncclCommDestroy");
  g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(g_nccl.h, "ncclAllReduce");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(g_nccl.h, "ncclGetErrorString");
  g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy && g_nccl.AllReduce;
}
bool nccl() {
  std::call_once(g_nccl_once, load_nccl);
  if (!g_nccl.ok) stb::set_error("NCCL (libnccl.so.2) could not be loaded");
  return g_nccl.ok;
}
bem_status nccl_fail(ncclResult_t r, const char* where) {
  stb::set_error(std::string(where) + ": " + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "nccl error"));
  return BEM_E_NCCL;
}
}  // namespace

namespace stb {
bem_status allreduce_sum(const bem_mesh* m, double* buf, long long n, cudaStream_t st) {
  if (!m->comm) return BEM_OK;
  if (!nccl()) return BEM_E_NCCL;
  ncclResult_t r = g_nccl.AllReduce(buf, buf, (size_t)n, ncclDouble, ncclSum, (ncclComm_t)m->comm->nccl, st);
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
  count_launch();
  return BEM_OK;
}
}  // namespace stb

extern "C" {

bem_status bem_nccl_get_unique_id(void* out128) {
  if (!out128) { stb::set_error("bem_nccl_get_unique_id: null"); return BEM_E_INVALID; }
  if (!nccl()) return BEM_E_NCCL;
  ncclUniqueId id;
  ncclResult_t r = g_nccl.GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
  return BEM_OK;
}

bem_status bem_comm_create(const void* id128, int nranks, int rank, int cuda_device, bem_comm** out) {
  if (!id128 || !out || nranks < 1 || rank < 0 || rank >= nranks) { stb::set_error("bem_comm_create: bad argument"); return BEM_E_INVALID; }
  *out = nullptr;
  cudaError_t e = cudaSetDevice(cuda_device);
  if (e != cudaSuccess) return stb::cuda_fail(e, "bem_comm_create/cudaSetDevice");
  bem_comm* c = new bem_comm_s();
  c->nranks = nranks;
  c->rank = rank;
  c->device = cuda_device;
  {   // also for one rank: the distributed code path then runs on a real (1-rank) communicator
    if (!nccl()) { delete c; return BEM_E_NCCL; }
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t comm;
    ncclResult_t r = g_nccl.CommInitRank(&comm, nranks, id, rank);
    if (r != ncclSuccess) { delete c; return nccl_fail(r, "ncclCommInitRank"); }
    c->nccl = comm;
  }
  *out = c;
  return BEM_OK;
}

void bem_comm_destroy(bem_comm* c) {
  if (!c) return;
  if (c->nccl && g_nccl.ok) g_nccl.CommDestroy((ncclComm_t)c->nccl);
  delete c;
}

}  // extern "C"
