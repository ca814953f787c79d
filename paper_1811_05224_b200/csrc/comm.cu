// comm.cpp — collectives for the multi-GPU distribution: one process per GPU, blocks
// of the P x P temporal structure owned by the cyclic K_P plan, partial matrix-vector products
// summed with one all-reduce (= reduce-scatter of the partial products + all-gather of the result)
// per product.
//   * NCCL over NVLink / NVSwitch (bem_comm_create).  NCCL is loaded at run time (dlopen of the
//     libnccl.so.2 that torch already mapped), so the library loads on machines without NCCL and
//     links no second copy.  The collectives run on the communicator's own stream so that a
//     product's all-reduce of one row chunk overlaps the GEMV of the next (linalg.cu); host waits
//     poll ncclCommGetAsyncError and abort the communicator on an error.
//   * Emulated ranks on ONE device (bem_comm_create_group, tests): the ranks are host threads; an
//     all-reduce synchronises the rank's stream, meets the other ranks at a host barrier, sums all
//     ranks' buffers in rank order with a kernel (every rank the same sum: identical results, as
//     NCCL gives) and copies it back after a second barrier.  No kernel ever waits on another
//     rank's kernel (B200_PROFILING.md: ranks whose kernels wait on one another must not share a
//     GPU), so the emulation cannot deadlock the device.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>

#include "internal.h"

namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
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
  g_nccl.CommAbort = (decltype(g_nccl.CommAbort))dlsym(g_nccl.h, "ncclCommAbort");
  g_nccl.CommGetAsyncError = (decltype(g_nccl.CommGetAsyncError))dlsym(g_nccl.h, "ncclCommGetAsyncError");
  g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(g_nccl.h, "ncclAllReduce");
  g_nccl.AllGather = (decltype(g_nccl.AllGather))dlsym(g_nccl.h, "ncclAllGather");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(g_nccl.h, "ncclGetErrorString");
  g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy && g_nccl.AllReduce && g_nccl.AllGather;
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
thread_local stb::CommTimer* t_timer = nullptr;
double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

namespace stb {

// ------------------------------------------------------------------ emulated ranks (one device)
constexpr int GROUP_MAX = 16;
struct CommGroup {
  int n = 0, device = 0, alive = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  double* bufs[GROUP_MAX] = {nullptr};
  // false after 300 s without the other ranks (a rank that stopped calling the collectives)
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    return cv.wait_for(lk, std::chrono::seconds(300), [&] { return gen != g; });
  }
};
struct Ptrs {
  const double* p[GROUP_MAX];
};
// out = sum_r bufs[r], r = 0 .. n-1 in rank order (the same doubles on every rank)
__global__ void k_group_sum(Ptrs b, int n, long long len, double* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= len) return;
  double s = 0.0;
  for (int r = 0; r < n; ++r) s += b.p[r][i];
  out[i] = s;
}

static bem_status group_allreduce(bem_comm* c, double* buf, long long n, cudaStream_t st) {
  CommGroup* G = c->group;
  const double t0 = now_s();
  double* tmp = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&tmp, sizeof(double) * (size_t)std::max<long long>(1, n), st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);          // this rank's partial sums are complete
  if (e != cudaSuccess) return cuda_fail(e, "group all-reduce");
  G->bufs[c->rank] = buf;
  if (!G->barrier()) {                                           // every rank's partials are complete
    cudaFreeAsync(tmp, st);
    set_error("emulated-rank all-reduce: the other ranks did not arrive (300 s)");
    return BEM_E_STATE;
  }
  Ptrs P;
  for (int r = 0; r < G->n; ++r) P.p[r] = G->bufs[r];
  if (n > 0) k_group_sum<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(P, G->n, n, tmp);
  count_launch();
  e = cudaStreamSynchronize(st);
  if (!G->barrier()) {                                           // nobody reads the partials any more
    cudaFreeAsync(tmp, st);
    set_error("emulated-rank all-reduce: the other ranks did not arrive (300 s)");
    return BEM_E_STATE;
  }
  if (e == cudaSuccess && n > 0) e = cudaMemcpyAsync(buf, tmp, sizeof(double) * n, cudaMemcpyDeviceToDevice, st);
  cudaFreeAsync(tmp, st);
  if (t_timer) t_timer->host_s += now_s() - t0;
  return e == cudaSuccess ? BEM_OK : cuda_fail(e, "group all-reduce");
}

// in-place all-gather over the emulated ranks: each rank copies the other ranks' chunks into its
// own buffer between two barriers (every chunk complete before; nobody reads after)
static bem_status group_allgather(bem_comm* c, double* buf, long long chunk, cudaStream_t st) {
  CommGroup* G = c->group;
  const double t0 = now_s();
  cudaError_t e = cudaStreamSynchronize(st);                      // this rank's chunk is complete
  if (e != cudaSuccess) return cuda_fail(e, "group all-gather");
  G->bufs[c->rank] = buf;
  if (!G->barrier()) {
    set_error("emulated-rank all-gather: the other ranks did not arrive (300 s)");
    return BEM_E_STATE;
  }
  for (int r = 0; r < G->n && e == cudaSuccess; ++r)
    if (r != c->rank && chunk > 0)
      e = cudaMemcpyAsync(buf + r * chunk, G->bufs[r] + r * chunk, sizeof(double) * chunk, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (!G->barrier()) {
    set_error("emulated-rank all-gather: the other ranks did not arrive (300 s)");
    return BEM_E_STATE;
  }
  if (t_timer) t_timer->host_s += now_s() - t0;
  return e == cudaSuccess ? BEM_OK : cuda_fail(e, "group all-gather");
}

// ------------------------------------------------------------------ NCCL
static bem_status nccl_check(bem_comm* c) {
  if (!c || !c->nccl) return BEM_OK;
  if (c->failed) { set_error("NCCL communicator aborted after an asynchronous error"); return BEM_E_NCCL; }
  if (!g_nccl.CommGetAsyncError) return BEM_OK;
  ncclResult_t ar = ncclSuccess;
  ncclResult_t r = g_nccl.CommGetAsyncError((ncclComm_t)c->nccl, &ar);
  if (r == ncclSuccess && (ar == ncclSuccess || ar == ncclInProgress)) return BEM_OK;
  // an asynchronous error (a failed peer, a network error): abort so that no rank blocks forever
  c->failed = true;
  if (g_nccl.CommAbort) g_nccl.CommAbort((ncclComm_t)c->nccl);
  return nccl_fail(r != ncclSuccess ? r : ar, "NCCL asynchronous error (communicator aborted)");
}

bem_status comm_wait_event(const bem_mesh* m, cudaEvent_t ev) {
  bem_comm* c = m ? m->comm : nullptr;
  if (!c || !c->nccl) {
    cudaError_t e = cudaEventSynchronize(ev);
    return e == cudaSuccess ? BEM_OK : cuda_fail(e, "event wait");
  }
  for (int spin = 0;; ++spin) {
    cudaError_t e = cudaEventQuery(ev);
    if (e == cudaSuccess) return BEM_OK;
    if (e != cudaErrorNotReady) return cuda_fail(e, "event wait");
    if ((spin & 63) == 0) {
      bem_status s = nccl_check(c);
      if (s != BEM_OK) return s;
    }
    if (spin > 256) std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

static void timer_mark(cudaStream_t st) {
  if (!t_timer) return;
  cudaEvent_t x;
  if (cudaEventCreate(&x) != cudaSuccess) { cudaGetLastError(); return; }
  cudaEventRecord(x, st);
  t_timer->ev.push_back(x);
}

static bem_status nccl_allreduce(bem_comm* c, double* buf, long long n, cudaStream_t st) {
  if (!nccl()) return BEM_E_NCCL;
  bem_status s = nccl_check(c);
  if (s != BEM_OK) return s;
  timer_mark(st);
  ncclResult_t r = g_nccl.AllReduce(buf, buf, (size_t)n, ncclDouble, ncclSum, (ncclComm_t)c->nccl, st);
  timer_mark(st);
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
  count_launch();
  return BEM_OK;
}

bem_status allreduce_sum(const bem_mesh* m, double* buf, long long n, cudaStream_t st) {
  bem_comm* c = m->comm;
  if (!c || c->solo) return BEM_OK;   // solo rank: its partial sums stay as they are
  if (c->group) return group_allreduce(c, buf, n, st);
  return nccl_allreduce(c, buf, n, st);
}

int record_ranks(const bem_mesh* m) {
  const bem_comm* c = m->comm;
  return (!c || c->solo) ? 1 : c->nranks;
}

bem_status allgather_chunks(const bem_mesh* m, double* buf, long long chunk, cudaStream_t st) {
  bem_comm* c = m->comm;
  if (!c || c->solo || c->nranks == 1) return BEM_OK;
  if (c->group) return group_allgather(c, buf, chunk, st);
  if (!nccl()) return BEM_E_NCCL;
  bem_status s = nccl_check(c);
  if (s != BEM_OK) return s;
  timer_mark(st);
  // in place: the send buffer is the rank's own slot of the receive buffer
  ncclResult_t r = g_nccl.AllGather(buf + (long long)c->rank * chunk, buf, (size_t)chunk, ncclDouble,
                                    (ncclComm_t)c->nccl, st);
  timer_mark(st);
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
  count_launch();
  return BEM_OK;
}

bool comm_overlaps(const bem_mesh* m) { return m->comm && m->comm->nccl && m->comm->stream; }

bem_status allreduce_sum_async(const bem_mesh* m, double* buf, long long n, cudaStream_t st, cudaEvent_t ready) {
  if (!comm_overlaps(m)) return allreduce_sum(m, buf, n, st);
  bem_comm* c = m->comm;
  cudaStreamWaitEvent(c->stream, ready, 0);
  return nccl_allreduce(c, buf, n, c->stream);
}

bem_status comm_join(const bem_mesh* m, cudaStream_t st) {
  if (!comm_overlaps(m)) return BEM_OK;
  cudaEvent_t x;
  cudaError_t e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(x, m->comm->stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st, x, 0);
  cudaEventDestroy(x);
  return e == cudaSuccess ? BEM_OK : cuda_fail(e, "comm join");
}

void comm_timer_set(CommTimer* t) { t_timer = t; }

double comm_timer_seconds(CommTimer* t) {
  if (!t) return 0.0;
  double s = t->host_s;
  for (size_t k = 0; k + 1 < t->ev.size(); k += 2) {
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, t->ev[k], t->ev[k + 1]) == cudaSuccess) s += 1e-3 * ms;
  }
  for (auto x : t->ev) cudaEventDestroy(x);
  t->ev.clear();
  cudaGetLastError();
  return s;
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
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    c->stream = nullptr;   // collectives then run on the caller's stream (no overlap)
  }
  *out = c;
  return BEM_OK;
}

bem_status bem_comm_create_group(int nranks, int cuda_device, bem_comm** out) {
  if (!out || nranks < 1 || nranks > stb::GROUP_MAX) { stb::set_error("bem_comm_create_group: 1 <= nranks <= 16"); return BEM_E_INVALID; }
  cudaError_t e = cudaSetDevice(cuda_device);
  if (e != cudaSuccess) return stb::cuda_fail(e, "bem_comm_create_group/cudaSetDevice");
  stb::CommGroup* G = new stb::CommGroup();
  G->n = nranks;
  G->device = cuda_device;
  G->alive = nranks;
  for (int r = 0; r < nranks; ++r) {
    bem_comm* c = new bem_comm_s();
    c->nranks = nranks;
    c->rank = r;
    c->device = cuda_device;
    c->group = G;
    out[r] = c;
  }
  return BEM_OK;
}

bem_status bem_comm_create_solo(int nranks, int rank, int cuda_device, bem_comm** out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks) { stb::set_error("bem_comm_create_solo: bad argument"); return BEM_E_INVALID; }
  cudaError_t e = cudaSetDevice(cuda_device);
  if (e != cudaSuccess) return stb::cuda_fail(e, "bem_comm_create_solo/cudaSetDevice");
  bem_comm* c = new bem_comm_s();
  c->nranks = nranks;
  c->rank = rank;
  c->device = cuda_device;
  c->solo = true;
  *out = c;
  return BEM_OK;
}

void bem_comm_destroy(bem_comm* c) {
  if (!c) return;
  if (c->nccl && g_nccl.ok) {
    if (c->failed) { /* already aborted */ }
    else g_nccl.CommDestroy((ncclComm_t)c->nccl);
  }
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->group) {
    stb::CommGroup* G = c->group;
    bool last;
    {
      std::lock_guard<std::mutex> lk(G->mu);
      last = --G->alive == 0;
    }
    if (last) delete G;
  }
  delete c;
}

}  // extern "C"
