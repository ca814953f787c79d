// api.cpp — C-ABI entry points (include/stbem.h): assembly drivers, products, preconditioned
// GMRES, matrix access.  Host orchestration only: every arithmetic
// step on vectors or matrices runs in the CUDA kernels of assemble.cu / linalg.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <mutex>
#include <cstring>
#include <vector>

#include "internal.h"

using namespace stb;

namespace stb {

// ---------------------------------------------------------------- matrix storage cache
// Dense matrix storage (tens of GB per matrix) is kept by the library when a matrix is destroyed
// and handed to the next assembly of a size that fits (at most 25% larger): repeated solves then
// neither map new physical memory nor depend on the stream-ordered pool's fragmentation (which
// cost a 65-130 ms stall about once per five C3 steps).  Reuse is stream-ordered: the destroy
// records an event on the matrix's stream and the next user's stream waits on it.
// bem_release_storage() returns the cached blocks to the device pool.
struct CachedBlock {
  void* ptr;
  size_t bytes;
  cudaEvent_t freed;
};
static std::mutex g_cache_mu;
static std::vector<CachedBlock> g_cache[64];

static bool g_pool_ready[64] = {false};
bool pool_ready(int device) { return g_pool_ready[device & 63]; }

void pool_setup(int device) {
  bool* ready = g_pool_ready;
  if (ready[device & 63]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    unsigned long long thr = ~0ULL;   // keep freed pool memory mapped (no re-mapping cost)
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  ready[device & 63] = true;
}

constexpr size_t CACHE_MIN_BYTES = 1 << 20;

cudaError_t storage_acquire(int device, size_t bytes, cudaStream_t st, void** out) {
  pool_setup(device);
  if (bytes < CACHE_MIN_BYTES) return cudaMallocAsync(out, bytes, st);
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto& c = g_cache[device & 63];
    int best = -1;
    for (int k = 0; k < (int)c.size(); ++k)
      if (c[k].bytes >= bytes && c[k].bytes <= bytes + bytes / 4 && (best < 0 || c[k].bytes < c[best].bytes)) best = k;
    if (best >= 0) {
      CachedBlock b = c[best];
      c.erase(c.begin() + best);
      cudaStreamWaitEvent(st, b.freed, 0);
      cudaEventDestroy(b.freed);
      *out = b.ptr;
      return cudaSuccess;
    }
  }
  cudaError_t e = cudaMallocAsync(out, bytes, st);
  if (e == cudaErrorMemoryAllocation) {
    // release the cache to the pool and retry once
    cudaGetLastError();
    bem_release_storage();
    e = cudaMallocAsync(out, bytes, st);
  }
  return e;
}

void storage_release(int device, void* ptr, size_t bytes, cudaStream_t st) {
  if (!ptr) return;
  if (bytes < CACHE_MIN_BYTES) {
    cudaFreeAsync(ptr, st);
    return;
  }
  cudaEvent_t ev;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess || cudaEventRecord(ev, st) != cudaSuccess) {
    cudaGetLastError();
    cudaFreeAsync(ptr, st);
    return;
  }
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_cache[device & 63].push_back({ptr, bytes, ev});
}

}  // namespace stb

namespace {

inline cudaStream_t S(bem_stream s) { return reinterpret_cast<cudaStream_t>(s); }

bem_matrix* new_dense(const bem_mesh* m, int kind, bool sym, cudaStream_t stream, bem_status* st,
                      bool toeplitz = false) {
  bem_matrix* A = new bem_matrix_s();
  A->kind = kind;
  A->mesh = m;
  A->stream = stream;
  if (toeplitz) {
    // the first block column: T_d = A(d, 0), d = 0 .. N_I - 1 (one temporal "block" (a in [0, N_I),
    // b in [0, 1)) of the assembly machinery)
    A->toeplitz = 1;
    Block b;
    b.I = b.J = 0;
    b.a0 = 0; b.a1 = m->nt; b.b0 = 0; b.b1 = 1;
    b.off = 0;
    A->own_blocks.push_back(b);
    sym = false;
  }
  A->sym = sym ? 1 : 0;
  const int ng = m->ng;
  A->blk_elems = sym ? sym_blk_elems(ng) : 0;
  long long off = 0;
  for (size_t bi = 0; bi < blocks_of(A).size(); ++bi) {
    const Block& b = blocks_of(A)[bi];
    A->poff_base.push_back((int)A->poff.size());
    for (int a = b.a0; a < b.a1; ++a) {
      A->poff.push_back(off);
      off += sym ? (long long)panel_nb(a, b.b0, b.b1) * A->blk_elems
                 : (long long)ng * pad4((long long)panel_nb(a, b.b0, b.b1) * ng);
    }
  }
  A->entries = off;
  const size_t bytes = sizeof(double) * std::max<long long>(off, 4);
  cudaError_t e = storage_acquire(m->device, bytes, stream, (void**)&A->data);
  if (e != cudaSuccess) {
    *st = BEM_E_NOMEM;
    set_error(std::string("matrix allocation of ") + std::to_string(8.0 * off / 1e9) + " GB failed: " + cudaGetErrorString(e));
    cudaGetLastError();
    delete A;
    return nullptr;
  }
  A->data_bytes = bytes;
  *st = BEM_OK;
  return A;
}

bem_status assemble(int kind, const bem_mesh* m, const bem_quad_opts* o, bem_stream s, bem_matrix** out) {
  if (!m || !out) { set_error("bem_assemble: null argument"); return BEM_E_INVALID; }
  *out = nullptr;
  QuadCfg qc;
  bem_status qs = resolve_quad(kind, m, o, "bem_assemble", &qc);
  if (qs != BEM_OK) return qs;
  if (m->ng < 6) { set_error("bem_assemble: N_Gamma >= 6 required"); return BEM_E_INVALID; }
  cudaSetDevice(m->device);
  bem_status st;
  // V_h and D_h: symmetric packed spatial blocks unless BEM_QUAD_FULL_STORAGE
  const bool sym = (kind == STB_V || kind == STB_D) && !(o && (o->flags & BEM_QUAD_FULL_STORAGE));
  bem_matrix* A = new_dense(m, kind, sym, S(s), &st);
  if (!A) return st;
  // no memset: the bulk kernel writes every entry of the cells d >= 2 and the near kernel every
  // entry of the cells d <= 1 (the row padding is never read)
  st = launch_assembly(kind, m, A, qc, S(s));
  if (st == BEM_OK) st = gemv_setup(A);
  if (st != BEM_OK) { bem_matrix_destroy(A); return st; }
  *out = A;
  return BEM_OK;
}

int slice_of(const bem_mesh* m, int a) {
  int p = (int)(std::upper_bound(m->slice_first.begin(), m->slice_first.end(), a) - m->slice_first.begin()) - 1;
  return std::min(std::max(p, 0), m->P - 1);
}

// device offset of entry (a,i,b,j) or -1 (causality zero / not owned)
long long entry_offset(const bem_matrix* A, int a, int i, int b, int j) {
  const bem_mesh* m = A->mesh;
  if (b > a) return -1;
  if (A->toeplitz) {   // T_{a-b}(i, j)
    const int d = a - b;
    return A->poff[d] + (long long)i * pad4((long long)m->ng) + j;
  }
  const int I = slice_of(m, a), J = slice_of(m, b);
  for (size_t bi = 0; bi < m->blocks.size(); ++bi) {
    const Block& B = m->blocks[bi];
    if (B.I == I && B.J == J) {
      const long long p0 = A->poff[A->poff_base[bi] + (a - B.a0)];
      if (A->sym) {
        if (!sym_stored(i, j)) std::swap(i, j);   // the lower triangle mirrors the stored upper one
        return p0 + (long long)(b - B.b0) * A->blk_elems + sym_in_block(i, j, sym_nt(m->ng));
      }
      long long ld = pad4((long long)panel_nb(a, B.b0, B.b1) * m->ng);
      return p0 + (long long)i * ld + (long long)(b - B.b0) * m->ng + j;
    }
  }
  return -1;
}

__attribute__((unused)) double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

namespace stb {
bem_status gather_entries(const double* data, const long long* offs_dev, long long n, double* out_dev, cudaStream_t st);
}

extern "C" {

bem_status bem_assemble_toeplitz(const bem_mesh* m, int kind, const bem_quad_opts* o, bem_stream s,
                                 bem_matrix** out) {
  if (!m || !out) { set_error("bem_assemble_toeplitz: null argument"); return BEM_E_INVALID; }
  *out = nullptr;
  if (kind < STB_V || kind > STB_D) { set_error("bem_assemble_toeplitz: kind must be 0 (V), 1 (K) or 2 (D)"); return BEM_E_INVALID; }
  if (!m->uniform) { set_error("bem_assemble_toeplitz: needs equal time steps"); return BEM_E_STATE; }
  if (m->nranks > 1) { set_error("bem_assemble_toeplitz: one process (the Toeplitz blocks are replicated)"); return BEM_E_STATE; }
  QuadCfg qc;
  bem_status qs = resolve_quad(kind, m, o, "bem_assemble_toeplitz", &qc);
  if (qs != BEM_OK) return qs;
  qc.flags &= ~BEM_QUAD_FULL_STORAGE;   // the Toeplitz blocks are stored full anyway
  if (m->ng < 6) { set_error("bem_assemble_toeplitz: N_Gamma >= 6 required"); return BEM_E_INVALID; }
  cudaSetDevice(m->device);
  bem_status st;
  bem_matrix* A = new_dense(m, kind, false, S(s), &st, true);
  if (!A) return st;
  st = launch_assembly(kind, m, A, qc, S(s));
  if (st != BEM_OK) { bem_matrix_destroy(A); return st; }
  *out = A;
  return BEM_OK;
}

bem_status bem_assemble_V(const bem_mesh* m, const bem_quad_opts* o, bem_stream s, bem_matrix** out) {
  return assemble(STB_V, m, o, s, out);
}
bem_status bem_assemble_K(const bem_mesh* m, const bem_quad_opts* o, bem_stream s, bem_matrix** out) {
  return assemble(STB_K, m, o, s, out);
}
bem_status bem_assemble_D(const bem_mesh* m, const bem_quad_opts* o, bem_stream s, bem_matrix** out) {
  return assemble(STB_D, m, o, s, out);
}

bem_status bem_assemble_M(const bem_mesh* m, bem_mass_kind kind, bem_stream s, bem_matrix** out) {
  if (!m || !out) { set_error("bem_assemble_M: null argument"); return BEM_E_INVALID; }
  if (kind < BEM_MASS_PRIMAL || kind > BEM_MASS_DUAL_LUMPED) { set_error("bem_assemble_M: bad kind"); return BEM_E_INVALID; }
  cudaSetDevice(m->device);
  bem_matrix* M = new bem_matrix_s();
  M->kind = STB_MASS;
  M->mesh = m;
  M->stream = S(s);
  bem_status st = mass_setup(M, kind);
  if (st != BEM_OK) { bem_matrix_destroy(M); return st; }
  *out = M;
  return BEM_OK;
}

bem_status bem_matvec(const bem_matrix* A, double a, const double* x, double b, double* y, bem_stream s) {
  if (!A || !x || !y) { set_error("bem_matvec: null argument"); return BEM_E_INVALID; }
  if (x == y) { set_error("bem_matvec: x and y must not alias"); return BEM_E_INVALID; }
  if (A->kind == STB_MASS) return mass_apply(A, a, x, b, y, S(s));
  return gemv_launch(A, a, x, b, y, S(s));
}

bem_status bem_mass_solve(const bem_matrix* M, int transpose, const double* x, double* y, bem_stream s) {
  if (!M || !x || !y) { set_error("bem_mass_solve: null argument"); return BEM_E_INVALID; }
  if (M->kind != STB_MASS || M->mass_kind == BEM_MASS_PRIMAL) {
    set_error("bem_mass_solve: needs a dual (exact or lumped) mass matrix");
    return BEM_E_STATE;
  }
  return mass_solve(M, transpose, x, y, S(s));
}

bem_status bem_rhs(const bem_matrix* K, const bem_matrix* Mp, const double* g, double* b, bem_stream s) {
  if (!K || !Mp || !g || !b) { set_error("bem_rhs: null argument"); return BEM_E_INVALID; }
  if (K->kind != STB_K || Mp->kind != STB_MASS || Mp->mass_kind != BEM_MASS_PRIMAL) {
    set_error("bem_rhs: needs K_h and the primal mass matrix");
    return BEM_E_STATE;
  }
  bem_status st = gemv_launch(K, 1.0, g, 0.0, b, S(s));
  if (st != BEM_OK) return st;
  return mass_apply(Mp, 0.5, g, 1.0, b, S(s));
}

bem_status bem_rhs_fused(const bem_mesh* m, const bem_quad_opts* o, const bem_matrix* Mp,
                         const double* g, double* b, bem_assembly_stats* stats, bem_stream s) {
  if (!m || !Mp || !g || !b) { set_error("bem_rhs_fused: null argument"); return BEM_E_INVALID; }
  if (g == b) { set_error("bem_rhs_fused: g and b must not alias"); return BEM_E_INVALID; }
  if (Mp->kind != STB_MASS || Mp->mass_kind != BEM_MASS_PRIMAL) { set_error("bem_rhs_fused: needs the primal mass matrix"); return BEM_E_STATE; }
  if (m->ng < 6) { set_error("bem_rhs_fused: N_Gamma >= 6 required"); return BEM_E_INVALID; }
  QuadCfg qc;
  bem_status qs = resolve_quad(STB_K, m, o, "bem_rhs_fused", &qc);
  if (qs != BEM_OK) return qs;
  const int flags = qc.flags;
  if (!touching_records_ok(STB_K, m, flags)) {
    // large kappa: the per-lag singular kernel needs stored entries; assemble K_h, multiply
    bem_matrix* K = nullptr;
    bem_status st = assemble(STB_K, m, o, s, &K);
    if (st == BEM_OK) st = bem_rhs(K, Mp, g, b, s);
    if (st == BEM_OK && stats) st = bem_matrix_stats(K, stats);
    bem_matrix_destroy(K);
    return st;
  }
  cudaSetDevice(m->device);
  bem_matrix* A = new bem_matrix_s();   // statistics only: K_h is never stored
  A->kind = STB_K;
  A->mesh = m;
  A->stream = S(s);
  for (size_t bi = 0; bi < m->blocks.size(); ++bi) {
    A->poff_base.push_back((int)A->poff.size());
    for (int a = m->blocks[bi].a0; a < m->blocks[bi].a1; ++a) A->poff.push_back(0);
  }
  bem_status st = launch_assembly(STB_K, m, A, qc, S(s), g, b);
  if (st == BEM_OK && m->comm) st = allreduce_sum(m, b, (long long)m->ng * m->nt, S(s));
  if (st == BEM_OK) st = mass_apply(Mp, 0.5, g, 1.0, b, S(s));
  if (st == BEM_OK && stats) st = bem_matrix_stats(A, stats);
  bem_matrix_destroy(A);
  return st;
}

bem_status bem_rhs_initial(const bem_mesh* m, int n_nodes, const double* nodes_xy, int n_tri,
                           const int* tris, const double* u0, int qx, int qt_far, int qt_near,
                           double* b, bem_stream s) {
  if (!m || n_nodes < 3 || n_tri < 1 || !nodes_xy || !tris || !u0 || !b) { set_error("bem_rhs_initial: bad argument"); return BEM_E_INVALID; }
  if (qx <= 0) qx = 4;
  if (qt_far <= 0) qt_far = 4;
  if (qt_near <= 0) qt_near = 12;
  if (qx > QMAX || qt_far > QMAX || qt_near > QMAX) { set_error("bem_rhs_initial: orders must be <= 16"); return BEM_E_INVALID; }
  for (int k = 0; k < 3 * n_tri; ++k)
    if (tris[k] < 0 || tris[k] >= n_nodes) { set_error("bem_rhs_initial: triangle index out of range"); return BEM_E_INVALID; }
  if (m->nranks > 1) { set_error("bem_rhs_initial: one process"); return BEM_E_STATE; }
  cudaSetDevice(m->device);
  return initial_rhs(m, n_nodes, nodes_xy, n_tri, tris, u0, qx, qt_far, qt_near, b, S(s));
}

bem_status bem_eval_potential(const bem_mesh* m, const double* w, const double* g, long long npts,
                              const double* pts, double* u, bem_stream s) {
  if (!m || !w || !g || (npts > 0 && (!pts || !u)) || npts < 0) { set_error("bem_eval_potential: bad argument"); return BEM_E_INVALID; }
  cudaSetDevice(m->device);
  return eval_potential(m, w, g, npts, pts, u, S(s));
}

bem_status bem_eval_potential_initial(const bem_mesh* m, int n_nodes, const double* nodes_xy, int n_tri,
                                      const int* tris, const double* u0, long long npts, const double* pts,
                                      double* u, bem_stream s) {
  if (!m || n_nodes < 3 || n_tri < 1 || !nodes_xy || !tris || !u0 || npts < 0 || (npts > 0 && (!pts || !u))) {
    set_error("bem_eval_potential_initial: bad argument");
    return BEM_E_INVALID;
  }
  for (int k = 0; k < 3 * n_tri; ++k)
    if (tris[k] < 0 || tris[k] >= n_nodes) { set_error("bem_eval_potential_initial: triangle index out of range"); return BEM_E_INVALID; }
  cudaSetDevice(m->device);
  return eval_potential_initial(m, n_nodes, nodes_xy, n_tri, tris, u0, npts, pts, u, S(s));
}

bem_status bem_eval_special(int which, long long count, const double* x, double* out, bem_stream s) {
  if (which < 0 || which > 3 || count < 0) { set_error("bem_eval_special: bad argument"); return BEM_E_INVALID; }
  return eval_special(which, count, x, out, S(s));
}

bem_status bem_diag_fp64_rate(double seconds, double* tflops_host) {
  if (!tflops_host || !(seconds > 0.0) || seconds > 60.0) { set_error("bem_diag_fp64_rate: 0 < seconds <= 60, non-null output"); return BEM_E_INVALID; }
  return diag_fp64_rate(seconds, tflops_host);
}

// ------------------------------------------------------------------ GMRES
bem_status bem_solve_gmres(const bem_matrix* V, const bem_matrix* D, const bem_matrix* M,
                           const double* b, double* w, const bem_gmres_opts* opts,
                           bem_solve_report* rep, double* hist, bem_stream stream) {
  if (!V || !b || !w || !opts) { set_error("bem_solve_gmres: null argument"); return BEM_E_INVALID; }
  if (V->kind != STB_V) { set_error("bem_solve_gmres: first matrix must be V_h"); return BEM_E_STATE; }
  const int prec = opts->precond;
  if (prec < 0 || prec > 2) { set_error("bem_solve_gmres: precond must be 0, 1 or 2"); return BEM_E_INVALID; }
  if (prec > 0) {
    if (!D || !M || D->kind != STB_D || M->kind != STB_MASS) { set_error("bem_solve_gmres: preconditioner needs D_h and a dual mass matrix"); return BEM_E_STATE; }
    if ((prec == 1 && M->mass_kind != BEM_MASS_DUAL_LUMPED) || (prec == 2 && M->mass_kind != BEM_MASS_DUAL)) {
      set_error("bem_solve_gmres: precond 1 needs BEM_MASS_DUAL_LUMPED, precond 2 needs BEM_MASS_DUAL");
      return BEM_E_STATE;
    }
  }
  if (!(opts->rel_tol > 0) || opts->max_iter < 1) { set_error("bem_solve_gmres: rel_tol > 0 and max_iter >= 1 required"); return BEM_E_INVALID; }
  if (opts->flags & ~BEM_GMRES_FRESH_RESIDUAL) { set_error("bem_solve_gmres: unknown flags"); return BEM_E_INVALID; }
  const bool fresh_res = (opts->flags & BEM_GMRES_FRESH_RESIDUAL) != 0;
  if (V->mesh->comm && V->mesh->comm->solo) { set_error("bem_solve_gmres: a solo rank holds partial products only"); return BEM_E_STATE; }
  const bem_mesh* m = V->mesh;
  cudaSetDevice(m->device);
  const long long n = (long long)m->ng * m->nt;
  const int kmax = opts->max_iter;
  cudaStream_t st = S(stream);
  double *Q = nullptr, *tmp = nullptr, *u = nullptr, *v = nullptr, *dh = nullptr, *wk = nullptr;
  double* CQ = nullptr;    // C V q_k as the products leave them (true residual without products)
  double* hpin = nullptr;  // pinned host copy of the Hessenberg column (persistent, grow-only)
  cudaError_t e;
  // per host thread (concurrent solves on several threads, e.g. emulated ranks, each own theirs)
  struct PinBuf {
    double* p = nullptr;
    size_t n = 0;
    ~PinBuf() { if (p) cudaFreeHost(p); }
  };
  static thread_local PinBuf pin;
  const size_t slot = (size_t)2 * (kmax + 2);      // one Hessenberg column copy
  if (pin.n < 3 * slot) {                          // slots 0, 1 (alternating iterations), 2 (misc)
    if (pin.p) cudaFreeHost(pin.p);
    pin.p = nullptr;
    pin.n = 0;
    if (cudaMallocHost(&pin.p, sizeof(double) * 3 * slot) != cudaSuccess) {
      cudaGetLastError();
      set_error("bem_solve_gmres: pinned allocation failed");
      return BEM_E_NOMEM;
    }
    pin.n = 3 * slot;
  }
  hpin = pin.p;
  mesh_wait(m, st);
  // stream-ordered allocations: no device-wide synchronisation
  const size_t q_bytes = sizeof(double) * n * (kmax + 1);
  if ((e = storage_acquire(m->device, q_bytes, st, (void**)&Q)) != cudaSuccess ||
      (!fresh_res && (e = storage_acquire(m->device, q_bytes, st, (void**)&CQ)) != cudaSuccess) ||
      (e = cudaMallocAsync(&tmp, sizeof(double) * n, st)) != cudaSuccess ||
      (e = cudaMallocAsync(&u, sizeof(double) * n, st)) != cudaSuccess ||
      (e = cudaMallocAsync(&v, sizeof(double) * n, st)) != cudaSuccess ||
      (e = cudaMallocAsync(&wk, sizeof(double) * n, st)) != cudaSuccess ||
      (e = cudaMallocAsync(&dh, sizeof(double) * 2 * (kmax + 2), st)) != cudaSuccess) {
    storage_release(m->device, Q, q_bytes, st); cudaFreeAsync(tmp, st); cudaFreeAsync(u, st); cudaFreeAsync(v, st);
    if (CQ) storage_release(m->device, CQ, q_bytes, st);
    cudaFreeAsync(wk, st); cudaFreeAsync(dh, st);
    cudaGetLastError();
    set_error("bem_solve_gmres: allocation failed");
    return BEM_E_NOMEM;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  CommTimer ctimer;                 // device / host time of the collectives of this solve
  comm_timer_set(m->comm ? &ctimer : nullptr);
  // GEMV timing: an event pair per product, read once after the solve (no host sync per product)
  std::vector<cudaEvent_t> mvev;
  auto mv_mark = [&]() {
    cudaEvent_t x;
    cudaEventCreate(&x);
    cudaEventRecord(x, st);
    mvev.push_back(x);
  };
  double t_mv = 0.0;
  int nmv_V = 0, nmv_D = 0;
  cudaEventRecord(e0, st);
  bem_status status = BEM_OK;
  // z = C r  (C = M^{-1} D M^{-T}, lumped or exact), out may alias nothing else
  auto apply_C = [&](const double* r, double* out) -> bem_status {
    if (prec == 0) {
      return cudaMemcpyAsync(out, r, sizeof(double) * n, cudaMemcpyDeviceToDevice, st) == cudaSuccess ? BEM_OK : BEM_E_CUDA;
    }
    bem_status s1 = mass_solve(M, 1, r, u, st);
    if (s1 != BEM_OK) return s1;
    mv_mark();
    s1 = gemv_launch(D, 1.0, u, 0.0, v, st);
    ++nmv_D;
    mv_mark();
    if (s1 != BEM_OK) return s1;
    return mass_solve(M, 0, v, out, st);
  };
  auto apply_V = [&](const double* x, double* out) -> bem_status {
    mv_mark();
    bem_status s1 = gemv_launch(V, 1.0, x, 0.0, out, st);
    ++nmv_V;
    mv_mark();
    return s1;
  };
  cudaEvent_t nev;
  cudaEventCreateWithFlags(&nev, cudaEventDisableTiming);
  auto norm = [&](const double* x) -> double {
    vec_dots(x, 0, 1, x, n, dh, st);
    cudaMemcpyAsync(hpin + 2 * slot, dh, sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaEventRecord(nev, st);
    if (comm_wait_event(m, nev) != BEM_OK) {
      status = BEM_E_NCCL;
      return 0.0;
    }
    return std::sqrt(hpin[2 * slot]);
  };
  // one Arnoldi step k, enqueued only (no host wait): w = C V q_k, CGS2 against q_0..q_k with
  // both coefficient passes and ||w||^2 in dh, their copy to pinned slot k % 2 + an event, and
  // q_{k+1} = w / ||w|| scaled on the device
  cudaEvent_t hev[2];
  cudaEventCreateWithFlags(&hev[0], cudaEventDisableTiming);
  cudaEventCreateWithFlags(&hev[1], cudaEventDisableTiming);
  auto enqueue_step = [&](int k) -> bem_status {
    double* qk = Q + (long long)k * n;
    bem_status s1 = apply_V(qk, tmp);
    double* cq = CQ ? CQ + (long long)k * n : wk;
    if (s1 == BEM_OK) s1 = apply_C(tmp, cq);
    if (s1 != BEM_OK) return s1;
    if (CQ && cudaMemcpyAsync(wk, cq, sizeof(double) * n, cudaMemcpyDeviceToDevice, st) != cudaSuccess) return BEM_E_CUDA;
    vec_dots(Q, n, k + 1, wk, n, dh, st);
    vec_update(wk, Q, n, k + 1, dh, n, st);
    vec_dots(Q, n, k + 1, wk, n, dh + (k + 1), st);
    vec_update(wk, Q, n, k + 1, dh + (k + 1), n, st);
    vec_dots(wk, 0, 1, wk, n, dh + 2 * (k + 1), st);
    cudaMemcpyAsync(hpin + (k & 1) * slot, dh, sizeof(double) * (2 * k + 3), cudaMemcpyDeviceToHost, st);
    cudaEventRecord(hev[k & 1], st);
    if (k + 1 <= kmax) vec_scale_rnorm(Q + (long long)(k + 1) * n, wk, dh + 2 * (k + 1), n, st);
    return BEM_OK;
  };
  std::vector<double> H((size_t)(kmax + 1) * kmax, 0.0), cs(kmax), sn(kmax), g(kmax + 1, 0.0);
  int iters = 0;
  bool converged = false, breakdown = false;
  double resid = 1.0;
  status = apply_C(b, Q);
  double beta = status == BEM_OK ? norm(Q) : 0.0;
  if (status != BEM_OK) beta = 0.0;
  if (hist) hist[0] = 1.0;
  if (status == BEM_OK && beta == 0.0) {
    cudaMemsetAsync(w, 0, sizeof(double) * n, st);
    converged = true;
    resid = 0.0;
  } else if (status == BEM_OK) {
    vec_scale(Q, Q, 1.0 / beta, n, st);
    g[0] = beta;
    // Pipelined Arnoldi: step k + 1 is enqueued before the host waits for step k's Hessenberg
    // column (its vector q_{k+1} is scaled on the device), so the GPU never idles across the host's
    // Givens update -- unless the residual trend predicts that step k converges, in which case
    // the speculative step (one V and one D product) would be wasted and is not enqueued.
    int enq = -1;                                    // last enqueued step
    double r_prev = 1.0, r_prev2 = 1.0;
    if ((status = enqueue_step(0)) == BEM_OK) enq = 0;
    for (int k = 0; k < kmax && status == BEM_OK; ++k) {
      const double pred = k >= 2 ? r_prev * (r_prev / r_prev2) : 1.0;
      if (enq == k && k + 1 < kmax && pred > 2.0 * opts->rel_tol) {
        if ((status = enqueue_step(k + 1)) != BEM_OK) break;
        enq = k + 1;
      }
      // host wait for the column (polls NCCL for asynchronous errors: a failed peer aborts the
      // communicator instead of hanging the solve)
      if ((status = comm_wait_event(m, hev[k & 1])) != BEM_OK) break;
      const double* hcol = hpin + (k & 1) * slot;
      const double hk1 = std::sqrt(hcol[2 * k + 2]);
      double* Hk = &H[(size_t)k * (kmax + 1)];
      for (int j = 0; j <= k; ++j) Hk[j] = hcol[j] + hcol[(k + 1) + j];
      Hk[k + 1] = hk1;
      for (int j = 0; j < k; ++j) {
        double t1 = cs[j] * Hk[j] + sn[j] * Hk[j + 1];
        Hk[j + 1] = -sn[j] * Hk[j] + cs[j] * Hk[j + 1];
        Hk[j] = t1;
      }
      double den = std::hypot(Hk[k], Hk[k + 1]);
      cs[k] = Hk[k] / den;
      sn[k] = Hk[k + 1] / den;
      Hk[k] = den;
      Hk[k + 1] = 0.0;
      g[k + 1] = -sn[k] * g[k];
      g[k] = cs[k] * g[k];
      resid = std::fabs(g[k + 1]) / beta;
      iters = k + 1;
      if (hist) hist[k + 1] = resid;
      if (resid <= opts->rel_tol) { converged = true; break; }
      if (hk1 <= 1e-300) { breakdown = true; break; }
      r_prev2 = r_prev;
      r_prev = resid;
      if (enq == k && k + 1 < kmax) {               // not speculated: enqueue the next step now
        if ((status = enqueue_step(k + 1)) != BEM_OK) break;
        enq = k + 1;
      }
    }
    if (status == BEM_OK && iters > 0) {
      std::vector<double> y(iters);
      for (int i = iters - 1; i >= 0; --i) {
        double s = g[i];
        for (int j = i + 1; j < iters; ++j) s -= H[(size_t)j * (kmax + 1) + i] * y[j];
        y[i] = s / H[(size_t)i * (kmax + 1) + i];
      }
      // slot 2: a speculative step may still be copying its column into slot 0 or 1
      double* ypin = hpin + 2 * slot;
      for (int i = 0; i < iters; ++i) ypin[i] = y[i];
      cudaMemcpyAsync(dh, ypin, sizeof(double) * iters, cudaMemcpyHostToDevice, st);
      vec_combine(w, Q, n, iters, dh, n, st);
    }
  }
  double true_res = resid;
  if (status == BEM_OK && beta > 0.0 && !fresh_res) {
    // true preconditioned residual ||C(b - V w)|| / ||C b|| from the kept products:
    // C b - C V w = beta q_0 - sum_i y_i (C V q_i)  (y still in dh; no Hessenberg data involved)
    if (iters > 0) {
      vec_combine(wk, CQ, n, iters, dh, n, st);
      vec_axpby(wk, beta, Q, -1.0, n, st);
    } else {
      vec_axpby(wk, beta, Q, 0.0, n, st);
    }
    const double nr = norm(wk);
    if (status == BEM_OK) true_res = nr / beta;
  } else if (status == BEM_OK && beta > 0.0) {
    // true preconditioned residual ||C(b - V w)|| / ||C b|| from fresh products
    status = apply_V(w, tmp);
    if (status == BEM_OK) {
      vec_axpby(tmp, 1.0, b, -1.0, n, st);
      status = apply_C(tmp, wk);
      if (status == BEM_OK) {
        const double nr = norm(wk);
        if (status == BEM_OK) true_res = nr / beta;
      }
    }
  }
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms_total = 0;
  cudaEventElapsedTime(&ms_total, e0, e1);
  for (size_t k = 0; k + 1 < mvev.size(); k += 2) {
    float ms = 0;
    cudaEventElapsedTime(&ms, mvev[k], mvev[k + 1]);
    t_mv += ms * 1e-3;
  }
  for (auto x : mvev) cudaEventDestroy(x);
  e = cudaGetLastError();
  storage_release(m->device, Q, q_bytes, st); cudaFreeAsync(tmp, st); cudaFreeAsync(u, st); cudaFreeAsync(v, st);
  if (CQ) storage_release(m->device, CQ, q_bytes, st);
  cudaFreeAsync(wk, st); cudaFreeAsync(dh, st);
  cudaStreamSynchronize(st);
  comm_timer_set(nullptr);
  const double t_comm = comm_timer_seconds(&ctimer);
  cudaEventDestroy(e0); cudaEventDestroy(e1); cudaEventDestroy(nev);
  cudaEventDestroy(hev[0]); cudaEventDestroy(hev[1]);
  if (e != cudaSuccess) return cuda_fail(e, "bem_solve_gmres");
  if (rep) {
    rep->iterations = iters;
    rep->converged = converged ? 1 : 0;
    rep->rel_residual = resid;
    rep->true_rel_residual = true_res;
    rep->seconds_total = ms_total * 1e-3;
    rep->seconds_matvec = t_mv;
    rep->seconds_comm = t_comm;
    rep->n_matvec_V = nmv_V;
    rep->n_matvec_D = nmv_D;
  }
  if (status != BEM_OK) return status;
  if (!converged) {
    set_error(breakdown ? "bem_solve_gmres: Arnoldi breakdown" : "bem_solve_gmres: max_iter reached");
    return breakdown ? BEM_E_BREAKDOWN : BEM_E_NOT_CONVERGED;
  }
  return BEM_OK;
}

// ------------------------------------------------------------------ access
bem_status bem_matrix_get_entries(const bem_matrix* A, long long count, const long long* rows,
                                  const long long* cols, double* out) {
  if (!A || (count > 0 && (!rows || !cols || !out))) { set_error("bem_matrix_get_entries: null argument"); return BEM_E_INVALID; }
  if (A->kind == STB_MASS) { set_error("bem_matrix_get_entries: dense matrices only"); return BEM_E_STATE; }
  const bem_mesh* m = A->mesh;
  const long long n = (long long)m->ng * m->nt;
  std::vector<long long> offs(count);
  for (long long k = 0; k < count; ++k) {
    if (rows[k] < 0 || rows[k] >= n || cols[k] < 0 || cols[k] >= n) { set_error("bem_matrix_get_entries: index out of range"); return BEM_E_INVALID; }
    offs[k] = entry_offset(A, (int)(rows[k] / m->ng), (int)(rows[k] % m->ng), (int)(cols[k] / m->ng), (int)(cols[k] % m->ng));
  }
  cudaSetDevice(m->device);
  // the matrix may have been assembled on a non-blocking stream that the legacy stream used below
  // does not order against: wait for its assembly first
  if (A->stream) cudaStreamSynchronize(A->stream);
  const long long CH = 1 << 22;
  long long* d_off = nullptr;
  double* d_out = nullptr;
  long long cap = std::min(count, CH);
  if (cap <= 0) return BEM_OK;
  cudaError_t e;
  if ((e = cudaMalloc(&d_off, sizeof(long long) * cap)) != cudaSuccess) return cuda_fail(e, "get_entries");
  if ((e = cudaMalloc(&d_out, sizeof(double) * cap)) != cudaSuccess) { cudaFree(d_off); return cuda_fail(e, "get_entries"); }
  bem_status st = BEM_OK;
  for (long long k0 = 0; k0 < count && st == BEM_OK; k0 += CH) {
    long long nk = std::min(CH, count - k0);
    cudaMemcpy(d_off, offs.data() + k0, sizeof(long long) * nk, cudaMemcpyHostToDevice);
    st = gather_entries(A->data, d_off, nk, d_out, 0);
    cudaMemcpy(out + k0, d_out, sizeof(double) * nk, cudaMemcpyDeviceToHost);
  }
  e = cudaGetLastError();
  cudaFree(d_off);
  cudaFree(d_out);
  if (e != cudaSuccess) return cuda_fail(e, "get_entries");
  return st;
}

bem_status bem_matrix_get(const bem_matrix* A, long long r0, long long nr, long long c0, long long nc,
                          double* host) {
  if (!A || !host || nr < 0 || nc < 0) { set_error("bem_matrix_get: bad argument"); return BEM_E_INVALID; }
  std::vector<long long> rows((size_t)(nr * nc)), cols((size_t)(nr * nc));
  for (long long r = 0; r < nr; ++r)
    for (long long c = 0; c < nc; ++c) {
      rows[r * nc + c] = r0 + r;
      cols[r * nc + c] = c0 + c;
    }
  return bem_matrix_get_entries(A, nr * nc, rows.data(), cols.data(), host);
}

bem_status bem_matrix_stats(const bem_matrix* A, bem_assembly_stats* o) {
  if (!A || !o) { set_error("bem_matrix_stats: null"); return BEM_E_INVALID; }
  bem_status fs = finalize_assembly_stats(const_cast<bem_matrix*>(A));
  if (fs != BEM_OK) return fs;
  o->ms_bulk = A->ms_bulk;
  o->ms_near = A->ms_near;
  o->ms_sing = A->ms_sing;
  o->evals_bulk = A->ev_bulk;
  o->evals_near = A->ev_near;
  o->q_bulk = A->q_bulk;
  o->q_sing = A->q_sing;
  o->launches = A->launches;
  long long ent = 0;
  int kind = 0;
  bem_matrix_info(A, &kind, &ent, nullptr);
  o->entries = ent;
  o->flops_bulk = A->flops_bulk;
  o->ms_records = A->ms_records;
  o->fused_sing = A->fused_sing;
  o->nodes_bulk_tab = A->nodes_tab;
  for (int k = 0; k < 4; ++k) {
    o->nodes_bulk[k] = A->nodes_bulk[k];
    o->nodes_near[k] = A->nodes_near[k];
  }
  return BEM_OK;
}

bem_status bem_matrix_info(const bem_matrix* A, int* kind, long long* entries, long long* bytes) {
  if (!A) { set_error("bem_matrix_info: null"); return BEM_E_INVALID; }
  if (kind) *kind = A->kind;
  long long ent = 0;
  if (A->kind != STB_MASS) {
    // distinct stored entries (sym: the entries (i, j) with i / 32 <= j / 32, i, j < N_Gamma)
    const bem_mesh* m = A->mesh;
    long long per_block = (long long)m->ng * m->ng;
    if (A->sym) per_block = (long long)m->ng * (m->ng + 1) / 2;   // (i, j), i <= j
    for (auto& b : blocks_of(A))
      for (int a = b.a0; a < b.a1; ++a) ent += per_block * panel_nb(a, b.b0, b.b1);
  } else {
    ent = 3LL * A->mesh->ng * A->mesh->nt;
  }
  if (entries) *entries = ent;
  if (bytes) *bytes = A->kind == STB_MASS ? 8 * ent : 8 * A->entries;
  return BEM_OK;
}

bem_status bem_release_storage(void) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  for (int dev = 0; dev < 64; ++dev) {
    auto& c = g_cache[dev];
    for (auto& b : c) {
      cudaEventSynchronize(b.freed);
      cudaEventDestroy(b.freed);
      cudaFree(b.ptr);
    }
    c.clear();
  }
  // the device pool keeps freed memory mapped (release threshold: infinite, pool_setup): hand it
  // back to the driver so that other allocators in the process (torch) can use it
  int cur = 0;
  cudaGetDevice(&cur);
  for (int dev = 0; dev < 64; ++dev) {
    if (!pool_ready(dev)) continue;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      cudaSetDevice(dev);
      cudaDeviceSynchronize();
      cudaMemPoolTrimTo(pool, 0);
    }
  }
  cudaSetDevice(cur);
  cudaGetLastError();
  return BEM_OK;
}

void bem_matrix_destroy(bem_matrix* A) {
  if (!A) return;
  // stream-ordered: the storage returns to the pool after the work queued on the matrix's
  // stream (callers that used the matrix on another stream synchronise that stream first)
  const cudaStream_t st = A->stream;
  if (A->data) storage_release(A->mesh ? A->mesh->device : 0, A->data, A->data_bytes, st);
  storage_release(A->mesh ? A->mesh->device : 0, A->d_partials, A->partials_bytes, st);
  for (int c = 0; c < bem_matrix_s::COMM_CHUNKS; ++c)
    if (A->chunk_ev[c]) cudaEventDestroy(A->chunk_ev[c]);
  for (void* p : {(void*)A->d_segs, (void*)A->d_segs_ch, (void*)A->d_row_pbase,
                  (void*)A->d_row_pstride, (void*)A->d_ysum, (void*)A->d_rowcnt, (void*)A->d_lo, (void*)A->d_di,
                  (void*)A->d_up, (void*)A->d_work, (void*)A->d_ctr})
    if (p) cudaFreeAsync(p, st);
  for (auto x : A->ev) cudaEventDestroy(x);
  delete A;
}

}  // extern "C"
