// internal.h — data structures shared by the host runtime and the CUDA kernels of libstbem.
// Not part of the C-ABI (include/stbem.h is).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/stbem.h"

namespace stb {

// boundary element (primal segment or half segment): endpoints, length, unit tangent, outward normal
struct Seg {
  double ax, ay, bx, by;
  double h;
  double tx, ty;
  double nx, ny;
};

// dual hat psi_l (R6): values at the primal nodes x_l (vm) and x_{l+1} (vp),
// dual element lengths Lm = (h_{l-1}+h_l)/2 and Lp = (h_l+h_{l+1})/2
struct Dual {
  double vm, vp, Lm, Lp;
};

// one owned block (I,J) of the P x P temporal block structure:
// test steps a in [a0,a1), trial steps b in [b0,b1) with b <= a, packed as row panels
struct Block {
  int I, J;
  int a0, a1, b0, b1;
  long long off;  // first entry of the block in the matrix storage
};

// row-panel geometry of block blk for test step a: nb trial steps, ld (padded) row stride
inline __host__ __device__ int panel_nb(int a, int b0, int b1) {
  int last = a < b1 - 1 ? a : b1 - 1;
  return a >= b0 ? last - b0 + 1 : 0;
}
inline __host__ __device__ long long pad4(long long v) { return (v + 3) & ~3LL; }

// symmetric packed storage of the spatial blocks of V_h and D_h (V_ab(i,j) = V_ab(j,i): the
// kernels of P:86 and P:123 depend on |x - y| and on (x, y) symmetrically, test and trial spaces
// coincide).  Each N_Gamma x N_Gamma block (a,b) keeps the tiles (ti <= tj) of its upper tile
// triangle in row-major tile order: off-diagonal tiles 32 x 32 row-major, diagonal tiles as their
// upper triangle (row r holds columns r..31, 528 doubles), so that a block holds the upper
// triangle of the 32-tiled block plus nothing else (the full diagonal tiles were 7.5% / 10.8% of
// the stored doubles at C5 / C3, read by every product).
constexpr int SYM_TS = 32;
constexpr int SYM_TT = SYM_TS * SYM_TS;                 // off-diagonal tile
constexpr int SYM_TD = SYM_TS * (SYM_TS + 1) / 2;       // diagonal tile (upper triangle)
inline __host__ __device__ int sym_nt(int ng) { return (ng + SYM_TS - 1) / SYM_TS; }
inline __host__ __device__ long long sym_blk_elems(int ng) {
  const long long nt = sym_nt(ng);
  return nt * (nt + 1) / 2 * SYM_TT - nt * (SYM_TT - SYM_TD);
}
inline __host__ __device__ long long sym_tile_index(int ti, int tj, int nt) {
  return (long long)ti * nt - (long long)ti * (ti - 1) / 2 + (tj - ti);
}
// first stored double of tile (ti, tj), ti <= tj (ti + (tj > ti) diagonal tiles precede it)
inline __host__ __device__ long long sym_tile_offset(int ti, int tj, int nt) {
  return sym_tile_index(ti, tj, nt) * SYM_TT - (long long)(ti + (tj > ti ? 1 : 0)) * (SYM_TT - SYM_TD);
}
// offset of row r inside a tile such that + column c (c >= r in a diagonal tile) is the entry
inline __host__ __device__ int sym_row_base(int r, bool diag) {
  return diag ? r * SYM_TS - r * (r - 1) / 2 - r : r * SYM_TS;
}
// (i, j) is a stored entry: upper tile triangle, and i <= j inside a diagonal tile
inline __host__ __device__ bool sym_stored(int i, int j) {
  return i / SYM_TS < j / SYM_TS || (i / SYM_TS == j / SYM_TS && i <= j);
}
// offset inside a block of the stored entry (i, j) (sym_stored(i, j))
inline __host__ __device__ long long sym_in_block(int i, int j, int nt) {
  const int ti = i / SYM_TS, tj = j / SYM_TS;
  return sym_tile_offset(ti, tj, nt) + sym_row_base(i % SYM_TS, ti == tj) + (j % SYM_TS);
}

// flat description of the quadrature rules on the device
constexpr int QMAX = 16;
constexpr int QSING_MAX = 16;

}  // namespace stb

namespace stb { struct CommGroup; }
struct bem_comm_s {
  int nranks = 1, rank = 0, device = 0;
  void* nccl = nullptr;            // ncclComm_t (NCCL communicator), or
  stb::CommGroup* group = nullptr; // emulated ranks on one device (host-thread group, tests)
  cudaStream_t stream = nullptr;   // NCCL: the collectives' stream (overlap with the GEMV)
  bool failed = false;             // an asynchronous NCCL error was seen: the communicator is aborted
  bool solo = false;               // one rank of nranks alone: collectives are no-ops (partial sums)
};

struct bem_mesh_s {
  int ng = 0, nt = 0, P = 1;
  double alpha = 1.0;
  int device = 0;
  std::vector<double> t;          // n_steps + 1
  std::vector<stb::Seg> seg;      // ng primal segments
  std::vector<stb::Seg> half;     // 2 ng half segments
  std::vector<stb::Dual> dual;    // ng dual hats
  std::vector<int> slice_first;   // P + 1
  std::vector<int> owner;         // P * P, -1 above the diagonal
  std::vector<stb::Block> blocks; // blocks owned by this rank
  long long entries_owned = 0;
  double hmax = 0, htmin = 0, kappa = 0;
  bool uniform = false;           // equal time steps (block-Toeplitz variant allowed)
  int q_bulk = 4;     // V_h, K_h (primal segments)
  int q_bulk_d = 4;   // D_h (half segments)
  bem_comm* comm = nullptr;
  int rank = 0, nranks = 1;
  // device copies
  double* d_t = nullptr;
  stb::Seg* d_seg = nullptr;
  stb::Seg* d_half = nullptr;
  stb::Dual* d_dual = nullptr;
  double4* d_lag = nullptr;       // (s, ln s, 1/s, 0) for time nodes x > y: index x*(nt+1)+y
  cudaEvent_t ready = nullptr;    // the uploads above are complete (waited on by every user stream)
};

// matrix kinds
enum { STB_V = 0, STB_K = 1, STB_D = 2, STB_MASS = 3 };

struct bem_matrix_s {
  int bulk_r = 0;                  // band height (test steps) of the bulk kernel of the last assembly
  int kind = 0;
  const bem_mesh* mesh = nullptr;
  // every device buffer of the matrix is allocated and freed stream-ordered on this stream (the
  // stream of bem_assemble_*): assembly, setup and destroy never block the host
  cudaStream_t stream = nullptr;
  // lazily finalised assembly statistics (events + counters read on the first stats query)
  std::vector<cudaEvent_t> ev;
  std::vector<int> ev_fam;
  unsigned long long* d_ctr = nullptr;
  bool stats_ready = true;
  // dense block-lower-triangular storage (V, K, D)
  double* data = nullptr;
  int sym = 0;                 // symmetric packed spatial blocks (V, D)
  int toeplitz = 0;            // block-Toeplitz variant: stores T_d = A(d, 0), d < N_I (full blocks)
  std::vector<stb::Block> own_blocks;   // toeplitz: the single first-block-column block
  long long blk_elems = 0;     // sym: stored doubles per (a,b) block
  size_t data_bytes = 0;       // size of the storage block (>= 8 * entries; cached on destroy)
  long long entries = 0;       // stored doubles (with row padding)
  std::vector<long long> poff; // per block, per local test step: panel offset (flattened)
  std::vector<int> poff_base;  // per block: index of its first panel in poff
  // GEMV work decomposition
  struct GemvSeg {
    long long item0;   // first work item
    long long off;     // panel offset in data
    long long ld;      // padded row stride
    long long len;     // row length (unpadded)
    long long xoff;    // first column (global index) of the panel
    long long pbase;   // partial index of (row i = 0, chunk 0) of this segment
    int nch;           // chunks per row in this segment
    int pstride;       // partials per row (all blocks of this test step)
    int a;             // test step
    int pad;
  };
  std::vector<GemvSeg> segs;
  GemvSeg* d_segs = nullptr;
  // multi-GPU, symmetric packed: the same items split into row chunks (test steps), so that the
  // all-reduce of one chunk's rows overlaps the GEMV of the next (linalg.cu)
  static constexpr int COMM_CHUNKS = 4;
  int nchunks = 0;
  int chunk_seg0[COMM_CHUNKS + 1] = {0};       // segment range of chunk c in d_segs_ch
  long long chunk_items[COMM_CHUNKS] = {0};
  int chunk_row0[COMM_CHUNKS + 1] = {0};       // test steps [row0[c], row0[c+1])
  GemvSeg* d_segs_ch = nullptr;
  cudaEvent_t chunk_ev[COMM_CHUNKS] = {nullptr};
  long long n_items = 0, n_partials = 0;
  std::vector<long long> row_pbase;  // per test step: partial base, stride = row_pstride[a]
  std::vector<int> row_pstride;
  long long* d_row_pbase = nullptr;
  int* d_row_pstride = nullptr;
  double* d_partials = nullptr;
  size_t partials_bytes = 0;
  double* d_ysum = nullptr;  // multi-GPU partial y
  int* d_rowcnt = nullptr;   // SYMV: finished blocks per row (last block reduces; self-resetting)
  bool empty_rows = false;   // some test step owns no block here (multi-GPU): y = b y there
  // mass matrices: three cyclic diagonals per row (lower = col i-1, diag, upper = col i+1)
  int mass_kind = -1;
  double* d_lo = nullptr;
  double* d_di = nullptr;
  double* d_up = nullptr;
  double* d_work = nullptr;  // dual mass: cyclic-tridiagonal factors, 2 x N_I x (4 N_Gamma + 2)
  // assembly statistics
  double ms_bulk = 0, ms_near = 0, ms_sing = 0, ms_records = 0;
  long long ev_bulk = 0, ev_near = 0, nodes_expected = 0;
  long long nodes_bulk[4] = {0, 0, 0, 0}, nodes_near[4] = {0, 0, 0, 0};  // regimes A, B, Z, C
  double flops_bulk = 0;
  long long nodes_tab = 0;   // K_h g: bulk regime-A nodes summed by the trial-moment table
  double flops_tab = 0;      // its algorithmic flops (host count at launch)
  int kg_tab = 0;
  int q_bulk = 0, q_sing = 0, launches = 0, fused_sing = 0;
};

namespace stb {
inline const std::vector<Block>& blocks_of(const bem_matrix_s* A);
// error handling
void set_error(const std::string& msg);
// the mesh's device data are ready on stream st (stream-ordered wait on the upload event)
inline void mesh_wait(const bem_mesh* m, cudaStream_t st) {
  if (m && m->ready) cudaStreamWaitEvent(st, m->ready, 0);
}
bem_status cuda_fail(cudaError_t e, const char* where);
void count_launch(long long k = 1);

// host quadrature tables
struct Rules {
  double x[QMAX + 1][QMAX];  // Gauss-Legendre nodes on [0,1], n = 1..QMAX
  double w[QMAX + 1][QMAX];
  double lw[QMAX + 1][QMAX]; // log-weights: int_0^1 l_k(r) ln r dr for the same nodes
};
const Rules& host_rules();
bem_status upload_rules();  // copy to __constant__ memory (per device, once)

// device storage (api.cpp): blocks >= 1 MB are cached after release and reused stream-ordered by
// the next acquire of a size that fits (<= 25% larger); smaller ones use the device pool
cudaError_t storage_acquire(int device, size_t bytes, cudaStream_t st, void** out);
void storage_release(int device, void* ptr, size_t bytes, cudaStream_t st);

// kernels (assemble.cu)
// touching pairs through moment records (regime A) whenever every touching sub-pair satisfies
// c_max / min h_t < 4 with c_max <= alpha (h_X + h_Y)^2 / 4
inline bool touching_records_ok(int kind, const bem_mesh* m, int flags) {
  const double hpair = (kind == STB_D ? 1.0 : 2.0) * m->hmax;
  return !(flags & BEM_QUAD_LEGACY_SING) && 0.25 * m->alpha * hpair * hpair / m->htmin < 0.99 * 4.0;
}
// resolved quadrature options (bem_quad_opts with the defaults applied)
struct QuadCfg {
  int q_far;        // Gauss order of the bulk time cells d >= 2
  int q_near;       // near cells (d <= 1): order of the pairs at distance ratio >= near_gap
  double near_gap;  // near cells: distance ratio below which the measured orders 10 / 8 / 6 apply
  int q_sing;       // touching pairs: singular rules
  int flags;
};
// defaults and validation of bem_quad_opts for matrix kind `kind` (BEM_E_INVALID with a message)
bem_status resolve_quad(int kind, const bem_mesh* m, const bem_quad_opts* o, const char* where, QuadCfg* out);
// prod_g != nullptr: product mode (K_h only): prod_y = K_h prod_g over the owned blocks, K_h is
// not stored (A carries statistics only)
bem_status launch_assembly(int kind, const bem_mesh* m, bem_matrix* A, const QuadCfg& qc,
                           cudaStream_t st, const double* prod_g = nullptr,
                           double* prod_y = nullptr);
// linear algebra (linalg.cu)
bem_status gemv_setup(bem_matrix* A);
bem_status gemv_launch(const bem_matrix* A, double a, const double* x, double b, double* y,
                       cudaStream_t st);
bem_status mass_setup(bem_matrix* M, int kind);
bem_status finalize_assembly_stats(bem_matrix* A);
bem_status mass_apply(const bem_matrix* M, double a, const double* x, double b, double* y,
                      cudaStream_t st);
bem_status mass_solve(const bem_matrix* M, int transpose, const double* x, double* y,
                      cudaStream_t st);
bem_status eval_special(int which, long long n, const double* x, double* out, cudaStream_t st);
bem_status diag_fp64_rate(double seconds, double* tflops);
bem_status eval_potential_initial(const bem_mesh* m, int nnode, const double* nodes, int ntri, const int* tris,
                                  const double* u0, long long npts, const double* pts, double* out,
                                  cudaStream_t st);
bem_status initial_rhs(const bem_mesh* m, int nnode, const double* nodes, int ntri, const int* tris,
                       const double* u0, int qx, int qtf, int qtn, double* b, cudaStream_t st);
bem_status eval_potential(const bem_mesh* m, const double* w, const double* g, long long npts,
                          const double* pts, double* out, cudaStream_t st);
// vector kernels (linalg.cu)
void vec_dots(const double* Q, long long ldq, int k, const double* w, long long n, double* out,
              cudaStream_t st);
void vec_update(double* w, const double* Q, long long ldq, int k, const double* h, long long n,
                cudaStream_t st);
void vec_scale(double* y, const double* x, double s, long long n, cudaStream_t st);
void vec_scale_rnorm(double* y, const double* x, const double* nrm2_dev, long long n, cudaStream_t st);
void vec_axpby(double* y, double a, const double* x, double b, long long n, cudaStream_t st);
void vec_combine(double* out, const double* Q, long long ldq, int k, const double* coef,
                 long long n, cudaStream_t st);
void vec_mul(double* y, const double* d, const double* x, long long n, cudaStream_t st);
// collectives (comm.cpp)
bem_status allreduce_sum(const bem_mesh* m, double* buf, long long n, cudaStream_t st);
// ranks that share the pair-record computation (nranks of a NCCL or emulated-rank communicator;
// 1 without one and for a solo rank, which computes every record itself)
int record_ranks(const bem_mesh* m);
// in-place all-gather of G = record_ranks(m) chunks of `chunk` doubles: rank r's chunk is
// buf[r * chunk, (r + 1) * chunk); afterwards every rank holds all G chunks (stream-ordered on st)
bem_status allgather_chunks(const bem_mesh* m, double* buf, long long chunk, cudaStream_t st);
// stream on which allreduce_sum_async runs the NCCL collective after waiting on `ready` (recorded
// on the compute stream); the caller joins it back with comm_join.  Group / no communicator:
// the plain allreduce_sum on st.
bem_status allreduce_sum_async(const bem_mesh* m, double* buf, long long n, cudaStream_t st, cudaEvent_t ready);
bem_status comm_join(const bem_mesh* m, cudaStream_t st);
bool comm_overlaps(const bem_mesh* m);   // NCCL with its own collective stream
// host wait on an event that polls the communicator for asynchronous NCCL errors (and aborts it on
// one) instead of blocking: a failed peer cannot hang the solve.  BEM_E_NCCL on an error.
bem_status comm_wait_event(const bem_mesh* m, cudaEvent_t ev);
// collective timing sink of the calling thread (bem_solve_gmres): device time of the collectives
// (CUDA events around each NCCL call on its stream) and host time of the group collectives
struct CommTimer {
  std::vector<cudaEvent_t> ev;   // pairs (start, end)
  double host_s = 0.0;
};
void comm_timer_set(CommTimer* t);   // nullptr: off
double comm_timer_seconds(CommTimer* t);   // sums and destroys the events
}  // namespace stb

namespace stb {
// the temporal blocks a matrix stores: the mesh's owned blocks, or the toeplitz matrix's own
inline const std::vector<Block>& blocks_of(const bem_matrix_s* A) {
  return A->toeplitz ? A->own_blocks : A->mesh->blocks;
}
bem_status toeplitz_gemv(const bem_matrix* A, double a, const double* x, double b, double* y,
                         cudaStream_t st);
}  // namespace stb
