/*
 * stbem.h — C-ABI of the B200-native space-time boundary element library for the
 * heat equation (Dohr, Merta, Of, Steinbach, Zapletal, arXiv:1811.05224).
 *
 * Citations: P:n = PAPER.md line n.  All arithmetic is FP64.  Every function returns a
 * bem_status; on a non-OK status bem_last_error() returns a thread-local message.  No C++
 * exception crosses this boundary.  Nothing here ever falls back to the CPU: every
 * compute call runs CUDA kernels for sm_100a and returns BEM_E_CUDA if none can run.
 *
 * Index convention (R13): global unknown l = a * n_gamma + i, a = time step
 * (tau_a = (t_a, t_{a+1})), i = boundary element gamma_i (primal) or dual hat psi_i.
 *
 * Ownership: opaque handles are created by the library and freed only by the matching
 * *_destroy.  Vectors passed as `const double*` / `double*` with the suffix _dev are
 * caller-owned DEVICE memory on the handle's device, length n = n_gamma * n_steps
 * (full length on every rank: vectors are replicated; the multi-GPU layer reduces
 * partial products internally).  `_host` arrays are caller-owned host memory.
 * Streams are caller-owned (0 = legacy default stream).
 */
#ifndef STBEM_H
#define STBEM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BEM_OK = 0,
  BEM_E_INVALID = 1,       /* invalid argument or descriptor */
  BEM_E_NOMEM = 2,         /* device or host allocation failed */
  BEM_E_CUDA = 3,          /* CUDA error, or no CUDA device */
  BEM_E_NCCL = 4,          /* NCCL error */
  BEM_E_NOT_CONVERGED = 5, /* GMRES reached max_iter; w holds the last iterate */
  BEM_E_BREAKDOWN = 6,     /* Arnoldi breakdown (sub-diagonal < 1e-300) before convergence */
  BEM_E_STATE = 7          /* wrong object (kind / mesh mismatch) */
} bem_status;

typedef struct bem_comm_s bem_comm;
typedef struct bem_mesh_s bem_mesh;
typedef struct bem_matrix_s bem_matrix;
typedef void* bem_stream; /* a cudaStream_t */

/* Problem geometry and time grid (eq. 1, P:64 Sigma_h = Gamma_h x I_h).
 * vertices_xy: 2*n_vertices doubles, a simple counter-clockwise polygon.
 * segments_per_side[s] >= 1 equal segments on side s (from vertex s to s+1).
 * t_breaks: n_steps+1 strictly increasing values, t_breaks[0] = 0.
 * alpha > 0 heat capacity (eq. 1).  n_slices P: temporal submeshes, 1 <= P <= n_steps
 * (P:217).  All arrays are host memory and are copied. */
typedef struct {
  int n_vertices;
  const double* vertices_xy;
  const int* segments_per_side;
  int n_steps;
  const double* t_breaks;
  double alpha;
  int n_slices;
} bem_mesh_desc;

typedef struct {
  int n_gamma;             /* N_Gamma boundary elements (= dual hats) */
  int n_steps;             /* N_I time steps */
  long long n;             /* N = n_gamma * n_steps */
  int n_slices;            /* P */
  int n_owned_blocks;      /* blocks (I,J) of the P x P block structure owned by this rank */
  long long entries_owned; /* stored entries per matrix on this rank */
  long long entries_total; /* n_gamma^2 n_steps (n_steps+1) / 2 */
  int q_bulk;              /* Gauss points per direction for d = a-b >= 2 (per mesh) */
  double kappa;            /* alpha h_max^2 / (4 min h_t): smoothness ratio choosing q_bulk */
  int rank, nranks;        /* this process in the communicator (0, 1 without one) */
  /* vector layout (reading R27): vectors are REPLICATED -- every rank holds all n
   * entries, local_row0 = 0 and local_rows = n on every rank; a product's owned-block partials are
   * summed over the ranks inside the library, so the caller never exchanges vector pieces */
  long long local_rows, local_row0;
} bem_mesh_info;

/* Quadrature options (the paper's quadrature is unpublished, reading R1 and section
 * 4.3); NULL or 0 in a field = the documented default.  Negative values, q_far not in
 * {3,4,5,6,8}, q_near not in [3,16], q_sing not in [4,16] or unknown flags: BEM_E_INVALID. */
typedef struct {
  int q_far;    /* Gauss order per direction for the time cells d = a - b >= 2; default chosen from
                   kappa = alpha h_max^2 / (4 min h_t) (bem_mesh_info.q_bulk) */
  int q_near;   /* time cells d <= 1, non-touching pairs at distance ratio dist / h >= near_gap;
                   default min(6, q_far + 1) */
  int near_gap; /* time cells d <= 1: pairs closer than near_gap element lengths take the measured
                   orders 10 (ratio < 2.5), 8 (< 5), 6 (< near_gap); default 9 */
  int q_sing;   /* order of the Duffy / 1-D reduction rules for touching pairs (default 16) */
  int flags;    /* BEM_QUAD_* below */
} bem_quad_opts;
/* touching pairs by per-lag singular rules (k_sing) instead of moment records; without it the
 * records are used whenever alpha (h_X + h_Y)^2 / (4 min h_t) < 4 */
#define BEM_QUAD_LEGACY_SING 1
/* V_h and D_h store their symmetric spatial blocks packed (upper triangle: off-diagonal 32 x 32 tiles
 * and triangular diagonal tiles, about half the bytes and half the assembly work, DESIGN.md section
 * 4.1); this flag stores them full */
#define BEM_QUAD_FULL_STORAGE 2
/* bem_rhs_fused: evaluate every regime-A node of K_h pair by pair instead of summing the regime-A
 * fields of the trial pairs first (trial-moment table; same quadrature and
 * regime forms, re-associated over the trial index) -- the reference path for tests */
#define BEM_QUAD_KG_ENTRYWISE 4

typedef enum {
  BEM_MASS_PRIMAL = 0,      /* M_h of eq. (4): <phi^10_(a,n), phi^0_(a,i)> */
  BEM_MASS_DUAL = 1,        /* M_h of Thm 1: <phi^0_(a,k), psi_(a,l)>, cyclic tridiagonal */
  BEM_MASS_DUAL_LUMPED = 2  /* row sums of BEM_MASS_DUAL */
} bem_mass_kind;

typedef struct {
  double rel_tol;  /* stop when ||C(b - V w_k)|| <= rel_tol ||C b|| (Givens estimate) */
  int max_iter;    /* full GMRES, no restart */
  int precond;     /* 0 none, 1 lumped dual mass, 2 exact dual mass (cyclic tridiagonal) */
  int flags;       /* BEM_GMRES_* below (0: defaults) */
} bem_gmres_opts;
/* the true residual at exit from two fresh products C V w (one V_h and one D_h product more)
 * instead of from the products of the Arnoldi steps: C(b - V w) = C b - sum_i y_i (C V q_i) by
 * linearity, with the vectors C V q_i kept as they leave the products (before orthogonalisation),
 * so that the default check costs no product; both are independent of the Givens recurrence */
#define BEM_GMRES_FRESH_RESIDUAL 1

typedef struct {
  int iterations;
  int converged;
  double rel_residual;       /* Givens estimate at exit */
  double true_rel_residual;  /* ||C(b - V w)|| / ||C b|| recomputed at exit (BEM_GMRES_FRESH_RESIDUAL) */
  double seconds_total;
  double seconds_matvec;     /* V and D products (device time) */
  double seconds_comm;       /* collectives: device time of the NCCL calls (CUDA events on their
                                stream, overlapped with the GEMV where chunked), host time of the
                                emulated ranks' all-reduces; 0 without a communicator */
  int n_matvec_V;            /* V_h products performed (incl. a fresh true-residual check) */
  int n_matvec_D;            /* D_h products performed */
} bem_solve_report;

/* Per-matrix assembly statistics: device time of the assembly kernel families, measured with
 * CUDA events on the stream passed to bem_assemble_*, and the number of time-node evaluations
 * (entry-level spatial pair x time node) of the bulk (d >= 2) and near (d <= 1) kernels, split by
 * evaluation regime: [0] A moment polynomial, [1] B Taylor about the
 * cluster centre, [2] Z exponentially small, [3] C point by point. */
typedef struct {
  double ms_bulk, ms_near, ms_sing;
  long long evals_bulk, evals_near;   /* node evaluations (sum over regimes) */
  int q_bulk, q_sing;
  int launches;
  long long entries;         /* stored (unpadded) entries */
  double flops_bulk;         /* algorithmic FP64 flops of the bulk kernels */
  double ms_records;         /* pair-record (moment) kernels */
  long long nodes_bulk[4];   /* bulk node evaluations per regime A, B, Z, C */
  long long nodes_near[4];   /* near-cell node evaluations per regime */
  int fused_sing;            /* 1: touching pairs through moment records, 0: per-lag k_sing */
  long long nodes_bulk_tab;  /* bem_rhs_fused: bulk regime-A nodes summed over the trial index by the
                                trial-moment table (included in nodes_bulk[0]; 0 otherwise) */
} bem_assembly_stats;

/* ---------------------------------------------------------------- general */
const char* bem_version(void);
const char* bem_last_error(void);   /* thread-local text for the last non-OK status */
/* number of kernel launches issued by this thread since the last reset (instrumentation) */
long long bem_launch_count(int reset);

/* ----------------------------------------------------------- multi-GPU (NCCL) */
/* rank 0 creates the 128-byte NCCL unique id; the caller broadcasts it (torch.distributed). */
bem_status bem_nccl_get_unique_id(void* out128_host);
/* collective over nranks: one rank per GPU; cuda_device is this rank's device ordinal.  A mesh
 * created with a communicator runs the distributed code path (owned blocks of the cyclic plan,
 * partial products summed by ncclAllReduce on the caller's stream) -- also for nranks = 1, where
 * the all-reduce runs on a real one-rank communicator; a mesh without one never calls NCCL.
 * Errors: BEM_E_INVALID (arguments), BEM_E_NCCL (libnccl.so.2 not loadable or NCCL failure). */
bem_status bem_comm_create(const void* unique_id128_host, int nranks, int rank, int cuda_device,
                           bem_comm** out);
/* Emulated ranks on ONE device, without NCCL (tests of the multi-rank path on a single GPU):
 * writes nranks (1..16) communicator handles to out_host[0 .. nranks-1], rank r = out_host[r], all
 * on cuda_device.  Each rank must be driven by its own host thread, SPMD, exactly as one process per
 * GPU would (every rank calls every collective function).  A product's all-reduce synchronises the
 * rank's stream, meets the other ranks at a host barrier, sums all ranks' partial results in rank
 * order (identical on every rank) and copies the sum back after a second barrier -- no kernel waits
 * on another rank's kernel.  Each handle is freed with bem_comm_destroy.
 * Errors: BEM_E_INVALID (nranks out of range, null out_host), BEM_E_CUDA. */
bem_status bem_comm_create_group(int nranks, int cuda_device, bem_comm** out_host);
/* One rank of nranks ALONE on cuda_device, without NCCL (load-balance studies and partial-product
 * tests): a mesh created with it owns rank `rank`'s blocks of the cyclic plan, and every product or
 * fused right-hand side returns this rank's partial sums over its owned blocks (the collectives are
 * no-ops): the sum over the ranks' results is the full product (bem_rhs_fused adds its
 * 1/2 M_h g term on every rank).  bem_solve_gmres refuses such a mesh (BEM_E_STATE).
 * Errors: BEM_E_INVALID, BEM_E_CUDA. */
bem_status bem_comm_create_solo(int nranks, int rank, int cuda_device, bem_comm** out);
/* NCCL communicators: the collectives run on the communicator's own stream (a product's row
 * chunks are all-reduced while the GEMV of the next chunk runs); every host wait of the solver polls
 * ncclCommGetAsyncError and aborts the communicator on an asynchronous error (BEM_E_NCCL from then
 * on).  Frees the handle (NCCL or emulated). */
void bem_comm_destroy(bem_comm* comm);

/* ----------------------------------------------------- cyclic K_P plan (host) */
/* Cyclic decomposition of the complete graph K_P (Fig. 3, R15):
 * owner_host[i*P + j] = process owning block (i,j), j <= i (entries with j > i are -1).
 * Pure host code: callable without a GPU. */
bem_status bem_plan_build(int P, int* owner_host);
/* generator G_0: out_host[k] = k-th vertex of the difference cover (count in *n_out) */
bem_status bem_plan_generator(int P, int* out_host, int* n_out);
/* blocks (I,J) owned by `rank` of `nranks` GPUs when the P processes of the plan are mapped
 * round-robin to GPUs (process p -> GPU p mod nranks, R15): writes 2*count ints
 * (I, J pairs, row-major block order) to out_host (capacity P*(P+1) ints) and the count. */
bem_status bem_plan_owned_blocks(int P, int nranks, int rank, int* out_host, int* count);
/* balanced slice ranges (R14): slice p = time steps [first[p], first[p+1]) */
bem_status bem_slice_ranges(int n_steps, int P, int* first_host /* P+1 */);

/* ---------------------------------------------------------------- mesh */
/* Validates the descriptor, builds Gamma_h, the half segments of the dual mesh (R6),
 * the time grid, the slices and the block ownership (comm == NULL: one GPU owns all blocks),
 * and uploads them to the current CUDA device. */
bem_status bem_mesh_create(const bem_mesh_desc* desc, bem_comm* comm, bem_mesh** out);
bem_status bem_mesh_info_get(const bem_mesh* mesh, bem_mesh_info* info);
void bem_mesh_destroy(bem_mesh* mesh);

/* ------------------------------------------------------------ assembly */
/* All three need N_Gamma >= 6 (the touching-pair enumeration of the dual half segments assumes
 * distinct neighbours); smaller boundaries return BEM_E_INVALID.  Any kappa = alpha h^2 /
 * (4 min h_t): above 1 the elements are integrated with composite rules (reading R24).
 * V_h[(a,i),(b,j)] = <V phi^0_(b,j), phi^0_(a,i)> with (1/alpha) U* (P:43).
 * Stored entries: owned blocks, b <= a, packed row panels. */
bem_status bem_assemble_V(const bem_mesh* mesh, const bem_quad_opts* opts, bem_stream stream,
                          bem_matrix** out);
/* K_h[(a,i),(b,n)] = <K phi^10_(b,n), phi^0_(a,i)> with (1/alpha) d_{n_y} U* (P:44). */
bem_status bem_assemble_K(const bem_mesh* mesh, const bem_quad_opts* opts, bem_stream stream,
                          bem_matrix** out);
/* D_h[(a,l),(b,k)] = <D psi_(b,k), psi_(a,l)> (Thm 1; D = -d_n W) in the
 * integration-by-parts form of DESIGN.md R7, dual hats of R6. */
bem_status bem_assemble_D(const bem_mesh* mesh, const bem_quad_opts* opts, bem_stream stream,
                          bem_matrix** out);
/* mass matrices (block diagonal in time): see bem_mass_kind */
/* Block-Toeplitz variant (uniform time steps only): on equal steps the
 * entries depend on the test and trial steps through d = a - b only, A(a, b) = T_d.  Assembles
 * the first block column T_d = A(d, 0), d = 0 .. N_I - 1 (N_I N_Gamma^2 entries instead of
 * N_Gamma^2 N_I (N_I + 1) / 2) with the kernels and quadrature of bem_assemble_*; bem_matvec then
 * evaluates y_a = sum_{d <= a} T_d x_{a-d} as one FP64 GEMM over the stacked index (d, j), and
 * bem_solve_gmres / bem_rhs / bem_matrix_get_entries accept the result like a dense matrix.
 * This avoids the dense work the paper does: report its rates separately.  kind: 0 V_h, 1 K_h,
 * 2 D_h.  Errors: BEM_E_STATE (non-uniform steps, more than one process), BEM_E_INVALID
 * (options), BEM_E_NOMEM, BEM_E_CUDA. */
bem_status bem_assemble_toeplitz(const bem_mesh* mesh, int kind, const bem_quad_opts* opts,
                                 bem_stream stream, bem_matrix** out);
bem_status bem_assemble_M(const bem_mesh* mesh, bem_mass_kind kind, bem_stream stream,
                          bem_matrix** out);

/* --------------------------------------------------------------- products */
/* y = a A x + b y for an assembled V/K/D matrix (block-lower-triangular FP64 GEMV) or a mass
 * matrix.  x_dev, y_dev: device, length n, must not alias.  Multi-GPU: partial products of the
 * owned blocks are summed over ranks (NCCL) so y is complete on every rank. */
bem_status bem_matvec(const bem_matrix* A, double a, const double* x_dev, double b, double* y_dev,
                      bem_stream stream);
/* y = M^{-1} x (transpose = 0) or M^{-T} x (transpose = 1) for a mass matrix (dual: N_I cyclic
 * tridiagonal solves of size N_Gamma; lumped: diagonal scaling). x_dev, y_dev may alias. */
bem_status bem_mass_solve(const bem_matrix* M, int transpose, const double* x_dev, double* y_dev,
                          bem_stream stream);
/* right-hand side of eq. (4) with u0 = 0: b = 1/2 M_primal g + K g */
bem_status bem_rhs(const bem_matrix* K, const bem_matrix* M_primal, const double* g_dev,
                   double* b_dev, bem_stream stream);
/* b = 1/2 M_h g + K_h g (eq. 4, u0 = 0) WITHOUT storing K_h ("fused K g"):
 * every entry of K_h is computed by the same kernels and quadrature as bem_assemble_K and is
 * multiplied by g at once; per (test row, trial tile) sums go to fixed partial slots (deterministic)
 * and are reduced in fixed order.  Multi-GPU: each rank sums its owned blocks, then one NCCL
 * all-reduce.  Meshes whose touching pairs fall outside regime A (alpha (h_X+h_Y)^2 / (4 min h_t) >= 4)
 * fall back to bem_assemble_K + bem_rhs.  g_dev, b_dev: device, N doubles, must not alias; stats
 * (host, may be NULL) receives the statistics of the K_h kernels (synchronises the stream).
 * Errors: BEM_E_INVALID (null / aliasing / options), BEM_E_STATE (M not primal), BEM_E_CUDA. */
bem_status bem_rhs_fused(const bem_mesh* mesh, const bem_quad_opts* opts, const bem_matrix* M_primal,
                         const double* g_dev, double* b_dev, bem_assembly_stats* stats, bem_stream stream);

/* ----------------------------------------------------------------- solver */
/* Initial potential term of eq. (4): b <- b - M_h^0 u0 with
 * M_h^0[(a,i), j] = <M_0 phi^1_j, phi^0_(a,i)>, u0 in S_h^1(Omega_h) given by its nodal values on a
 * triangulation of Omega (nodes_xy: n_nodes x 2, tris: n_tri x 3 node indices, both HOST; u0_dev,
 * b_dev: device).  Exact time integrals; qx Gauss points per boundary element, qt_far^2 /
 * qt_near^2 collapsed Gauss points per triangle, the log-singular first step by an apex-split rule
 * (reading R22); 0 selects the defaults 4 / 4 / 12 (<= 16 each).  M_h^0 is never
 * stored (its product only).  One process.  Errors: BEM_E_INVALID, BEM_E_STATE, BEM_E_CUDA. */
bem_status bem_rhs_initial(const bem_mesh* mesh, int n_nodes, const double* nodes_xy, int n_tri,
                           const int* tris, const double* u0_dev, int qx, int qt_far, int qt_near,
                           double* b_dev, bem_stream stream);
/* Representation formula in the space-time cylinder (eq. 2), u0 = 0:
 * u(x,t) = (Vt w)(x,t) - (W g)(x,t) for the Neumann density w (piecewise constant, as solved by
 * bem_solve_gmres) and the Dirichlet data g (nodal, as in bem_rhs).  Time integrals exact, Gauss
 * order per element from the distance (16 / 12 / 8).  pts_dev: npts x 3 doubles (x1, x2, t),
 * device; u_dev: npts doubles, device; w_dev, g_dev: N doubles, device.  Synchronises the stream.
 * Errors: BEM_E_INVALID (bad argument, or a point closer than h_max to Gamma), BEM_E_CUDA. */
bem_status bem_eval_potential(const bem_mesh* mesh, const double* w_dev, const double* g_dev,
                              long long npts, const double* pts_dev, double* u_dev, bem_stream stream);
/* Initial potential of the representation formula (eq. 2; row f2 with u0 != 0):
 * u_dev[k] += (M~_0 u0)(x_k, t_k) = int_Omega U*(x_k - y, t_k) u0_h(y) dy, U*(z,t) = alpha/(4 pi t)
 * exp(-alpha |z|^2 / (4t)), u0_h in S_h^1 on the triangulation (nodes_xy, tris: host, as in
 * bem_rhs_initial; u0_dev: device, one value per node).  Add it to the result of
 * bem_eval_potential for the full u = M~_0 u0 + Vt w - W g.  pts_dev: npts x 3 (x1, x2, t > 0),
 * device.  Collapsed Gauss (order 6) per triangle on ceil(l / ell)^2 cells, ell = sqrt(4 t/alpha)
 * (reading R24); triangles farther than 7 ell skipped.  Synchronises the stream.
 * Errors: BEM_E_INVALID (bad argument, index out of range, t <= 0), BEM_E_CUDA. */
bem_status bem_eval_potential_initial(const bem_mesh* mesh, int n_nodes, const double* nodes_xy, int n_tri,
                                      const int* tris, const double* u0_dev, long long npts,
                                      const double* pts_dev, double* u_dev, bem_stream stream);
/* Preconditioned full GMRES for V w = b with left preconditioner
 * C_V^{-1} = M^{-1} D M^{-T}; D and M are ignored when opts->precond == 0.
 * M must be BEM_MASS_DUAL_LUMPED for precond 1 and BEM_MASS_DUAL for precond 2.
 * x0 = 0.  b_dev, w_dev device vectors of length n.  res_hist_host: NULL or max_iter+1 doubles
 * (relative preconditioned residual estimates, [0] = 1).  Runs on `stream` (ordered after the work
 * already queued there, e.g. the right-hand side) and synchronises it once per iteration (the
 * Hessenberg column goes to the host for the Givens rotation).  Returns BEM_E_NOT_CONVERGED /
 * BEM_E_BREAKDOWN with w and the report filled. */
bem_status bem_solve_gmres(const bem_matrix* V, const bem_matrix* D, const bem_matrix* M,
                           const double* b_dev, double* w_dev, const bem_gmres_opts* opts,
                           bem_solve_report* report, double* res_hist_host, bem_stream stream);

/* ---------------------------------------------------------------- access */
/* dense window [r0, r0+nr) x [c0, c0+nc) into host_dst (row-major nr x nc); causality zeros
 * (b > a) and entries of blocks not owned by this rank read as 0. */
bem_status bem_matrix_get(const bem_matrix* A, long long r0, long long nr, long long c0,
                          long long nc, double* host_dst);
/* count sampled entries (rows_host[k], cols_host[k]) into out_host[k] */
bem_status bem_matrix_get_entries(const bem_matrix* A, long long count, const long long* rows_host,
                                  const long long* cols_host, double* out_host);
/* stored entries and bytes on this rank; kind: 0 V, 1 K, 2 D, 3 mass */
bem_status bem_matrix_info(const bem_matrix* A, int* kind, long long* entries, long long* bytes);
bem_status bem_matrix_stats(const bem_matrix* A, bem_assembly_stats* out);
void bem_matrix_destroy(bem_matrix* A);
/* Dense matrix storage is cached by the library after bem_matrix_destroy and reused (stream-
 * ordered) by the next assembly of a size that fits (<= 25% larger).  This returns every cached
 * block to the CUDA device pool (synchronising with the pending frees).  Always BEM_OK. */
bem_status bem_release_storage(void);

/* ---------------------------------------------------------- diagnostics */
/* device evaluation of the special functions used by the kernels (for the GPU pins):
 * which = 0 E1(x), 1 Ein(x), 2 (1+x)E1(x) - e^{-x}, 3 e^{-x}/x - 1/x - E1(x).
 * x_dev, out_dev: device arrays of length count. */
bem_status bem_eval_special(int which, long long count, const double* x_dev, double* out_dev,
                            bem_stream stream);
/* live FP64 DFMA rate of the current device (TFLOP/s, an FMA = 2 flops): a DFMA loop run back to
 * back for `seconds` (0 < seconds <= 60) on a private stream, the rate of the second half written
 * to *tflops_host.  The denominator of the assembly roofline in the power state of the moment (the
 * FP64-bound kernels run under the board power cap: clocks below the maximum).  Synchronous.
 * Errors: BEM_E_INVALID, BEM_E_CUDA. */
bem_status bem_diag_fp64_rate(double seconds, double* tflops_host);

#ifdef __cplusplus
}
#endif
#endif /* STBEM_H */
