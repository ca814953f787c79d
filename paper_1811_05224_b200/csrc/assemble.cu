// assemble.cu — CUDA sm_100a assembly of the dense block-lower-triangular space-time BEM
// matrices V_h, K_h, D_h in FP64.
//
// Time integrals are exact (special.cuh).  An entry of time cell (a,b) is the four-lag second
// difference of a double time antiderivative G evaluated at the time-node pairs (x,y):
//   A_ab = Phi(a+1,b) - Phi(a,b) - Phi(a+1,b+1) + Phi(a,b+1),   Phi(x,y) = int int G(t_x - t_y; r)
// (lags s = t_{a+1}-t_b, t_a-t_b, t_{a+1}-t_{b+1}, t_a-t_{b+1}, signs +,-,-,+).
//
// Kernels:
//   bulk   : cells with d = a - b >= 2, all spatial pairs.  One thread owns one spatial pair
//            (segment or half-segment pair) and a band of R test steps; it sweeps the trial
//            steps b and evaluates each node Phi(x, y) ONCE for the whole band (R+1 nodes per
//            column serve 2R corner uses), Gauss q_bulk x q_bulk in space.  Coalesced stores
//            along the trial element index j.
//   near   : cells d in {0,1}, pairs that do not touch; Gauss order from the distance ratio.
//   sing   : cells d in {0,1}, touching pairs (identical: 1-D reduction; shared vertex:
//            Duffy map), kernel split R(c) + P(c) ln c with the ln part integrated exactly by
//            log-weighted Gauss rules; one warp per entry, added onto the near result.
// D_h: thread per half-segment pair computing 5 moments (curl + 4 linear-shape normal
// moments), combined into dual-hat entries through shared memory (no atomics, deterministic).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.h"
#include "special.cuh"

namespace stb {

__constant__ double c_gx[QMAX + 1][QMAX];
__constant__ double c_gw[QMAX + 1][QMAX];
__constant__ double c_glw[QMAX + 1][QMAX];

static int g_rules_uploaded_dev = -1;
bem_status upload_rules() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (g_rules_uploaded_dev == dev) return BEM_OK;
  const Rules& R = host_rules();
  cudaError_t e;
  if ((e = cudaMemcpyToSymbol(c_gx, R.x, sizeof(R.x))) != cudaSuccess) return cuda_fail(e, "upload_rules");
  if ((e = cudaMemcpyToSymbol(c_gw, R.w, sizeof(R.w))) != cudaSuccess) return cuda_fail(e, "upload_rules");
  if ((e = cudaMemcpyToSymbol(c_glw, R.lw, sizeof(R.lw))) != cudaSuccess) return cuda_fail(e, "upload_rules");
  g_rules_uploaded_dev = dev;
  return BEM_OK;
}

// ------------------------------------------------------------------ common
struct BlockArgs {
  double* out;            // matrix storage
  const long long* poff;  // panel offsets for this block (index a - a0)
  int a0, a1, b0, b1;
  int ng;                 // entries per panel row block (N_Gamma)
  const double4* lag;     // (s, ln s, 1/s) per time-node pair
  int ldlag;              // n_steps + 1
  int sym;                // symmetric packed spatial blocks (only tiles ti <= tj are written)
  int nt;                 // sym: tiles per block side
  long long blk;          // sym: stored doubles per (a,b) block
  // product mode (K_h g, K_h not stored): trial vector and partial sums
  const double* g;
  double* part;           // partials of this block: [(a - a0) * ng + i] * pslots + slot
  long long pbase;
  int pslots;             // 2 * ntile + 6: bulk trial tiles, near trial tiles, touching records, k_kg_tab
  int ntile;              // ceil(ng / 32)
  int kgtab = 0;          // product mode: regime-A nodes with y <= x - 3 summed by k_kg_tab
  int nsub = 1;           // k_bulk_m (list form): CTAs per band sharing the listed blocks
  double ell;             // sqrt(4 min h_t / alpha): composite singular rules when h > ell
};

// sym: the caller guarantees sym_stored(i, j)
__device__ __forceinline__ double* entry_ptr(const BlockArgs& B, int a, int i, int b, int j) {
  if (B.sym) return B.out + B.poff[a - B.a0] + (long long)(b - B.b0) * B.blk + sym_in_block(i, j, B.nt);
  long long ld = pad4((long long)panel_nb(a, B.b0, B.b1) * B.ng);
  return B.out + B.poff[a - B.a0] + (long long)i * ld + (long long)(b - B.b0) * B.ng + j;
}

struct Lags {
  int n;
  double s[4], e[4], lns[4];
  double S;  // sum eps s over positive lags: h_a (d = 0), 0 (d >= 1)
};
__device__ __forceinline__ Lags make_lags(const double* __restrict__ t, int a, int b) {
  Lags L;
  L.n = 0;
  double s[4] = {t[a + 1] - t[b], t[a] - t[b], t[a + 1] - t[b + 1], t[a] - t[b + 1]};
  const double e[4] = {1.0, -1.0, -1.0, 1.0};
#pragma unroll
  for (int m = 0; m < 4; ++m)
    if (s[m] > 0.0) {
      L.s[L.n] = s[m];
      L.e[L.n] = e[m];
      L.lns[L.n] = log(s[m]);
      L.n++;
    }
  L.S = (a == b) ? (t[a + 1] - t[a]) : 0.0;
  return L;
}

__host__ __device__ inline double seg_dist(const Seg& X, const Seg& Y) {
  auto pd = [](double px, double py, const Seg& S) {
    double dx = px - S.ax, dy = py - S.ay;
    double f = dx * S.tx + dy * S.ty;
    f = fmin(fmax(f, 0.0), S.h);
    double qx = S.ax + f * S.tx - px, qy = S.ay + f * S.ty - py;
    return sqrt(qx * qx + qy * qy);
  };
  return fmin(fmin(pd(X.ax, X.ay, Y), pd(X.bx, X.by, Y)), fmin(pd(Y.ax, Y.ay, X), pd(Y.bx, Y.by, X)));
}
// Gauss order for non-touching pairs in cells d <= 1 (measured table)
// qfar: order for well-separated pairs (rho >= gap; bem_quad_opts q_near, default min(6, q_far + 1)),
// gap: bem_quad_opts near_gap (default 9)
__host__ __device__ inline int near_order(const Seg& X, const Seg& Y, int qfar, double gap) {
  double rho = seg_dist(X, Y) / fmax(X.h, Y.h);
  return rho < fmin(2.5, gap) ? 10 : (rho < fmin(5.0, gap) ? 8 : (rho < gap ? 6 : qfar));
}
// relation of elements p, q of a closed chain of n: 0 disjoint, 1 identical,
// 2 X.end == Y.start, 3 X.start == Y.end
__host__ __device__ inline int chain_rel(int p, int q, int n) {
  if (p == q) return 1;
  if ((p + 1) % n == q) return 2;
  if ((q + 1) % n == p) return 3;
  return 0;
}
__host__ __device__ inline bool collinear(const Seg& X, const Seg& Y) {
  double d0 = (X.ax - Y.ax) * Y.nx + (X.ay - Y.ay) * Y.ny;
  double d1 = (X.bx - Y.ax) * Y.nx + (X.by - Y.ay) * Y.ny;
  double tol = 1e-13 * fmax(X.h, Y.h);
  return fabs(d0) < tol && fabs(d1) < tol;
}

}  // namespace stb

#include "moments.cuh"
#include "potential.cuh"
#include "initial.cuh"

namespace stb {

// ================================================================= singular (touching) pairs
// split-form kernel at a point: R + P ln c, for the lag set (ker 0 H, 1 F, 2 Q without dot)
template <int KER>
__device__ __forceinline__ void split_RP(const Lags& Lg, double alpha, double c, double lnc,
                                         double& R, double& P) {
  double r = 0.0, pp = 0.0;
  for (int m = 0; m < Lg.n; ++m) {
    const double s = Lg.s[m], e = Lg.e[m];
    if (KER == 0) {
      r = fma(e, split_h_R(s, c, Lg.lns[m]), r);
      pp = fma(e, s + c, pp);
    } else if (KER == 1) {
      r = fma(e, split_f_R(s, c, Lg.lns[m]), r);
      pp += e;
    } else {
      r = fma(e, split_q_R(s, c, Lg.lns[m], lnc), r);
      pp += e;
    }
  }
  if (KER == 0) { R = r / (4.0 * STB_PI); P = -pp / (4.0 * STB_PI); }
  else if (KER == 1) { R = alpha * r / (4.0 * STB_PI); P = -alpha * pp / (4.0 * STB_PI); }
  else { R = alpha / (8.0 * STB_PI) * ((Lg.S != 0.0 ? Lg.S / c : 0.0) + r); P = alpha / (8.0 * STB_PI) * pp; }
}

__device__ __forceinline__ double lin(double v0, double v1, double f) { return fma(v1 - v0, f, v0); }

// warp-cooperative integral over a touching pair; the result is valid in all lanes
template <int KER>
__device__ double pair_touching(const Seg& X, const Seg& Y, int rel, const Lags& Lg, double alpha,
                                int n, double sx0, double sx1, double sy0, double sy1, double ell) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  // composite in the radial coordinate (and in eta for vertex pairs) when the elements are longer
  // than ell = sqrt(4 min h_t / alpha), the length on which the kernel varies at the smallest lag:
  // cell 0 keeps the log-weighted rule (scaled: ln rho = ln t - ln ns), the other cells take plain
  // Gauss with ln rho evaluated
  const double hmax = fmax(X.h, Y.h);
  const int ns = (ell > 0.0 && hmax > ell) ? min(24, (int)ceil(hmax / ell)) : 1;
  const double ins = 1.0 / ns, lnns = log((double)ns);
  if (rel == 1) {
    if (KER == 2) return 0.0;  // dot = 0 on a straight segment
    const double h = X.h;
    const double L0 = log(0.25 * alpha) + 2.0 * log(h);
    for (int idx = lane; idx < ns * n; idx += 32) {
      const int cell = idx / n, k = idx % n;
      const double rho = (cell + c_gx[n][k]) * ins, w = h * rho, len = h - w;
      // G(w) = int_0^{h-w} [Sx(v+w) Sy(v) + Sx(v) Sy(v+w)] dv (quadratic integrand: 2-point Gauss)
      double G = 0.0;
      for (int r = 0; r < 2; ++r) {
        const double v = len * c_gx[2][r];
        G += c_gw[2][r] * (lin(sx0, sx1, (v + w) / h) * lin(sy0, sy1, v / h) +
                           lin(sx0, sx1, v / h) * lin(sy0, sy1, (v + w) / h));
      }
      G *= len;
      const double c = 0.25 * alpha * w * w;
      double R, P;
      split_RP<KER>(Lg, alpha, c, log(c), R, P);
      const double wt = cell == 0 ? c_gw[n][k] * (R + P * (L0 - 2.0 * lnns)) + 2.0 * c_glw[n][k] * P
                                  : c_gw[n][k] * (R + P * (L0 + 2.0 * log(rho)));
      acc += G * ins * wt;
    }
    acc *= h;
  } else {
    const double h1 = X.h, h2 = Y.h;
    double e1x, e1y, e2x, e2y, sxV, sxF, syV, syF;
    if (rel == 2) {
      e1x = -X.tx; e1y = -X.ty; sxV = sx1; sxF = sx0;
      e2x = Y.tx; e2y = Y.ty; syV = sy0; syF = sy1;
    } else {
      e1x = X.tx; e1y = X.ty; sxV = sx0; sxF = sx1;
      e2x = -Y.tx; e2y = -Y.ty; syV = sy1; syF = sy0;
    }
    const double cth = e1x * e2x + e1y * e2y;
    const double e1n = e1x * Y.nx + e1y * Y.ny;
    if (KER == 2 && fabs(e1n) < 1e-14) return 0.0;
    const int ne = ns * acute_cells(cth);          // eta cells: composite (R24) x acute angle (R25)
    const double ine = 1.0 / ne;
    const int nq = ns * n, nqe = ne * n, npts = 2 * nqe * nq;
    for (int idx = lane; idx < npts; idx += 32) {
      const int tri = idx / (nqe * nq), ie = (idx / nq) % nqe, ir = idx % nq;
      const int rc = ir / n, rk = ir % n;
      const double eta = (ie / n + c_gx[n][ie % n]) * ine, weta = c_gw[n][ie % n] * ine;
      const double rho = (rc + c_gx[n][rk]) * ins;
      const double A = tri == 0 ? (h1 * h1 + h2 * h2 * eta * eta - 2.0 * h1 * h2 * eta * cth)
                                : (h1 * h1 * eta * eta + h2 * h2 - 2.0 * h1 * h2 * eta * cth);
      const double u = tri == 0 ? h1 * rho : h1 * rho * eta;
      const double v = tri == 0 ? h2 * rho * eta : h2 * rho;
      double f = lin(sxV, sxF, u / h1) * lin(syV, syF, v / h2) * h1 * h2 * rho;
      if (KER == 2) f *= u * e1n;
      const double c = 0.25 * alpha * rho * rho * A;
      const double lnA = log(0.25 * alpha * A);
      double R, P;
      split_RP<KER>(Lg, alpha, c, lnA + 2.0 * log(rho), R, P);
      const double wr = rc == 0 ? c_gw[n][rk] * (R + P * (lnA - 2.0 * lnns)) + 2.0 * c_glw[n][rk] * P
                                : c_gw[n][rk] * (R + P * (lnA + 2.0 * log(rho)));
      acc += weta * f * ins * wr;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

// one warp per (cell, entry) with touching pairs: adds their contribution to the entry
template <int KIND>
__global__ void __launch_bounds__(128) k_sing(BlockArgs B, const Seg* __restrict__ seg,
                                              const Seg* __restrict__ half,
                                              const Dual* __restrict__ dual,
                                              const double* __restrict__ t, double alpha, int nsing,
                                              long long nwarps) {
  const long long gw = (long long)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (gw >= nwarps) return;
  const int ng = B.ng;
  const int per_row = (KIND == STB_V) ? 3 : (KIND == STB_K ? 4 : 5);
  const int off = (int)(gw % per_row);
  const long long r1 = gw / per_row;
  const int i = (int)(r1 % ng);
  const int cell = (int)(r1 / ng);
  const int a = B.a0 + cell / 2, b = a - (cell % 2);
  if (a >= B.a1 || b < B.b0 || b >= B.b1) return;
  const Lags Lg = make_lags(t, a, b);
  double add = 0.0;
  int jcol;
  if (KIND == STB_V) {
    jcol = ((i + off - 1) % ng + ng) % ng;       // i-1, i, i+1
    const int rel = chain_rel(i, jcol, ng);
    add = pair_touching<0>(seg[i], seg[jcol], rel, Lg, alpha, nsing, 1, 1, 1, 1, B.ell);
  } else if (KIND == STB_K) {
    jcol = ((i + off - 1) % ng + ng) % ng;       // n = i-1 .. i+2
    const int jl = (jcol - 1 + ng) % ng;
    const int rl = chain_rel(i, jl, ng), rr = chain_rel(i, jcol, ng);
    if (rl) add += pair_touching<2>(seg[i], seg[jl], rl, Lg, alpha, nsing, 1, 1, 0, 1, B.ell);
    if (rr) add += pair_touching<2>(seg[i], seg[jcol], rr, Lg, alpha, nsing, 1, 1, 1, 0, B.ell);
  } else {
    const int l = i;
    jcol = ((l + off - 2) % ng + ng) % ng;       // k = l-2 .. l+2
    const int k = jcol, nh = 2 * ng;
    const Dual dl = dual[l], dk = dual[k];
    const double dvl[4] = {1.0 / dl.Lm, 1.0 / dl.Lm, -1.0 / dl.Lp, -1.0 / dl.Lp};
    const double dvk[4] = {1.0 / dk.Lm, 1.0 / dk.Lm, -1.0 / dk.Lp, -1.0 / dk.Lp};
    const double vl[4][2] = {{0.0, dl.vm}, {dl.vm, 1.0}, {1.0, dl.vp}, {dl.vp, 0.0}};
    const double vk[4][2] = {{0.0, dk.vm}, {dk.vm, 1.0}, {1.0, dk.vp}, {dk.vp, 0.0}};
    for (int m = 0; m < 4; ++m)
      for (int nn_ = 0; nn_ < 4; ++nn_) {
        const int p = ((2 * l - 1 + m) % nh + nh) % nh, q = ((2 * k - 1 + nn_) % nh + nh) % nh;
        const int rel = chain_rel(p, q, nh);
        if (!rel) continue;
        const Seg X = half[p], Y = half[q];
        add += dvl[m] * dvk[nn_] * pair_touching<0>(X, Y, rel, Lg, alpha, nsing, 1, 1, 1, 1, B.ell);
        const double nn = X.nx * Y.nx + X.ny * Y.ny;
        if (nn != 0.0)
          add += nn * pair_touching<1>(X, Y, rel, Lg, alpha, nsing, vl[m][0], vl[m][1], vk[nn_][0], vk[nn_][1], B.ell);
      }
  }
  if ((threadIdx.x & 31) == 0 && !(B.sym && !sym_stored(i, jcol))) *entry_ptr(B, a, i, b, jcol) += add;
}

// ================================================================= launch
#ifndef STB_NEAR_CHUNK
#define STB_NEAR_CHUNK 32   // test steps per k_near_m CTA (the per-pair setup is paid once per chunk)
#endif
static int max_smem_optin() {
  static int v = 0;
  if (!v) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || v <= 0) v = 48 * 1024;
  }
  return v;
}
// which: 0 bulk cells (k_bulk_m), 1 near cells (k_near_m)
template <int KIND, int R, bool PROD, bool MULTI>
static void launch_bulk_t(const BlockArgs& BA, const MomArgs& M, dim3 grid, cudaStream_t st, BulkList L) {
  constexpr size_t smem = bulk_smem_bytes<KIND, R>();
  static bool attr = false;   // per template instance
  if (!attr) {
    cudaFuncSetAttribute(k_bulk_m<KIND, R, PROD, MULTI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_bulk_m<KIND, R, PROD, MULTI><<<grid, 128, smem, st>>>(BA, L, M);
}
// one block: its geometry in BA (the single-block kernel); several: the list L
template <int KIND, int R, bool PROD>
static void launch_bulk(const BlockArgs& BA, const MomArgs& M, dim3 grid, cudaStream_t st, BulkList L) {
  // the list kernel also for one block of the K_h g product: its register allocation spills less
  // there (stack 32 vs 72 B; C5 bulk 15.2 vs 15.7 ms), the stored kinds keep the one-block kernel
  if (L.n > 1 || (KIND == STB_K && PROD)) launch_bulk_t<KIND, R, PROD, true>(BA, M, grid, st, L);
  else launch_bulk_t<KIND, R, PROD, false>(BA, M, grid, st, L);
}
template <int KIND, bool PROD = false>
static void launch_kind(int which, const BlockArgs& BA, const MomArgs& M, int ng, int nband_or_chunk,
                        int nz, cudaStream_t st, BulkList L = BulkList{nullptr, 0}, int R_ = 0,
                        const NearItem* items = nullptr) {
  dim3 grid((ng + 31) / 32, (ng + 3) / 4, nz);
  BlockArgs B2 = BA;
  if (which == 0 && L.n > 1) {
    // the listed blocks split over nsub CTAs per band until the grid holds ~16 waves of 2 CTAs / SM
    const long long per_z = (long long)grid.x * grid.y * nz;
    int nsub = 1;
    while (nsub < L.n && per_z * nsub < 16LL * 2 * 148) nsub *= 2;
    B2.nsub = std::min(nsub, L.n);
    grid.z = nz * B2.nsub;
  }
  if (which == 0 && KIND != STB_D && R_ == 8) {
    launch_bulk<KIND, 8, PROD>(B2, M, grid, st, L);
  } else if (which == 0) {
    launch_bulk<KIND, bulk_r<KIND>(), PROD>(B2, M, grid, st, L);
  }
  else k_near_m<KIND, PROD><<<grid, 128, 0, st>>>(BA, M, nband_or_chunk, items);
  count_launch();
}

// product mode: y[a ng + i] = sum over the owned blocks containing test step a of the partials
// (bulk trial tiles, near trial tiles, touching records) in fixed order
__global__ void k_prod_reduce(const double* __restrict__ part, const int* __restrict__ rstart,
                              const long long* __restrict__ roff, int ng, int nt, int pslots,
                              double* __restrict__ y) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (long long)ng * nt) return;
  const int a = (int)(r / ng);
  double s = 0.0;
  for (int k = rstart[a]; k < rstart[a + 1]; ++k) {
    const double* p = part + roff[k] + r * pslots;
    for (int q = 0; q < pslots; ++q) s += p[q];
  }
  y[r] = s;
}
// distributed records: staging chunk c = [nfc fields x cs pairs] -> field-major rec[f npairs + p]
__global__ void k_rec_reorder(const double* __restrict__ stage, double* __restrict__ rec, int nfc, long long npairs,
                              long long cs) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (long long)nfc * npairs) return;
  const long long f = k / npairs, p = k - f * npairs, c = p / cs;
  rec[k] = stage[c * nfc * cs + f * cs + (p - c * cs)];
}
template <int KIND>
static void launch_records(const MomArgs& MB, const MomArgs& MN, const MomArgs* MS, int q_sing,
                           cudaStream_t st) {
  const unsigned nblk = (unsigned)((MB.p_hi - MB.p_lo + 127) / 128);   // this rank's pairs
  // D_h near records: the pairs with touching or close half-segment sub-pairs (distance-dependent
  // orders, skipped sub-pairs) warp per pair, the others thread per pair (k_records near_special)
  k_records<KIND, false><<<nblk, 128, 0, st>>>(MB);
  if (KIND == STB_D) {
    cudaMemsetAsync(MN.list, 0, sizeof(int), st);
    k_records<KIND, true, true><<<nblk, 128, 0, st>>>(MN);
    static int nsm = 0;
    if (!nsm) {
      int dev = 0;
      cudaGetDevice(&dev);
      if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || nsm <= 0) nsm = 148;
    }
    k_records_warp<KIND, true><<<nsm * 2, 128, 0, st>>>(MN);   // persistent: the resident warps walk the list
    count_launch();
  } else {
    k_records<KIND, true><<<nblk, 128, 0, st>>>(MN);
  }
  count_launch(2);
  if (MS) {
    k_sing_records<KIND><<<(unsigned)((MS->npairs * 32 + 127) / 128), 128, 0, st>>>(*MS, q_sing);   // warp per record
    count_launch();
  }
}
template <int KIND, bool PROD = false>
static void launch_sing_m(const BlockArgs& BA, const MomArgs& MS, int nsteps, cudaStream_t st) {
  const int chunk = 16;
  dim3 grid((unsigned)((MS.npairs + 127) / 128), (nsteps + chunk - 1) / chunk);
  k_sing_m<KIND, PROD><<<grid, 128, 0, st>>>(BA, MS, chunk);
  count_launch();
}

// time nodes evaluated per entry-level pair by the bulk kernel of one block (host count,
// same loop bounds as k_bulk_m)
static long long bulk_nodes(const Block& b, int R) {
  long long nodes = 0;
  const int nband = (b.a1 - b.a0 + R - 1) / R;
  for (int band = 0; band < nband; ++band) {
    const int r_hi = b.a1 - R * band, r_lo = std::max(b.a0, r_hi - R);
    const int bmax = std::min(b.b1 - 1, r_hi - 1 - 2);
    if (bmax < b.b0) continue;
    for (int y = b.b0; y <= bmax + 1; ++y)
      for (int x = r_lo; x <= r_hi; ++x)
        if (x > y) ++nodes;
  }
  return nodes;
}

bem_status resolve_quad(int kind, const bem_mesh* m, const bem_quad_opts* o, const char* where, QuadCfg* out) {
  QuadCfg q;
  q.q_far = (o && o->q_far > 0) ? o->q_far : (kind == STB_D ? m->q_bulk_d : m->q_bulk);
  q.q_near = (o && o->q_near > 0) ? o->q_near : std::min(6, q.q_far + 1);
  q.near_gap = (o && o->near_gap > 0) ? (double)o->near_gap : 9.0;
  q.q_sing = (o && o->q_sing > 0) ? o->q_sing : 16;
  q.flags = o ? o->flags : 0;
  if (o && (o->q_far < 0 || o->q_near < 0 || o->near_gap < 0 || o->q_sing < 0)) {
    set_error(std::string(where) + ": negative quadrature option");
    return BEM_E_INVALID;
  }
  if (q.q_far < 3 || q.q_far > 8 || q.q_far == 7) { set_error(std::string(where) + ": q_far must be one of 3,4,5,6,8"); return BEM_E_INVALID; }
  if (q.q_near < 3 || q.q_near > QMAX) { set_error(std::string(where) + ": q_near must be in [3,16]"); return BEM_E_INVALID; }
  if (q.q_sing < 4 || q.q_sing > QSING_MAX) { set_error(std::string(where) + ": q_sing must be in [4,16]"); return BEM_E_INVALID; }
  if (q.flags & ~(BEM_QUAD_LEGACY_SING | BEM_QUAD_FULL_STORAGE | BEM_QUAD_KG_ENTRYWISE)) { set_error(std::string(where) + ": unknown flags"); return BEM_E_INVALID; }
  *out = q;
  return BEM_OK;
}

bem_status launch_assembly(int kind, const bem_mesh* m, bem_matrix* A, const QuadCfg& qc,
                           cudaStream_t st, const double* prod_g, double* prod_y) {
  const int q_bulk = qc.q_far, q_sing = qc.q_sing, flags = qc.flags;
  const int ng = m->ng;
  const bool prod = prod_g != nullptr;
  if (prod && kind != STB_K) { set_error("assemble: product mode is K_h only"); return BEM_E_INVALID; }
  // the touching-pair enumeration (offsets J = I + jo - 2) needs distinct neighbours: below six
  // elements two offsets name the same pair and its contribution would be counted twice
  if (ng < 6) { set_error("assemble: N_Gamma >= 6 required"); return BEM_E_INVALID; }
  mesh_wait(m, st);
  long long* d_poff = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&d_poff, sizeof(long long) * std::max<size_t>(1, A->poff.size()), st);
  if (e != cudaSuccess) return cuda_fail(e, "assemble/poff");
  e = cudaMemcpyAsync(d_poff, A->poff.data(), sizeof(long long) * A->poff.size(), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) { cudaFreeAsync(d_poff, st); return cuda_fail(e, "assemble/poff copy"); }
  // pair records (bulk order and near orders) and regime counters, stream-ordered
  const long long npairs = (long long)ng * ng;
  const long long nsrec = 5LL * ng;
  const int nf = kind == STB_D ? rec_fields<STB_D>() : rec_fields<STB_V>();
  const int nfn = kind == STB_D ? rec_fields_near<STB_D>() : rec_fields_near<STB_V>();   // + regime B2
  // touching pairs through moment records (regime A) when every touching sub-pair satisfies
  // c_max / min h_t < 4 with c_max <= alpha (h_X + h_Y)^2 / 4; otherwise the per-lag k_sing
  const bool fused_sing = touching_records_ok(kind, m, flags);
  A->fused_sing = fused_sing ? 1 : 0;
  if (prod && !fused_sing) { set_error("assemble: product mode needs the touching-pair records"); return BEM_E_STATE; }
  // product mode: partial sums per block, row (a, i) and slot (bulk / near trial tiles, records)
  const int ntile = (ng + 31) / 32, pslots = 2 * ntile + 6;
  double* d_part = nullptr;
  size_t part_bytes = 0;
  std::vector<long long> pbase(blocks_of(A).size(), 0);
  if (prod) {
    long long tot = 0;
    for (size_t bi = 0; bi < blocks_of(A).size(); ++bi) {
      pbase[bi] = tot;
      tot += (long long)(blocks_of(A)[bi].a1 - blocks_of(A)[bi].a0) * ng * pslots;
    }
    part_bytes = sizeof(double) * std::max<long long>(1, tot);
    if ((e = storage_acquire(m->device, part_bytes, st, (void**)&d_part)) != cudaSuccess ||
        (e = cudaMemsetAsync(d_part, 0, part_bytes, st)) != cudaSuccess) {
      cudaFreeAsync(d_poff, st);
      return cuda_fail(e, "assemble/partials");
    }
  }
  double* d_rec = nullptr;
  unsigned long long* d_ctr = nullptr;
  int* d_list = nullptr;   // D_h near records: the near_special pairs
  if (kind == STB_D && (e = cudaMallocAsync((void**)&d_list, sizeof(int) * (npairs + 1), st)) != cudaSuccess) {
    if (d_part) storage_release(m->device, d_part, part_bytes, st);
    cudaFreeAsync(d_poff, st);
    return cuda_fail(e, "assemble/list");
  }
  // pair records, field-major with stride npairs: [bulk fields | near fields | touching records].
  // With G = record_ranks > 1 ranks, rank r computes the pairs of test segments [r rpc, (r+1) rpc)
  // into chunk r of a staging buffer (chunk c = [bulk | near fields], stride cs = rpc N_Gamma), an
  // in-place all-gather completes the other chunks and one kernel reorders them into the layout
  // above (the bulk and near kernels address a record as rec + pair: a chunked address costs them
  // registers)
  const int G = record_ranks(m);
  const int rpc = (ng + G - 1) / G;                    // test segments per chunk
  const long long cs = (long long)rpc * ng;
  const long long rec_main = (long long)(nf + nfn) * npairs;
  const size_t rec_bytes = sizeof(double) * ((size_t)rec_main + (size_t)nf * nsrec);
  const size_t stage_bytes = G > 1 ? sizeof(double) * (size_t)(nf + nfn) * cs * G : 0;
  double* d_stage = nullptr;
  if (G > 1 && (e = storage_acquire(m->device, stage_bytes, st, (void**)&d_stage)) != cudaSuccess) {
    if (d_part) storage_release(m->device, d_part, part_bytes, st);
    if (d_list) cudaFreeAsync(d_list, st);
    cudaFreeAsync(d_poff, st);
    return cuda_fail(e, "assemble/record staging");
  }
  if ((e = storage_acquire(m->device, rec_bytes, st, (void**)&d_rec)) != cudaSuccess ||
      (e = cudaMallocAsync((void**)&d_ctr, sizeof(unsigned long long) * CTR_N, st)) != cudaSuccess ||
      (e = cudaMemsetAsync(d_ctr, 0, sizeof(unsigned long long) * CTR_N, st)) != cudaSuccess) {
    if (d_rec) storage_release(m->device, d_rec, rec_bytes, st);
    if (d_stage) storage_release(m->device, d_stage, stage_bytes, st);
    if (d_part) storage_release(m->device, d_part, part_bytes, st);
    if (d_list) cudaFreeAsync(d_list, st);
    cudaFreeAsync(d_poff, st);
    return cuda_fail(e, "assemble/records");
  }
  // CUDA events on the launching stream around each kernel family, per block; read (with the
  // counters) on the first statistics query, so that the assembly never blocks the host
  A->d_ctr = d_ctr;
  A->stats_ready = false;
  std::vector<cudaEvent_t>& ev = A->ev;
  auto mark = [&]() {
    cudaEvent_t x;
    cudaEventCreate(&x);
    cudaEventRecord(x, st);
    ev.push_back(x);
  };
  std::vector<int>& fam = A->ev_fam;  // family of the interval ending at ev[k+1]: 0 bulk, 1 near, 2 sing, 3 records
  A->q_bulk = q_bulk;
  A->q_sing = q_sing;
  A->launches = 0;
  const int qfar = qc.q_near;
  MomArgs MB{d_rec, npairs, m->d_seg, m->d_half, m->d_dual, m->alpha, ng, q_bulk, qfar, d_ctr};
  MB.near_gap = qc.near_gap;
  MB.cs = npairs;
  MB.rpc = ng;
  MB.nfc = nf + nfn;
  MB.p_lo = 0;
  MB.p_hi = npairs;
  MB.ell = m->htmin > 0.0 ? std::sqrt(4.0 * m->htmin / m->alpha) : 0.0;
  MomArgs MN = MB;
  MN.rec = d_rec + (long long)nf * npairs;
  MN.list = d_list;
  // the near cells' nodes: s = t_{a+1} - t_a and t_{a+1} - t_{a-1} (and t_a - t_{a-1})
  {
    double smin = 1e300, smax = 0.0;
    for (int a = 0; a < m->nt; ++a) {
      smin = std::min(smin, m->t[a + 1] - m->t[a]);
      smax = std::max(smax, m->t[a + 1] - m->t[a > 0 ? a - 1 : a]);
    }
    MN.u_near[0] = 1.0 / smax;
    MN.u_near[1] = 1.0 / smin;
  }
  MN.counters = d_ctr + 5;
  MomArgs MS = MB;
  MS.rec = d_rec + rec_main;
  MS.npairs = MS.cs = MS.p_hi = nsrec;
  MS.p_lo = 0;
  MS.counters = d_ctr + 10;
  // the records kernels' arguments: this rank's chunk of the staging buffer when distributed
  MomArgs MBr = MB, MNr = MN;
  if (G > 1) {
    MBr.rec = d_stage;
    MNr.rec = d_stage + (long long)nf * cs;
    MBr.cs = MNr.cs = cs;
    MBr.rpc = MNr.rpc = rpc;
    MBr.p_lo = MNr.p_lo = std::min(npairs, (long long)m->comm->rank * cs);
    MBr.p_hi = MNr.p_hi = std::min(npairs, MBr.p_lo + cs);
  }
  mark();
  if (kind == STB_V) launch_records<STB_V>(MBr, MNr, fused_sing ? &MS : nullptr, q_sing, st);
  else if (kind == STB_K) launch_records<STB_K>(MBr, MNr, fused_sing ? &MS : nullptr, q_sing, st);
  else launch_records<STB_D>(MBr, MNr, fused_sing ? &MS : nullptr, q_sing, st);
  if (G > 1) {
    bem_status gs = allgather_chunks(m, d_stage, (long long)(nf + nfn) * cs, st);
    if (gs == BEM_OK) {
      const long long tot = (long long)(nf + nfn) * npairs;
      k_rec_reorder<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(d_stage, d_rec, nf + nfn, npairs, cs);
      count_launch();
    }
    storage_release(m->device, d_stage, stage_bytes, st);
    if (gs != BEM_OK) {
      storage_release(m->device, d_rec, rec_bytes, st);
      if (d_part) storage_release(m->device, d_part, part_bytes, st);
      if (d_list) cudaFreeAsync(d_list, st);
      cudaFreeAsync(d_poff, st);
      return gs;
    }
  }
  mark();
  fam.push_back(3);
  A->launches += 2;
  A->nodes_expected = 0;
  long long npairs_computed = npairs;   // sym: the pairs (I, J) of the upper tile triangle
  if (A->sym) {
    npairs_computed = 0;
    for (int i = 0; i < ng; ++i) npairs_computed += ng - (i / SYM_TS) * SYM_TS;
  }
  // bulk cells: ONE launch over all owned blocks (band z of every block in each CTA: the per-pair
  // setup -- records, regime-B coefficients -- is paid once per CTA; a rank of the cyclic plan owns
  // ~P/2 + 1 small blocks, which per-block launches left setup-bound)
  // band height of k_bulk_m: every band evaluates R + 1 node rows per trial column whatever its
  // height, so the blocks' row counts decide: V_h and K_h g take 8 (one spill-penalised kernel, +4%
  // per node on C5) when that needs fewer node rows than 7 -- a rank's small blocks of 2^k steps
  // (16 steps: bands 7 + 7 + 2 cost 24 rows per column against 2 x 9 = 18); D_h always 8
  auto node_rows = [&](int R) {
    double c = 0.0;
    for (size_t bi = 0; bi < blocks_of(A).size(); ++bi) {
      const Block& b = blocks_of(A)[bi];
      const int nband = (b.a1 - b.a0 + R - 1) / R;
      for (int band = 0; band < nband; ++band) {
        const int r_hi = b.a1 - R * band;
        const int bmax = std::min(b.b1 - 1, r_hi - 1 - 2);
        if (bmax >= b.b0) c += (double)(R + 1) * (bmax + 2 - b.b0);
      }
    }
    return c;
  };
  const int Rb = (kind == STB_D && !prod) ? bulk_r<STB_D>()
                 : (node_rows(8) * 1.04 < node_rows(7) ? 8 : bulk_r<STB_V>());
  A->bulk_r = Rb;
  {
    std::vector<BulkBlock> bl;
    int nzmax = 0;
    for (size_t bi = 0; bi < blocks_of(A).size(); ++bi) {
      const Block& blk = blocks_of(A)[bi];
      if (blk.a1 - 1 - blk.b0 < 2) continue;    // no cell with d >= 2
      bl.push_back(BulkBlock{d_poff + A->poff_base[bi], blk.a0, blk.a1, blk.b0, blk.b1, pbase[bi]});
      nzmax = std::max(nzmax, (blk.a1 - blk.a0 + Rb - 1) / Rb);
      A->nodes_expected += bulk_nodes(blk, Rb) * npairs_computed;
    }
    // the blocks of one trial range contiguous (k_kg_tab shares a trial slice's tables between them);
    // every kernel takes the list in any order (per-block partial slots)
    std::stable_sort(bl.begin(), bl.end(), [](const BulkBlock& x, const BulkBlock& y) {
      return x.b0 != y.b0 ? x.b0 < y.b0 : (x.b1 != y.b1 ? x.b1 < y.b1 : x.a0 < y.a0);
    });
    std::vector<int> gsv;   // group starts in bl (+ end)
    for (size_t k = 0; k < bl.size(); ++k)
      if (k == 0 || bl[k].b0 != bl[k - 1].b0 || bl[k].b1 != bl[k - 1].b1) gsv.push_back((int)k);
    gsv.push_back((int)bl.size());
    if (!bl.empty()) {
      BulkBlock* d_bl = nullptr;
      if ((e = cudaMallocAsync((void**)&d_bl, sizeof(BulkBlock) * bl.size(), st)) != cudaSuccess ||
          (e = cudaMemcpyAsync(d_bl, bl.data(), sizeof(BulkBlock) * bl.size(), cudaMemcpyHostToDevice, st)) != cudaSuccess)
        return cuda_fail(e, "assemble/bulk list");
      BlockArgs BA;
      BA.out = A->data;
      BA.poff = nullptr;
      BA.a0 = BA.a1 = BA.b0 = BA.b1 = 0;
      BA.ng = ng;
      BA.lag = m->d_lag;
      BA.ldlag = m->nt + 1;
      BA.sym = A->sym;
      BA.nt = sym_nt(ng);
      BA.blk = A->blk_elems;
      BA.g = prod_g;
      BA.part = d_part;
      BA.pbase = 0;
      BA.pslots = pslots;
      BA.ntile = ntile;
      BA.ell = MB.ell;
      // K_h g: the regime-A nodes of the interior columns as trial-moment sums (k_kg_tab) when its
      // shared-memory tables fit (N_Gamma up to ~590) and not disabled by BEM_QUAD_KG_ENTRYWISE
      int nxmax = 0;   // test nodes of the largest trial-range group
      for (size_t gi = 0; gi + 1 < gsv.size(); ++gi) {
        int nx = 0;
        for (int k = gsv[gi]; k < gsv[gi + 1]; ++k) nx += bl[k].a1 - bl[k].a0 + 1;
        nxmax = std::max(nxmax, nx);
      }
      const size_t tab_smem = kg_tab_smem(ng, nxmax);
      BA.kgtab = prod && !(flags & BEM_QUAD_KG_ENTRYWISE) && tab_smem + 2048 <= (size_t)max_smem_optin() &&
                 nxmax <= KGT_NODE && ng <= KGT_THREADS && kg_ch(ng) <= 20 ? 1 : 0;
      A->kg_tab = BA.kgtab;
      if (bl.size() == 1) {   // the single-block kernel takes the block from its parameters
        BA.poff = bl[0].poff;
        BA.a0 = bl[0].a0; BA.a1 = bl[0].a1; BA.b0 = bl[0].b0; BA.b1 = bl[0].b1;
        BA.pbase = bl[0].pbase;
      }
      const BulkList L{d_bl, (int)bl.size()};
      if (prod) {
        launch_kind<STB_K, true>(0, BA, MB, ng, nzmax, nzmax, st, L, Rb);
        if (BA.kgtab) {
          static bool attr = false;
          if (!attr) {
            cudaFuncSetAttribute(k_kg_tab<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem_optin() - 2048);
            cudaFuncSetAttribute(k_kg_tab<20>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem_optin() - 2048);
            attr = true;
          }
          int* d_gs = nullptr;
          if ((e = cudaMallocAsync((void**)&d_gs, sizeof(int) * gsv.size(), st)) != cudaSuccess ||
              (e = cudaMemcpyAsync(d_gs, gsv.data(), sizeof(int) * gsv.size(), cudaMemcpyHostToDevice, st)) != cudaSuccess)
          {
            cudaFreeAsync(d_bl, st);
            return cuda_fail(e, "assemble/table groups");
          }
          const dim3 tg((unsigned)ng, (unsigned)(gsv.size() - 1));
          if (kg_chm(ng) == 12) k_kg_tab<12><<<tg, KGT_THREADS, tab_smem, st>>>(BA, L, MB, nxmax, d_gs);
          else k_kg_tab<20><<<tg, KGT_THREADS, tab_smem, st>>>(BA, L, MB, nxmax, d_gs);
          cudaFreeAsync(d_gs, st);
          count_launch();
          A->launches++;
          // algorithmic flops of the table: per (i, trial step y) of a trial-range group the 22 prefix
          // scans (one FMA per pair and field), per covered node (x, y, i) the 21-term chain and ln s term
          for (size_t gi = 0; gi + 1 < gsv.size(); ++gi) {
            const BulkBlock& g0 = bl[gsv[gi]];
            int a1max = g0.a1;
            for (int k = gsv[gi]; k < gsv[gi + 1]; ++k) a1max = std::max(a1max, bl[k].a1);
            for (int y = g0.b0; y <= std::min(g0.b1, a1max - 3); ++y) {
              double nodes = 0.0;
              for (int k = gsv[gi]; k < gsv[gi + 1]; ++k)
                if (y <= std::min(bl[k].b1, bl[k].a1 - 3)) nodes += std::max(0, bl[k].a1 - std::max(bl[k].a0, y + 3) + 1);
              A->flops_tab += (double)ng * (2.0 * KGT_NF * ng + 44.0 * nodes);
            }
          }
        }
      } else if (kind == STB_V) launch_kind<STB_V>(0, BA, MB, ng, nzmax, nzmax, st, L, Rb);
      else if (kind == STB_K) launch_kind<STB_K>(0, BA, MB, ng, nzmax, nzmax, st, L, Rb);
      else launch_kind<STB_D>(0, BA, MB, ng, nzmax, nzmax, st, L, Rb);
      mark();
      fam.push_back(0);
      A->launches++;
      cudaFreeAsync(d_bl, st);
    }
  }
  // near cells of every owned block in ONE launch (grid z = (block, chunk of its test steps)): a rank
  // of the cyclic plan owns several small blocks, whose per-block launches were each setup-bound
  NearItem* d_items = nullptr;
  {
    std::vector<NearItem> items;
    const int chunk = STB_NEAR_CHUNK;
    for (size_t bi = 0; bi < blocks_of(A).size(); ++bi) {
      const Block& blk = blocks_of(A)[bi];
      if (!(blk.b1 - 1 >= blk.a0 - 1 && blk.b0 <= blk.a1 - 1)) continue;
      for (int a = blk.a0; a < blk.a1; a += chunk)
        items.push_back(NearItem{BulkBlock{d_poff + A->poff_base[bi], blk.a0, blk.a1, blk.b0, blk.b1, pbase[bi]},
                                 a, std::min(blk.a1, a + chunk)});
    }
    if (items.size() > 1) {
      if ((e = cudaMallocAsync((void**)&d_items, sizeof(NearItem) * items.size(), st)) != cudaSuccess ||
          (e = cudaMemcpyAsync(d_items, items.data(), sizeof(NearItem) * items.size(), cudaMemcpyHostToDevice, st)) != cudaSuccess)
        return cuda_fail(e, "assemble/near items");
      BlockArgs BA;
      BA.out = A->data;
      BA.poff = nullptr;
      BA.a0 = BA.a1 = BA.b0 = BA.b1 = 0;
      BA.ng = ng;
      BA.lag = m->d_lag;
      BA.ldlag = m->nt + 1;
      BA.sym = A->sym;
      BA.nt = sym_nt(ng);
      BA.blk = A->blk_elems;
      BA.g = prod_g;
      BA.part = d_part;
      BA.pbase = 0;
      BA.pslots = pslots;
      BA.ntile = ntile;
      BA.ell = MB.ell;
      const int nz = (int)items.size();
      if (prod) launch_kind<STB_K, true>(1, BA, MN, ng, chunk, nz, st, BulkList{nullptr, 0}, 0, d_items);
      else if (kind == STB_V) launch_kind<STB_V>(1, BA, MN, ng, chunk, nz, st, BulkList{nullptr, 0}, 0, d_items);
      else if (kind == STB_K) launch_kind<STB_K>(1, BA, MN, ng, chunk, nz, st, BulkList{nullptr, 0}, 0, d_items);
      else launch_kind<STB_D>(1, BA, MN, ng, chunk, nz, st, BulkList{nullptr, 0}, 0, d_items);
      mark();
      fam.push_back(1);
      A->launches++;
      cudaFreeAsync(d_items, st);
    }
  }
  for (size_t bi = 0; bi < blocks_of(A).size(); ++bi) {
    const Block& blk = blocks_of(A)[bi];
    BlockArgs BA;
    BA.out = A->data;
    BA.poff = d_poff + A->poff_base[bi];
    BA.a0 = blk.a0; BA.a1 = blk.a1; BA.b0 = blk.b0; BA.b1 = blk.b1;
    BA.ng = ng;
    BA.lag = m->d_lag;
    BA.ldlag = m->nt + 1;
    BA.sym = A->sym;
    BA.nt = sym_nt(ng);
    BA.blk = A->blk_elems;
    BA.g = prod_g;
    BA.part = d_part;
    BA.pbase = pbase[bi];
    BA.pslots = pslots;
    BA.ntile = ntile;
    BA.ell = MB.ell;
    const bool has_near = blk.b1 - 1 >= blk.a0 - 1 && blk.b0 <= blk.a1 - 1;
    if (has_near) {
      if (!d_items) {   // a single slab: the one-block form
        const int chunk = STB_NEAR_CHUNK;
        const int nz = (blk.a1 - blk.a0 + chunk - 1) / chunk;
        if (prod) launch_kind<STB_K, true>(1, BA, MN, ng, chunk, nz, st);
        else if (kind == STB_V) launch_kind<STB_V>(1, BA, MN, ng, chunk, nz, st);
        else if (kind == STB_K) launch_kind<STB_K>(1, BA, MN, ng, chunk, nz, st);
        else launch_kind<STB_D>(1, BA, MN, ng, chunk, nz, st);
        mark();
        fam.push_back(1);
        A->launches++;
      }
      if (fused_sing) {
        if (prod) launch_sing_m<STB_K, true>(BA, MS, blk.a1 - blk.a0, st);
        else if (kind == STB_V) launch_sing_m<STB_V>(BA, MS, blk.a1 - blk.a0, st);
        else if (kind == STB_K) launch_sing_m<STB_K>(BA, MS, blk.a1 - blk.a0, st);
        else launch_sing_m<STB_D>(BA, MS, blk.a1 - blk.a0, st);
      } else {
        const int ncell = 2 * (blk.a1 - blk.a0);
        const int per_row = kind == STB_V ? 3 : (kind == STB_K ? 4 : 5);
        const long long nwarps = (long long)ncell * ng * per_row;
        const unsigned nblk = (unsigned)((nwarps + 3) / 4);
        if (kind == STB_V) k_sing<STB_V><<<nblk, 128, 0, st>>>(BA, m->d_seg, m->d_half, m->d_dual, m->d_t, m->alpha, q_sing, nwarps);
        else if (kind == STB_K) k_sing<STB_K><<<nblk, 128, 0, st>>>(BA, m->d_seg, m->d_half, m->d_dual, m->d_t, m->alpha, q_sing, nwarps);
        else k_sing<STB_D><<<nblk, 128, 0, st>>>(BA, m->d_seg, m->d_half, m->d_dual, m->d_t, m->alpha, q_sing, nwarps);
        count_launch();
      }
      mark();
      fam.push_back(2);
      A->launches++;
    }
  }
  if (prod) {
    // y = sum of the partials of the owned blocks of each test step (fixed order)
    std::vector<int> rstart(m->nt + 1, 0);
    std::vector<long long> roff;
    for (int a = 0; a < m->nt; ++a) {
      rstart[a] = (int)roff.size();
      for (size_t bi = 0; bi < blocks_of(A).size(); ++bi)
        if (blocks_of(A)[bi].a0 <= a && a < blocks_of(A)[bi].a1)
          roff.push_back(pbase[bi] - (long long)blocks_of(A)[bi].a0 * ng * pslots);
    }
    rstart[m->nt] = (int)roff.size();
    int* d_rs = nullptr;
    long long* d_ro = nullptr;
    if ((e = cudaMallocAsync((void**)&d_rs, sizeof(int) * rstart.size(), st)) != cudaSuccess ||
        (e = cudaMallocAsync((void**)&d_ro, sizeof(long long) * std::max<size_t>(1, roff.size()), st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(d_rs, rstart.data(), sizeof(int) * rstart.size(), cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (roff.size() && (e = cudaMemcpyAsync(d_ro, roff.data(), sizeof(long long) * roff.size(), cudaMemcpyHostToDevice, st)) != cudaSuccess))
      return cuda_fail(e, "assemble/product reduce");
    const long long n = (long long)ng * m->nt;
    k_prod_reduce<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d_part, d_rs, d_ro, ng, m->nt, pslots, prod_y);
    count_launch();
    cudaFreeAsync(d_rs, st);
    cudaFreeAsync(d_ro, st);
    storage_release(m->device, d_part, part_bytes, st);
  }
  storage_release(m->device, d_rec, rec_bytes, st);
  if (d_list) cudaFreeAsync(d_list, st);
  cudaFreeAsync(d_poff, st);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "assemble/launch");
  return BEM_OK;
}

bem_status finalize_assembly_stats(bem_matrix* A) {
  if (A->stats_ready) return BEM_OK;
  A->stats_ready = true;
  if (!A->ev.empty()) cudaEventSynchronize(A->ev.back());
  unsigned long long ctr[CTR_N] = {0};
  cudaError_t e = cudaMemcpy(ctr, A->d_ctr, sizeof(ctr), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "assembly stats");
  for (int k = 0; k < 4; ++k) {
    A->nodes_bulk[k] = (long long)ctr[k];
    A->nodes_near[k] = (long long)ctr[5 + k];
  }
  A->ms_bulk = A->ms_near = A->ms_sing = A->ms_records = 0.0;
  for (size_t k = 0; k + 1 < A->ev.size(); ++k) {
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, A->ev[k], A->ev[k + 1]);
    const int f = A->ev_fam[k];
    (f == 0 ? A->ms_bulk : f == 1 ? A->ms_near : f == 2 ? A->ms_sing : A->ms_records) += ms;
  }
  for (auto x : A->ev) cudaEventDestroy(x);
  A->ev.clear();
  // algorithmic FP64 flops of the bulk kernel, static counts of the shipped
  // forms (DFMA = 2): regime A per node = the Horner chain in u plus the closing s / ln s terms
  // (RegA::chain + RegA::finish): V 19 + 3, K 20 + 1, D 20 + 3 FMAs (D's two families are one
  // merged chain) = 44 / 42 / 46 flops; regime B per node 61 (E1 / GB3 and the closing terms, exp
  // not counted) + per Taylor order one FMA per Horner chain: V (S1, S2), K (S1, S3) 4,
  // D (S1, S2 of H, S1 of F) 6
  const int kind = A->kind;
  const double fA = kind == STB_V ? 44.0 : (kind == STB_K ? 42.0 : 46.0);
  const double fK = kind == STB_D ? 6.0 : 4.0;
  // K_h g with the trial-moment table: its nodes are not evaluated pair by pair (ctr[CTR_TAB]); the
  // table kernel's own flops (prefix scans, one chain per covered node and test segment) instead
  A->nodes_tab = (long long)ctr[CTR_TAB];
  A->flops_bulk = fA * (double)(A->nodes_bulk[0] - A->nodes_tab) + 61.0 * (double)A->nodes_bulk[1] +
                  fK * (double)ctr[4] + A->flops_tab;
  A->ev_bulk = A->nodes_bulk[0] + A->nodes_bulk[1] + A->nodes_bulk[2] + A->nodes_bulk[3];
  A->ev_near = A->nodes_near[0] + A->nodes_near[1] + A->nodes_near[2] + A->nodes_near[3];
  // self-checks of the kernels' coverage
  if (A->ev_bulk != A->nodes_expected) {
    set_error("assembly stats: bulk node count mismatch");
    return BEM_E_CUDA;
  }
  if (ctr[13] != 0) {
    set_error("assembly stats: touching-pair moment record outside regime A");
    return BEM_E_CUDA;
  }
  return BEM_OK;
}

// representation formula (row f2): u = Vt w - W g at npts interior points (device arrays)
bem_status eval_potential(const bem_mesh* m, const double* w, const double* g, long long npts,
                          const double* pts, double* out, cudaStream_t st) {
  if (npts <= 0) return BEM_OK;
  mesh_wait(m, st);
  int* d_bad = nullptr;
  cudaError_t e;
  if ((e = cudaMallocAsync((void**)&d_bad, sizeof(int), st)) != cudaSuccess ||
      (e = cudaMemsetAsync(d_bad, 0, sizeof(int), st)) != cudaSuccess)
    return cuda_fail(e, "eval_potential");
  const unsigned nblk = (unsigned)((npts * 32 + 127) / 128);
  k_potential<<<nblk, 128, 0, st>>>(m->d_seg, m->d_t, m->ng, m->nt, m->alpha, m->hmax, w, g, npts, pts, out, d_bad);
  count_launch();
  int bad = 0;
  cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d_bad, st);
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "eval_potential");
  if (bad) {
    set_error("bem_eval_potential: a point is closer than h_max to Gamma (the interior quadrature needs distance >= h_max)");
    return BEM_E_INVALID;
  }
  return BEM_OK;
}

// row f2 with u0 != 0: u += (M~_0 u0)(x, t) at interior points; nodes / tris on the host
bem_status eval_potential_initial(const bem_mesh* m, int nnode, const double* nodes, int ntri, const int* tris,
                                  const double* u0, long long npts, const double* pts, double* out,
                                  cudaStream_t st) {
  if (npts <= 0) return BEM_OK;
  mesh_wait(m, st);
  double* d_nodes = nullptr;
  int* d_tris = nullptr;
  int* d_bad = nullptr;
  cudaError_t e;
  if ((e = cudaMallocAsync((void**)&d_nodes, sizeof(double) * 2 * nnode, st)) != cudaSuccess ||
      (e = cudaMallocAsync((void**)&d_tris, sizeof(int) * 3 * ntri, st)) != cudaSuccess ||
      (e = cudaMallocAsync((void**)&d_bad, sizeof(int), st)) != cudaSuccess ||
      (e = cudaMemsetAsync(d_bad, 0, sizeof(int), st)) != cudaSuccess ||
      (e = cudaMemcpyAsync(d_nodes, nodes, sizeof(double) * 2 * nnode, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
      (e = cudaMemcpyAsync(d_tris, tris, sizeof(int) * 3 * ntri, cudaMemcpyHostToDevice, st)) != cudaSuccess)
    return cuda_fail(e, "eval_potential_initial");
  const unsigned nblk = (unsigned)((npts * 32 + 127) / 128);
  k_potential_initial<<<nblk, 128, 0, st>>>(d_nodes, d_tris, ntri, u0, m->alpha, npts, pts, out, d_bad);
  count_launch();
  int bad = 0;
  cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d_nodes, st);
  cudaFreeAsync(d_tris, st);
  cudaFreeAsync(d_bad, st);
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "eval_potential_initial");
  if (bad) {
    set_error("bem_eval_potential_initial: a point has t <= 0");
    return BEM_E_INVALID;
  }
  return BEM_OK;
}

// row f1: b <- b - M_h^0 u0 (eq. 4); nodes / tris on the host, u0 and b on the device
bem_status initial_rhs(const bem_mesh* m, int nnode, const double* nodes, int ntri, const int* tris,
                       const double* u0, int qx, int qtf, int qtn, double* b, cudaStream_t st) {
  mesh_wait(m, st);
  double* d_nodes = nullptr;
  int* d_tris = nullptr;
  double* d_part = nullptr;
  // chunks per element: enough CTAs for 8 per SM, each looping over its interleaved triangle batches
  const int nbt_all = (ntri + 255) / 256;
  const int nch = std::max(1, std::min(nbt_all, (8 * 148 + m->ng - 1) / m->ng));
  const int nbatch = (nbt_all + nch - 1) / nch;
  static const int use_moments = getenv("BEM_INITIAL_DIRECT") ? 0 : 1;
  const size_t part_bytes = sizeof(double) * (size_t)m->ng * nch * 8 * (m->nt + 2);   // one row per warp
  cudaError_t e;
  if ((e = cudaMallocAsync((void**)&d_nodes, sizeof(double) * 2 * nnode, st)) != cudaSuccess ||
      (e = cudaMallocAsync((void**)&d_tris, sizeof(int) * 3 * ntri, st)) != cudaSuccess ||
      (e = storage_acquire(m->device, part_bytes, st, (void**)&d_part)) != cudaSuccess ||
      (e = cudaMemcpyAsync(d_nodes, nodes, sizeof(double) * 2 * nnode, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
      (e = cudaMemcpyAsync(d_tris, tris, sizeof(int) * 3 * ntri, cudaMemcpyHostToDevice, st)) != cudaSuccess)
    return cuda_fail(e, "initial_rhs");
  dim3 grid(m->ng, nch);
  // the warps' node accumulators in shared memory when 8 (nt + 2) doubles fit, else in their rows
  const size_t wacc_bytes = sizeof(double) * 8 * (size_t)(m->nt + 2);
  const int use_wacc = wacc_bytes <= 160 * 1024;
  if (use_wacc) cudaFuncSetAttribute(k_initial, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wacc_bytes);
  k_initial<<<grid, 256, use_wacc ? wacc_bytes : 0, st>>>(m->d_seg, m->d_t, m->ng, m->nt, m->alpha, d_nodes, d_tris, ntri,
                                                          u0, qx, qtf, qtn, use_moments, nbatch, use_wacc, d_part);
  const long long n = (long long)m->ng * m->nt;
  k_initial_finish<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d_part, m->ng, m->nt, nch, m->alpha, b);
  count_launch(2);
  cudaFreeAsync(d_nodes, st);
  cudaFreeAsync(d_tris, st);
  storage_release(m->device, d_part, part_bytes, st);
  e = cudaGetLastError();
  return e == cudaSuccess ? BEM_OK : cuda_fail(e, "initial_rhs");
}

}  // namespace stb
