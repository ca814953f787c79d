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
  int qfar;               // near-cell Gauss order for well-separated pairs
};

__device__ __forceinline__ double* entry_ptr(const BlockArgs& B, int a, int i, int b, int j) {
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
// qfar: order for well-separated pairs (rho >= 9), min(6, q_bulk + 1) from the mesh's kappa
__host__ __device__ inline int near_order(const Seg& X, const Seg& Y, int qfar) {
  double rho = seg_dist(X, Y) / fmax(X.h, Y.h);
  return rho < 2.5 ? 10 : (rho < 5.0 ? 8 : (rho < 9.0 ? 6 : qfar));
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

// large-x forms, out of line: rare, and keeping them out of the unrolled point loops keeps the
// kernels inside the instruction cache
__device__ __noinline__ double large_h(double x, double lreg) {
  const double tt = 1.0 / x, e = exp(-x);
  return fma(1.0 + x, e1_large(tt, e) + lreg, -e);
}
__device__ __noinline__ double large_psi(double x) {
  const double tt = 1.0 / x, e = exp(-x);
  return e * tt - tt - e1_large(tt, e);
}
__device__ __noinline__ double2 large_h_e1(double x, double lreg) {
  const double tt = 1.0 / x, e = exp(-x);
  const double e1 = e1_large(tt, e) + lreg;
  return make_double2(fma(1.0 + x, e1, -e), e1);
}

// ================================================================= bulk V
// thread = segment pair (i, j): warp = row i, lane = column j; band of R test steps.
// Every point pair is first evaluated with the small-x form (branch-free, unrolled: the Q*Q
// Horner chains interleave); the rare points with x >= 4 are then overwritten by the large-x
// form (exp + polynomial in 1/x).
template <int Q, int R>
__global__ void __launch_bounds__(128) k_bulk_V(BlockArgs B, const Seg* __restrict__ seg,
                                                const double* __restrict__ t, double alpha,
                                                int nband) {
  constexpr int QQ = Q * Q;
  const int ng = B.ng;
  const int j = blockIdx.x * 32 + (threadIdx.x & 31);
  const int i = blockIdx.y * 4 + (threadIdx.x >> 5);
  if (i >= ng || j >= ng) return;
  const int band = blockIdx.z;
  const int r_hi = B.a1 - R * band;
  const int r_lo = max(B.a0, r_hi - R);
  if (r_hi <= r_lo) return;
  const int bmax = min(B.b1 - 1, r_hi - 1 - 2);
  if (bmax < B.b0) return;
  const Seg X = seg[i], Y = seg[j];
  const bool reg = (i == j);
  double c[QQ], L[QQ];
#pragma unroll
  for (int u = 0; u < Q; ++u) {
    double px = fma(c_gx[Q][u], X.bx - X.ax, X.ax), py = fma(c_gx[Q][u], X.by - X.ay, X.ay);
#pragma unroll
    for (int v = 0; v < Q; ++v) {
      double qx = fma(c_gx[Q][v], Y.bx - Y.ax, Y.ax), qy = fma(c_gx[Q][v], Y.by - Y.ay, Y.ay);
      double dx = px - qx, dy = py - qy;
      double cc = 0.25 * alpha * (dx * dx + dy * dy);
      c[u * Q + v] = cc;
      L[u * Q + v] = cc > 0.0 ? log(cc) : 0.0;
    }
  }
  const double scale = X.h * Y.h / (4.0 * STB_PI);
  double Gp[R];  // G_a(y-1) = Phi(a+1, y-1) - Phi(a, y-1) for the band rows
#pragma unroll
  for (int r = 0; r < R; ++r) Gp[r] = 0.0;
  for (int y = B.b0; y <= bmax + 1; ++y) {
    double phi_prev = 0.0;
#pragma unroll 1
    for (int r = 0; r <= R; ++r) {
      const int x = r_lo + r;
      double phi = 0.0;
      if (x <= r_hi && x > y) {
        const double4 nd = B.lag[x * B.ldlag + y];
        const double s = nd.x, lns = nd.y, is = nd.z;
        const double g0 = STB_GAMMA - lns;
        double hv[QQ];
        bool large = false;
#pragma unroll
        for (int p = 0; p < QQ; ++p) {
          const double xx = c[p] * is;
          hv[p] = fma(-(1.0 + xx), reg ? g0 : g0 + L[p], gh_poly(xx));
          large |= xx >= STB_XSPLIT;
        }
        if (large) {
#pragma unroll
          for (int p = 0; p < QQ; ++p) {
            const double xx = c[p] * is;
            if (xx >= STB_XSPLIT) hv[p] = large_h(xx, reg ? L[p] : 0.0);
          }
        }
        double acc = 0.0;
#pragma unroll
        for (int u = 0; u < Q; ++u) {
          double part = 0.0;
#pragma unroll
          for (int v = 0; v < Q; ++v) part = fma(c_gw[Q][v], hv[u * Q + v], part);
          acc = fma(c_gw[Q][u], part, acc);
        }
        phi = s * acc;
      }
      if (r > 0) {
        const int a = x - 1, b = y - 1;
        const double G = phi - phi_prev;
        if (y > B.b0 && a < r_hi && a - b >= 2) *entry_ptr(B, a, i, b, j) = scale * (Gp[r - 1] - G);
        Gp[r - 1] = G;
      }
      phi_prev = phi;
    }
  }
}

// ================================================================= bulk K
// lane l of a warp owns segment j = jt*31 + l - 1 (mod ng) and computes the two moments
// M_k = int int lambda_k(y) dot sum eps Q (lambda_0 = 1 - f falls, lambda_1 = f rises on gamma_j);
// K(i, n) = M_1(i, n-1) + M_0(i, n) (primal hat phi_n) via one shuffle.
template <int Q, int R>
__global__ void __launch_bounds__(128) k_bulk_K(BlockArgs B, const Seg* __restrict__ seg,
                                                const double* __restrict__ t, double alpha,
                                                int nband) {
  constexpr int QQ = Q * Q;
  const int ng = B.ng;
  const int lane = threadIdx.x & 31;
  const int n = blockIdx.x * 31 + lane - 1;       // output column (valid for lane >= 1)
  const int j = (n + ng) % ng;
  const int i = blockIdx.y * 4 + (threadIdx.x >> 5);
  if (i >= ng) return;                            // whole warp
  const bool out_ok = lane >= 1 && n < ng;
  const int band = blockIdx.z;
  const int r_hi = B.a1 - R * band;
  const int r_lo = max(B.a0, r_hi - R);
  if (r_hi <= r_lo) return;
  const int bmax = min(B.b1 - 1, r_hi - 1 - 2);
  if (bmax < B.b0) return;
  const Seg X = seg[i], Y = seg[j];
  const bool zero = collinear(X, Y) || (n >= ng && lane >= 1);
  double c[QQ], L[QQ], dw[QQ];
#pragma unroll
  for (int u = 0; u < Q; ++u) {
    double px = fma(c_gx[Q][u], X.bx - X.ax, X.ax), py = fma(c_gx[Q][u], X.by - X.ay, X.ay);
#pragma unroll
    for (int v = 0; v < Q; ++v) {
      double qx = fma(c_gx[Q][v], Y.bx - Y.ax, Y.ax), qy = fma(c_gx[Q][v], Y.by - Y.ay, Y.ay);
      double dx = px - qx, dy = py - qy;
      double cc = 0.25 * alpha * (dx * dx + dy * dy);
      cc = zero ? 1.0 : cc;
      c[u * Q + v] = cc;
      L[u * Q + v] = log(cc);
      dw[u * Q + v] = zero ? 0.0 : c_gw[Q][u] * c_gw[Q][v] * (dx * Y.nx + dy * Y.ny);
    }
  }
  const double scale = alpha / (8.0 * STB_PI) * X.h * Y.h;
  double Gp0[R], Gp1[R];
#pragma unroll
  for (int r = 0; r < R; ++r) Gp0[r] = Gp1[r] = 0.0;
  for (int y = B.b0; y <= bmax + 1; ++y) {
    double p0_prev = 0.0, p1_prev = 0.0;
#pragma unroll 1
    for (int r = 0; r <= R; ++r) {
      const int x = r_lo + r;
      double P0 = 0.0, P1 = 0.0;
      if (x <= r_hi && x > y && !zero) {
        const double4 nd = B.lag[x * B.ldlag + y];
        const double s = nd.x, lns = nd.y, is = nd.z;
        const double g0 = STB_GAMMA - lns;
        double ps[QQ];
        bool large = false;
#pragma unroll
        for (int p = 0; p < QQ; ++p) {
          const double xx = c[p] * is;
          ps[p] = psi_poly(xx) + (g0 + L[p]);
          large |= xx >= STB_XSPLIT;
        }
        if (large) {
#pragma unroll
          for (int p = 0; p < QQ; ++p) {
            const double xx = c[p] * is;
            if (xx >= STB_XSPLIT) ps[p] = large_psi(xx);
          }
        }
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int p = 0; p < QQ; ++p) {
          const double v = dw[p] * ps[p];
          a1 = fma(c_gx[Q][p % Q], v, a1);
          a0 += v;
        }
        P0 = a0 - a1;   // lambda_0 = 1 - f
        P1 = a1;
      }
      if (r > 0) {
        const int a = x - 1, b = y - 1;
        const double G0 = P0 - p0_prev, G1 = P1 - p1_prev;
        if (y > B.b0 && a < r_hi && a - b >= 2) {
          const double m0 = Gp0[r - 1] - G0, m1 = Gp1[r - 1] - G1;
          const double left = __shfl_up_sync(0xffffffffu, m1, 1);
          if (out_ok) *entry_ptr(B, a, i, b, n) = scale * (left + m0);
        }
        Gp0[r - 1] = G0;
        Gp1[r - 1] = G1;
      }
      p0_prev = P0;
      p1_prev = P1;
    }
  }
}

// ================================================================= D tiles
// CTA: warp w <-> half row p = 2 L0 - 1 + w (w < 2 TL + 2), lane <-> half column
// q = 2 K0 - 1 + lane; entries (l, k), l in [L0, L0+TL), k in [K0, K0+15).
// Combine (deterministic, no atomics): stage 1 contracts the 4 half columns of each dual hat k
// inside the warp with three shuffles per quantity; stage 2 contracts the 4 half rows of each
// dual hat l through shared memory.
constexpr int DTK = 15;
constexpr int DTL_BULK = 3;   // dual rows per CTA (8 warps)
constexpr int DTL_NEAR = 3;

struct DMom {
  double v, f00, f01, f10, f11;
};

struct DLane {
  double cv[2], c0[2], c1[2];  // role lo (n = lane&1) and hi (n + 2) coefficients of dual k
  double nn;                   // n_p . n_q
  __device__ void init(const Dual* __restrict__ dual, const Seg& X, const Seg& Y, int K0, int ng, int lane) {
    nn = X.nx * Y.nx + X.ny * Y.ny;
#pragma unroll
    for (int role = 0; role < 2; ++role) {
      const int n = (lane & 1) + 2 * role;
      const int jj = (lane - n) >> 1;
      const int k = K0 + jj;
      cv[role] = c0[role] = c1[role] = 0.0;
      if (lane - n >= 0 && jj < DTK && k < ng) {
        const Dual d = dual[k];
        cv[role] = n < 2 ? 1.0 / d.Lm : -1.0 / d.Lp;
        const double v0[4] = {0.0, d.vm, 1.0, d.vp}, v1[4] = {d.vm, 1.0, d.vp, 0.0};
        c0[role] = nn * v0[n];
        c1[role] = nn * v1[n];
      }
    }
  }
  // stage 1: T at even lanes 2j = sum over the 4 half columns of dual K0 + j; stored to smem
  __device__ void stage1(const DMom& M, double* __restrict__ T, int lane) const {
    double A[3], Bq[3];
#pragma unroll
    for (int role = 0; role < 2; ++role) {
      double* o = role ? Bq : A;
      o[0] = cv[role] * M.v;
      o[1] = c0[role] * M.f00 + c1[role] * M.f01;
      o[2] = c0[role] * M.f10 + c1[role] * M.f11;
    }
#pragma unroll
    for (int qn = 0; qn < 3; ++qn) {
      const double s = A[qn] + __shfl_down_sync(0xffffffffu, A[qn], 1) +
                       __shfl_down_sync(0xffffffffu, Bq[qn], 2) + __shfl_down_sync(0xffffffffu, Bq[qn], 3);
      if (!(lane & 1) && (lane >> 1) < DTK) T[(lane >> 1) * 3 + qn] = s;
    }
  }
};

// stage 2: entry (l, k) = sum_m [dv_l[m] T_v + v_l[m][0] T_f0 + v_l[m][1] T_f1](half row of m)
template <int TL>
__device__ __forceinline__ double d_stage2(const Dual& dl, const double* __restrict__ T, int lr, int kc) {
  const double dv[4] = {1.0 / dl.Lm, 1.0 / dl.Lm, -1.0 / dl.Lp, -1.0 / dl.Lp};
  const double v0[4] = {0.0, dl.vm, 1.0, dl.vp}, v1[4] = {dl.vm, 1.0, dl.vp, 0.0};
  double acc = 0.0;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const double* Tm = T + ((2 * lr + m) * DTK + kc) * 3;
    acc += dv[m] * Tm[0] + v0[m] * Tm[1] + v1[m] * Tm[2];
  }
  return acc;
}

template <int Q, int R, int TL>
__global__ void __launch_bounds__(32 * (2 * TL + 2), (TL <= 3 && Q <= 3 ? 2 : 1)) k_bulk_D(BlockArgs B, const Seg* __restrict__ half,
                                                            const Dual* __restrict__ dual,
                                                            const double* __restrict__ t, double alpha,
                                                            int nband) {
  constexpr int QQ = Q * Q;
  constexpr int NW = 2 * TL + 2;
  __shared__ double sT[R][NW * DTK * 3];
  const int ng = B.ng, nh = 2 * ng;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int K0 = blockIdx.x * DTK, L0 = blockIdx.y * TL;
  const int p = ((2 * L0 - 1 + w) % nh + nh) % nh;
  const int q = ((2 * K0 - 1 + lane) % nh + nh) % nh;
  const int band = blockIdx.z;
  const int r_hi = B.a1 - R * band;
  const int r_lo = max(B.a0, r_hi - R);
  if (r_hi <= r_lo) return;
  const int bmax = min(B.b1 - 1, r_hi - 1 - 2);
  if (bmax < B.b0) return;
  const Seg X = half[p], Y = half[q];
  const bool reg = (p == q);
  DLane DL;
  DL.init(dual, X, Y, K0, ng, lane);
  const bool do_f = DL.nn != 0.0;
  const bool any_f = __any_sync(0xffffffffu, do_f);
  double c[QQ], L[QQ];
#pragma unroll
  for (int u = 0; u < Q; ++u) {
    double px = fma(c_gx[Q][u], X.bx - X.ax, X.ax), py = fma(c_gx[Q][u], X.by - X.ay, X.ay);
#pragma unroll
    for (int v = 0; v < Q; ++v) {
      double qx = fma(c_gx[Q][v], Y.bx - Y.ax, Y.ax), qy = fma(c_gx[Q][v], Y.by - Y.ay, Y.ay);
      double dx = px - qx, dy = py - qy;
      double cc = 0.25 * alpha * (dx * dx + dy * dy);
      c[u * Q + v] = cc;
      L[u * Q + v] = cc > 0.0 ? log(cc) : 0.0;
    }
  }
  const double sv = X.h * Y.h / (4.0 * STB_PI), sf = alpha * X.h * Y.h / (4.0 * STB_PI);
  DMom Gp[R];
#pragma unroll
  for (int r = 0; r < R; ++r) Gp[r] = DMom{0, 0, 0, 0, 0};
  for (int y = B.b0; y <= bmax + 1; ++y) {
    DMom prev{0, 0, 0, 0, 0};
#pragma unroll 1
    for (int r = 0; r <= R; ++r) {
      const int x = r_lo + r;
      DMom phi{0, 0, 0, 0, 0};
      if (x <= r_hi && x > y) {
        const double4 nd = B.lag[x * B.ldlag + y];
        const double s = nd.x, lns = nd.y, is = nd.z;
        const double g0 = STB_GAMMA - lns;
        double hv[QQ], ev[QQ];
        bool large = false;
        if (any_f) {  // warp-uniform: some lane of the warp needs the normal term (n_p . n_q != 0)
#pragma unroll
          for (int pp = 0; pp < QQ; ++pp) {
            const double xx = c[pp] * is;
            const double gl = reg ? g0 : g0 + L[pp];
            ev[pp] = ein_poly(xx) - gl;
            hv[pp] = fma(-(1.0 + xx), gl, gh_poly(xx));
            large |= xx >= STB_XSPLIT;
          }
        } else {      // perpendicular half segments: only the curl kernel
#pragma unroll
          for (int pp = 0; pp < QQ; ++pp) {
            const double xx = c[pp] * is;
            ev[pp] = 0.0;
            hv[pp] = fma(-(1.0 + xx), reg ? g0 : g0 + L[pp], gh_poly(xx));
            large |= xx >= STB_XSPLIT;
          }
        }
        if (large) {
#pragma unroll
          for (int pp = 0; pp < QQ; ++pp) {
            const double xx = c[pp] * is;
            if (xx >= STB_XSPLIT) {
              const double2 he = large_h_e1(xx, reg ? L[pp] : 0.0);
              hv[pp] = he.x;
              ev[pp] = he.y;
            }
          }
        }
        double av = 0.0, a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0;
#pragma unroll
        for (int u = 0; u < Q; ++u) {
          double tv = 0.0, tf0 = 0.0, tf1 = 0.0;
#pragma unroll
          for (int v = 0; v < Q; ++v) {
            const double wv = c_gw[Q][v], fv = c_gx[Q][v];
            tv = fma(wv, hv[u * Q + v], tv);
            const double we = wv * ev[u * Q + v];
            tf1 = fma(fv, we, tf1);
            tf0 += we;
          }
          tf0 -= tf1;  // lambda_0 = 1 - f
          const double wu = c_gw[Q][u], fu = c_gx[Q][u];
          av = fma(wu, tv, av);
          const double w1 = wu * fu, w0 = wu - w1;
          a00 = fma(w0, tf0, a00);
          a01 = fma(w0, tf1, a01);
          a10 = fma(w1, tf0, a10);
          a11 = fma(w1, tf1, a11);
        }
        phi.v = sv * s * av;
        if (do_f) {
          phi.f00 = sf * a00;
          phi.f01 = sf * a01;
          phi.f10 = sf * a10;
          phi.f11 = sf * a11;
        }
      }
      if (r > 0) {
        const DMom G{phi.v - prev.v, phi.f00 - prev.f00, phi.f01 - prev.f01, phi.f10 - prev.f10, phi.f11 - prev.f11};
        const DMom& g = Gp[r - 1];
        const DMom M{g.v - G.v, g.f00 - G.f00, g.f01 - G.f01, g.f10 - G.f10, g.f11 - G.f11};
        if (y > B.b0) DL.stage1(M, sT[r - 1] + w * DTK * 3, lane);
        Gp[r - 1] = G;
      }
      prev = phi;
    }
    if (y > B.b0) {
      const int b = y - 1;
      __syncthreads();
      for (int e = threadIdx.x; e < R * TL * DTK; e += blockDim.x) {
        const int r = e / (TL * DTK), lr = (e / DTK) % TL, kc = e % DTK;
        const int a = r_lo + r, l = L0 + lr, k = K0 + kc;
        if (a < r_hi && a - b >= 2 && l < ng && k < ng)
          *entry_ptr(B, a, l, b, k) = d_stage2<TL>(dual[l], sT[r], lr, kc);
      }
      __syncthreads();
    }
  }
}

// ================================================================= near cells (d <= 1)
// regular (non-touching) pair integral with the direct four-lag kernel sum
// ker 0: H (V, D-curl), 1: F (D normal), 2: Q (K, dot and S/c included)
template <int KER>
__device__ double pair_regular(const Seg& X, const Seg& Y, const Lags& Lg, double alpha, int q,
                               double sx0, double sx1, double sy0, double sy1) {
  double acc = 0.0;
  for (int u = 0; u < q; ++u) {
    const double fu = c_gx[q][u];
    const double px = fma(fu, X.bx - X.ax, X.ax), py = fma(fu, X.by - X.ay, X.ay);
    double part = 0.0;
    for (int v = 0; v < q; ++v) {
      const double fv = c_gx[q][v];
      const double qx = fma(fv, Y.bx - Y.ax, Y.ax), qy = fma(fv, Y.by - Y.ay, Y.ay);
      const double dx = px - qx, dy = py - qy;
      const double c = 0.25 * alpha * (dx * dx + dy * dy);
      double k = 0.0;
      if (KER == 0) {
        for (int m = 0; m < Lg.n; ++m) k = fma(Lg.e[m] * Lg.s[m], dev_hfun(c / Lg.s[m]), k);
      } else if (KER == 1) {
        for (int m = 0; m < Lg.n; ++m) k = fma(Lg.e[m], dev_e1(c / Lg.s[m]), k);
      } else {
        for (int m = 0; m < Lg.n; ++m) k = fma(Lg.e[m], dev_psi(c / Lg.s[m]), k);
        k = (k + Lg.S / c) * (dx * Y.nx + dy * Y.ny);
      }
      part = fma(c_gw[q][v] * fma(fv, sy1 - sy0, sy0), k, part);
    }
    acc = fma(c_gw[q][u] * fma(fu, sx1 - sx0, sx0), part, acc);
  }
  const double pre = KER == 0 ? 1.0 / (4.0 * STB_PI) : (KER == 1 ? alpha / (4.0 * STB_PI) : alpha / (8.0 * STB_PI));
  return pre * X.h * Y.h * acc;
}

// V and K near cells: thread per entry; touching pairs are left to k_sing
template <int KIND>
__global__ void __launch_bounds__(128) k_near_VK(BlockArgs B, const Seg* __restrict__ seg,
                                                 const double* __restrict__ t, double alpha) {
  const int ng = B.ng;
  const int j = blockIdx.x * 32 + (threadIdx.x & 31);
  const int i = blockIdx.y * 4 + (threadIdx.x >> 5);
  const int cell = blockIdx.z;  // test step a = a0 + cell/2, d = cell % 2
  const int a = B.a0 + cell / 2, b = a - (cell % 2);
  if (i >= ng || j >= ng || a >= B.a1 || b < B.b0 || b >= B.b1) return;
  const Lags Lg = make_lags(t, a, b);
  const Seg X = seg[i];
  double val = 0.0;
  if (KIND == STB_V) {
    const Seg Y = seg[j];
    if (chain_rel(i, j, ng) == 0) val = pair_regular<0>(X, Y, Lg, alpha, near_order(X, Y, B.qfar), 1, 1, 1, 1);
  } else {
    const int jl = (j - 1 + ng) % ng;
    const Seg Yl = seg[jl], Yr = seg[j];
    if (chain_rel(i, jl, ng) == 0 && !collinear(X, Yl))
      val += pair_regular<2>(X, Yl, Lg, alpha, near_order(X, Yl, B.qfar), 1, 1, 0, 1);
    if (chain_rel(i, j, ng) == 0 && !collinear(X, Yr))
      val += pair_regular<2>(X, Yr, Lg, alpha, near_order(X, Yr, B.qfar), 1, 1, 1, 0);
  }
  *entry_ptr(B, a, i, b, j) = val;
}

// D near cells: half-pair threads in the D tile, the 5 moments in one pass over the points
__device__ __forceinline__ void dev_h_e1(double x, double& h, double& e1) {
  if (x < STB_XSPLIT) {
    const double gl = STB_GAMMA + log(x);
    e1 = ein_poly(x) - gl;
    h = fma(-(1.0 + x), gl, gh_poly(x));
  } else if (x > STB_XUNDER) {
    e1 = 0.0;
    h = 0.0;
  } else {
    const double tt = 1.0 / x, e = exp(-x);
    e1 = e1_large(tt, e);
    h = fma(1.0 + x, e1, -e);
  }
}

__device__ DMom near_moments(const Seg& X, const Seg& Y, const Lags& Lg, double alpha, int q, bool do_f) {
  double mv = 0.0, m00 = 0.0, m01 = 0.0, m10 = 0.0, m11 = 0.0;
  for (int u = 0; u < q; ++u) {
    const double fu = c_gx[q][u];
    const double px = fma(fu, X.bx - X.ax, X.ax), py = fma(fu, X.by - X.ay, X.ay);
    double tv = 0.0, tf0 = 0.0, tf1 = 0.0;
    for (int v = 0; v < q; ++v) {
      const double fv = c_gx[q][v];
      const double qx = fma(fv, Y.bx - Y.ax, Y.ax), qy = fma(fv, Y.by - Y.ay, Y.ay);
      const double dx = px - qx, dy = py - qy;
      const double c = 0.25 * alpha * (dx * dx + dy * dy);
      double kv = 0.0, kf = 0.0;
      for (int m = 0; m < Lg.n; ++m) {
        double h, e1;
        dev_h_e1(c / Lg.s[m], h, e1);
        kv = fma(Lg.e[m] * Lg.s[m], h, kv);
        kf = fma(Lg.e[m], e1, kf);
      }
      const double wv = c_gw[q][v];
      tv = fma(wv, kv, tv);
      const double we = wv * kf;
      tf1 = fma(fv, we, tf1);
      tf0 += we;
    }
    tf0 -= tf1;
    const double wu = c_gw[q][u];
    mv = fma(wu, tv, mv);
    const double w1 = wu * fu, w0 = wu - w1;
    m00 = fma(w0, tf0, m00);
    m01 = fma(w0, tf1, m01);
    m10 = fma(w1, tf0, m10);
    m11 = fma(w1, tf1, m11);
  }
  const double sv = X.h * Y.h / (4.0 * STB_PI), sf = do_f ? alpha * X.h * Y.h / (4.0 * STB_PI) : 0.0;
  return DMom{sv * mv, sf * m00, sf * m01, sf * m10, sf * m11};
}

template <int TL>
__global__ void __launch_bounds__(32 * (2 * TL + 2)) k_near_D(BlockArgs B, const Seg* __restrict__ half,
                                                            const Dual* __restrict__ dual,
                                                            const double* __restrict__ t, double alpha) {
  constexpr int NW = 2 * TL + 2;
  __shared__ double sT[NW * DTK * 3];
  const int ng = B.ng, nh = 2 * ng;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int K0 = blockIdx.x * DTK, L0 = blockIdx.y * TL;
  const int cell = blockIdx.z;
  const int a = B.a0 + cell / 2, b = a - (cell % 2);
  if (a >= B.a1 || b < B.b0 || b >= B.b1) return;
  const int p = ((2 * L0 - 1 + w) % nh + nh) % nh;
  const int q = ((2 * K0 - 1 + lane) % nh + nh) % nh;
  const Seg X = half[p], Y = half[q];
  const Lags Lg = make_lags(t, a, b);
  DLane DL;
  DL.init(dual, X, Y, K0, ng, lane);
  DMom M{0, 0, 0, 0, 0};
  if (chain_rel(p, q, nh) == 0) M = near_moments(X, Y, Lg, alpha, near_order(X, Y, B.qfar), DL.nn != 0.0);
  DL.stage1(M, sT + w * DTK * 3, lane);
  __syncthreads();
  for (int e = threadIdx.x; e < TL * DTK; e += blockDim.x) {
    const int lr = e / DTK, kc = e % DTK, l = L0 + lr, k = K0 + kc;
    if (l < ng && k < ng) *entry_ptr(B, a, l, b, k) = d_stage2<TL>(dual[l], sT, lr, kc);
  }
}

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
                                int n, double sx0, double sx1, double sy0, double sy1) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  if (rel == 1) {
    if (KER == 2) return 0.0;  // dot = 0 on a straight segment
    const double h = X.h;
    const double L0 = log(0.25 * alpha) + 2.0 * log(h);
    for (int k = lane; k < n; k += 32) {
      const double rho = c_gx[n][k], w = h * rho, len = h - w;
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
      acc += G * (c_gw[n][k] * (R + P * L0) + 2.0 * c_glw[n][k] * P);
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
    const int npts = 2 * n * n;
    for (int idx = lane; idx < npts; idx += 32) {
      const int tri = idx / (n * n), ie = (idx / n) % n, ir = idx % n;
      const double eta = c_gx[n][ie], rho = c_gx[n][ir];
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
      acc += c_gw[n][ie] * f * (c_gw[n][ir] * (R + P * lnA) + 2.0 * c_glw[n][ir] * P);
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
    add = pair_touching<0>(seg[i], seg[jcol], rel, Lg, alpha, nsing, 1, 1, 1, 1);
  } else if (KIND == STB_K) {
    jcol = ((i + off - 1) % ng + ng) % ng;       // n = i-1 .. i+2
    const int jl = (jcol - 1 + ng) % ng;
    const int rl = chain_rel(i, jl, ng), rr = chain_rel(i, jcol, ng);
    if (rl) add += pair_touching<2>(seg[i], seg[jl], rl, Lg, alpha, nsing, 1, 1, 0, 1);
    if (rr) add += pair_touching<2>(seg[i], seg[jcol], rr, Lg, alpha, nsing, 1, 1, 1, 0);
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
        add += dvl[m] * dvk[nn_] * pair_touching<0>(X, Y, rel, Lg, alpha, nsing, 1, 1, 1, 1);
        const double nn = X.nx * Y.nx + X.ny * Y.ny;
        if (nn != 0.0)
          add += nn * pair_touching<1>(X, Y, rel, Lg, alpha, nsing, vl[m][0], vl[m][1], vk[nn_][0], vk[nn_][1]);
      }
  }
  if ((threadIdx.x & 31) == 0) *entry_ptr(B, a, i, b, jcol) += add;
}

// ================================================================= launch
template <int Q>
static void launch_bulk_q(int kind, const BlockArgs& BA, const bem_mesh* m, cudaStream_t st,
                          int nband) {
  const int ng = m->ng;
  constexpr int R = 8;
  if (kind == STB_V) {
    dim3 grid((ng + 31) / 32, (ng + 3) / 4, nband);
    k_bulk_V<Q, R><<<grid, 128, 0, st>>>(BA, m->d_seg, m->d_t, m->alpha, nband);
  } else if (kind == STB_K) {
    dim3 grid((ng + 30) / 31, (ng + 3) / 4, nband);
    k_bulk_K<Q, R><<<grid, 128, 0, st>>>(BA, m->d_seg, m->d_t, m->alpha, nband);
  } else {
    constexpr int TL = (Q <= 3) ? 7 : DTL_BULK;   // 16 warps at <= 128 registers for Q = 3
    dim3 grid((ng + DTK - 1) / DTK, (ng + TL - 1) / TL, nband);
    k_bulk_D<Q, 8, TL><<<grid, 32 * (2 * TL + 2), 0, st>>>(BA, m->d_half, m->d_dual, m->d_t, m->alpha, nband);
  }
  count_launch();
}

// exact evaluation counts of the shipped quadrature (host side, same rules as the kernels)
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
static long long near_point_pairs(int kind, const bem_mesh* m, int qfar) {
  // sum over (half-)segment pairs of q^2 x (kernel passes), touching pairs excluded
  long long acc = 0;
  const int ng = m->ng;
  if (kind == STB_D) {
    const int nh = 2 * ng;
    for (int p = 0; p < nh; ++p)
      for (int q = 0; q < nh; ++q) {
        if (chain_rel(p, q, nh)) continue;
        const Seg &X = m->half[p], &Y = m->half[q];
        const int qo = near_order(X, Y, qfar);
        acc += (long long)qo * qo;
      }
  } else {
    for (int i = 0; i < ng; ++i)
      for (int j = 0; j < ng; ++j) {
        if (chain_rel(i, j, ng)) continue;
        if (kind == STB_K && collinear(m->seg[i], m->seg[j])) continue;
        const int qo = near_order(m->seg[i], m->seg[j], qfar);
        acc += (long long)qo * qo;
      }
  }
  return acc;
}

bem_status launch_assembly(int kind, const bem_mesh* m, bem_matrix* A, int q_bulk, int q_sing,
                           cudaStream_t st) {
  const int ng = m->ng;
  long long* d_poff = nullptr;
  cudaError_t e = cudaMalloc(&d_poff, sizeof(long long) * std::max<size_t>(1, A->poff.size()));
  if (e != cudaSuccess) return cuda_fail(e, "assemble/poff");
  e = cudaMemcpyAsync(d_poff, A->poff.data(), sizeof(long long) * A->poff.size(), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) { cudaFree(d_poff); return cuda_fail(e, "assemble/poff copy"); }
  // CUDA events on the launching stream around each kernel family, per block
  std::vector<cudaEvent_t> ev;
  auto mark = [&]() {
    cudaEvent_t x;
    cudaEventCreate(&x);
    cudaEventRecord(x, st);
    ev.push_back(x);
  };
  std::vector<int> fam;  // family of the interval ending at ev[k+1]: 0 bulk, 1 near, 2 sing
  A->q_bulk = q_bulk;
  A->q_sing = q_sing;
  A->ev_bulk = A->ev_near = 0;
  A->launches = 0;
  const int qfar = std::min(6, q_bulk + 1);
  const long long near_pp = near_point_pairs(kind, m, qfar);
  const long long spatial = (kind == STB_D) ? 4LL * ng * ng : (long long)ng * ng;
  // algorithmic FP64 flops per bulk kernel evaluation (static count of the small-x path,
  // DFMA = 2): V 41, K 39 (collinear pairs skipped: K = 0 there),
  // D 80 (curl + normal term) or 41 (perpendicular half segments: curl only)
  double flops_per_node = 0.0;  // sum over spatial pairs of flops per point pair
  if (kind == STB_V) {
    flops_per_node = 41.0 * ng * ng;
  } else if (kind == STB_K) {
    for (int i = 0; i < ng; ++i)
      for (int j = 0; j < ng; ++j)
        if (!collinear(m->seg[i], m->seg[j])) flops_per_node += 39.0;
  } else {
    for (int p = 0; p < 2 * ng; ++p)
      for (int q = 0; q < 2 * ng; ++q) {
        const Seg &X = m->half[p], &Y = m->half[q];
        flops_per_node += (X.nx * Y.nx + X.ny * Y.ny) != 0.0 ? 80.0 : 41.0;
      }
  }
  A->flops_bulk = 0.0;
  mark();
  for (size_t bi = 0; bi < m->blocks.size(); ++bi) {
    const Block& blk = m->blocks[bi];
    BlockArgs BA;
    BA.out = A->data;
    BA.poff = d_poff + A->poff_base[bi];
    BA.a0 = blk.a0; BA.a1 = blk.a1; BA.b0 = blk.b0; BA.b1 = blk.b1;
    BA.ng = ng;
    BA.lag = m->d_lag;
    BA.ldlag = m->nt + 1;
    BA.qfar = qfar;
    const int R = 8;
    const int nband = (blk.a1 - blk.a0 + R - 1) / R;
    if (blk.a1 - 1 - blk.b0 >= 2) {
      switch (q_bulk) {
        case 3: launch_bulk_q<3>(kind, BA, m, st, nband); break;
        case 4: launch_bulk_q<4>(kind, BA, m, st, nband); break;
        case 5: launch_bulk_q<5>(kind, BA, m, st, nband); break;
        case 6: launch_bulk_q<6>(kind, BA, m, st, nband); break;
        default: launch_bulk_q<8>(kind, BA, m, st, nband); break;
      }
      mark();
      fam.push_back(0);
      A->launches++;
      const long long nodes = bulk_nodes(blk, R);
      A->ev_bulk += nodes * spatial * q_bulk * q_bulk;
      A->flops_bulk += (double)nodes * q_bulk * q_bulk * flops_per_node;
    }
    const bool has_near = blk.b1 - 1 >= blk.a0 - 1 && blk.b0 <= blk.a1 - 1;
    if (has_near) {
      const int ncell = 2 * (blk.a1 - blk.a0);
      long long lags = 0;
      for (int a = blk.a0; a < blk.a1; ++a) {
        if (a >= blk.b0 && a < blk.b1) lags += 1;                // d = 0: one lag
        if (a - 1 >= blk.b0 && a - 1 < blk.b1) lags += 3;        // d = 1: three lags
      }
      A->ev_near += lags * near_pp;
      if (kind == STB_D) {
        dim3 grid((ng + DTK - 1) / DTK, (ng + DTL_NEAR - 1) / DTL_NEAR, ncell);
        k_near_D<DTL_NEAR><<<grid, 32 * (2 * DTL_NEAR + 2), 0, st>>>(BA, m->d_half, m->d_dual, m->d_t, m->alpha);
      } else {
        dim3 grid((ng + 31) / 32, (ng + 3) / 4, ncell);
        if (kind == STB_V) k_near_VK<STB_V><<<grid, 128, 0, st>>>(BA, m->d_seg, m->d_t, m->alpha);
        else k_near_VK<STB_K><<<grid, 128, 0, st>>>(BA, m->d_seg, m->d_t, m->alpha);
      }
      count_launch();
      mark();
      fam.push_back(1);
      const int per_row = kind == STB_V ? 3 : (kind == STB_K ? 4 : 5);
      const long long nwarps = (long long)ncell * ng * per_row;
      const unsigned nblk = (unsigned)((nwarps + 3) / 4);
      if (kind == STB_V) k_sing<STB_V><<<nblk, 128, 0, st>>>(BA, m->d_seg, m->d_half, m->d_dual, m->d_t, m->alpha, q_sing, nwarps);
      else if (kind == STB_K) k_sing<STB_K><<<nblk, 128, 0, st>>>(BA, m->d_seg, m->d_half, m->d_dual, m->d_t, m->alpha, q_sing, nwarps);
      else k_sing<STB_D><<<nblk, 128, 0, st>>>(BA, m->d_seg, m->d_half, m->d_dual, m->d_t, m->alpha, q_sing, nwarps);
      count_launch();
      mark();
      fam.push_back(2);
      A->launches += 2;
    }
  }
  e = cudaGetLastError();
  cudaStreamSynchronize(st);
  A->ms_bulk = A->ms_near = A->ms_sing = 0.0;
  for (size_t k = 0; k + 1 < ev.size(); ++k) {
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
    (fam[k] == 0 ? A->ms_bulk : fam[k] == 1 ? A->ms_near : A->ms_sing) += ms;
  }
  for (auto x : ev) cudaEventDestroy(x);
  cudaFree(d_poff);
  if (e != cudaSuccess) return cuda_fail(e, "assemble/launch");
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "assemble/kernels");
  return BEM_OK;
}

}  // namespace stb
