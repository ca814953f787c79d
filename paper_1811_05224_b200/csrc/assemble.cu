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

__device__ __forceinline__ double seg_dist(const Seg& X, const Seg& Y) {
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
__device__ __forceinline__ int near_order(const Seg& X, const Seg& Y) {
  double rho = seg_dist(X, Y) / fmax(X.h, Y.h);
  return rho < 2.5 ? 10 : (rho < 5.0 ? 8 : 6);
}
// relation of elements p, q of a closed chain of n: 0 disjoint, 1 identical,
// 2 X.end == Y.start, 3 X.start == Y.end
__device__ __forceinline__ int chain_rel(int p, int q, int n) {
  if (p == q) return 1;
  if ((p + 1) % n == q) return 2;
  if ((q + 1) % n == p) return 3;
  return 0;
}
__device__ __forceinline__ bool collinear(const Seg& X, const Seg& Y) {
  double d0 = (X.ax - Y.ax) * Y.nx + (X.ay - Y.ay) * Y.ny;
  double d1 = (X.bx - Y.ax) * Y.nx + (X.by - Y.ay) * Y.ny;
  double tol = 1e-13 * fmax(X.h, Y.h);
  return fabs(d0) < tol && fabs(d1) < tol;
}

// ================================================================= bulk V
// thread = segment pair (i, j): warp = row i, lane = column j; band of R test steps
template <int Q, int R>
__global__ void __launch_bounds__(128) k_bulk_V(BlockArgs B, const Seg* __restrict__ seg,
                                                const double* __restrict__ t, double alpha,
                                                int nband) {
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
  double c[Q * Q], L[Q * Q], ic[Q * Q];
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
      ic[u * Q + v] = cc > 0.0 ? 1.0 / cc : 0.0;
    }
  }
  const double scale = X.h * Y.h / (4.0 * STB_PI);
  double Gp[R];
#pragma unroll
  for (int r = 0; r < R; ++r) Gp[r] = 0.0;
  for (int y = B.b0; y <= bmax + 1; ++y) {
    const double ty = t[y];
    double Phi[R + 1];
#pragma unroll
    for (int r = 0; r <= R; ++r) {
      const int x = r_lo + r;
      Phi[r] = 0.0;
      if (x <= r_hi && x > y) {
        const double s = t[x] - ty;
        const double lns = log(s), is = 1.0 / s;
        double acc = 0.0;
#pragma unroll
        for (int u = 0; u < Q; ++u) {
          double part = 0.0;
#pragma unroll
          for (int v = 0; v < Q; ++v) {
            const int p = u * Q + v;
            const double xx = c[p] * is;
            const double gl = STB_GAMMA + (reg ? 0.0 : L[p]) - lns;
            part = fma(c_gw[Q][v], bulk_h(xx, gl, s * ic[p], reg ? L[p] : 0.0), part);
          }
          acc = fma(c_gw[Q][u], part, acc);
        }
        Phi[r] = s * acc;
      }
    }
    if (y > B.b0) {
      const int b = y - 1;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int a = r_lo + r;
        const double G = Phi[r + 1] - Phi[r];
        if (a < r_hi && a - b >= 2) *entry_ptr(B, a, i, b, j) = scale * (Gp[r] - G);
        Gp[r] = G;
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) Gp[r] = Phi[r + 1] - Phi[r];
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
  double c[Q * Q], L[Q * Q], ic[Q * Q], dw[Q * Q];
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
      ic[u * Q + v] = 1.0 / cc;
      dw[u * Q + v] = zero ? 0.0 : c_gw[Q][u] * c_gw[Q][v] * (dx * Y.nx + dy * Y.ny);
    }
  }
  const double scale = alpha / (8.0 * STB_PI) * X.h * Y.h;
  double Gp0[R], Gp1[R];
#pragma unroll
  for (int r = 0; r < R; ++r) Gp0[r] = Gp1[r] = 0.0;
  for (int y = B.b0; y <= bmax + 1; ++y) {
    const double ty = t[y];
    double P0[R + 1], P1[R + 1];
#pragma unroll
    for (int r = 0; r <= R; ++r) {
      const int x = r_lo + r;
      P0[r] = P1[r] = 0.0;
      if (x <= r_hi && x > y && !zero) {
        const double s = t[x] - ty;
        const double lns = log(s), is = 1.0 / s;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int p = 0; p < Q * Q; ++p) {
          const double xx = c[p] * is;
          const double ps = dw[p] * bulk_psi(xx, STB_GAMMA + L[p] - lns, s * ic[p]);
          const double f = c_gx[Q][p % Q];
          a1 = fma(f, ps, a1);
          a0 += ps;
        }
        P0[r] = a0 - a1;   // lambda_0 = 1 - f
        P1[r] = a1;
      }
    }
    if (y > B.b0) {
      const int b = y - 1;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int a = r_lo + r;
        const double G0 = P0[r + 1] - P0[r], G1 = P1[r + 1] - P1[r];
        if (a < r_hi && a - b >= 2) {
          const double m0 = Gp0[r] - G0, m1 = Gp1[r] - G1;
          const double left = __shfl_up_sync(0xffffffffu, m1, 1);
          if (out_ok) *entry_ptr(B, a, i, b, n) = scale * (left + m0);
        }
        Gp0[r] = G0;
        Gp1[r] = G1;
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        Gp0[r] = P0[r + 1] - P0[r];
        Gp1[r] = P1[r + 1] - P1[r];
      }
    }
  }
}

// ================================================================= D tiles
// CTA: warp w <-> half row p = 2 L0 - 1 + w (w < 2 TL + 2), lane <-> half column
// q = 2 K0 - 1 + lane; entries (l, k), l in [L0, L0+TL), k in [K0, K0+15).
constexpr int DTL = 3;
constexpr int DTK = 15;
constexpr int DWARPS = 2 * DTL + 2;  // 8

struct DMom {
  double v, f00, f01, f10, f11;
};

// combine the 5 half-pair moments of the CTA into D entries and store them
__device__ __forceinline__ void d_combine_store(const BlockArgs& B, const Dual* __restrict__ dual,
                                                const Seg* __restrict__ half, double (*sm)[32][5],
                                                int L0, int K0, int a, int b, bool add) {
  const int ng = B.ng, nh = 2 * ng;
  for (int e = threadIdx.x; e < DTL * DTK; e += blockDim.x) {
    const int l = L0 + e / DTK, k = K0 + e % DTK;
    if (l >= ng || k >= ng) continue;
    const Dual dl = dual[l], dk = dual[k];
    const double dvl[4] = {1.0 / dl.Lm, 1.0 / dl.Lm, -1.0 / dl.Lp, -1.0 / dl.Lp};
    const double dvk[4] = {1.0 / dk.Lm, 1.0 / dk.Lm, -1.0 / dk.Lp, -1.0 / dk.Lp};
    const double vl[4][2] = {{0.0, dl.vm}, {dl.vm, 1.0}, {1.0, dl.vp}, {dl.vp, 0.0}};
    const double vk[4][2] = {{0.0, dk.vm}, {dk.vm, 1.0}, {1.0, dk.vp}, {dk.vp, 0.0}};
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int pl = 2 * (l - L0) + m;
      const Seg& Hp = half[((2 * l - 1 + m) % nh + nh) % nh];
#pragma unroll
      for (int nn_ = 0; nn_ < 4; ++nn_) {
        const int ql = 2 * (k - K0) + nn_;
        const Seg& Hq = half[((2 * k - 1 + nn_) % nh + nh) % nh];
        const double nn = Hp.nx * Hq.nx + Hp.ny * Hq.ny;
        const double* M = sm[pl][ql];
        double fn = vl[m][0] * (vk[nn_][0] * M[1] + vk[nn_][1] * M[2]) +
                    vl[m][1] * (vk[nn_][0] * M[3] + vk[nn_][1] * M[4]);
        acc += dvl[m] * dvk[nn_] * M[0] + nn * fn;
      }
    }
    double* p = entry_ptr(B, a, l, b, k);
    if (add) *p += acc; else *p = acc;
  }
}

template <int Q, int R>
__global__ void __launch_bounds__(256) k_bulk_D(BlockArgs B, const Seg* __restrict__ half,
                                                const Dual* __restrict__ dual,
                                                const double* __restrict__ t, double alpha,
                                                int nband) {
  __shared__ double sm[R][DWARPS][32][5];
  const int ng = B.ng, nh = 2 * ng;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int K0 = blockIdx.x * DTK, L0 = blockIdx.y * DTL;
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
  const bool do_f = (X.nx * Y.nx + X.ny * Y.ny) != 0.0;
  double c[Q * Q], L[Q * Q], ic[Q * Q];
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
      ic[u * Q + v] = cc > 0.0 ? 1.0 / cc : 0.0;
    }
  }
  const double sv = X.h * Y.h / (4.0 * STB_PI), sf = alpha * X.h * Y.h / (4.0 * STB_PI);
  DMom Gp[R];
#pragma unroll
  for (int r = 0; r < R; ++r) Gp[r] = DMom{0, 0, 0, 0, 0};
  for (int y = B.b0; y <= bmax + 1; ++y) {
    const double ty = t[y];
    DMom Phi[R + 1];
#pragma unroll
    for (int r = 0; r <= R; ++r) {
      const int x = r_lo + r;
      Phi[r] = DMom{0, 0, 0, 0, 0};
      if (x <= r_hi && x > y) {
        const double s = t[x] - ty;
        const double lns = log(s), is = 1.0 / s;
        double av = 0.0, a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0;
#pragma unroll
        for (int u = 0; u < Q; ++u) {
          double tv = 0.0, tf0 = 0.0, tf1 = 0.0;
#pragma unroll
          for (int v = 0; v < Q; ++v) {
            const int pp = u * Q + v;
            const double xx = c[pp] * is;
            const double gl = STB_GAMMA + (reg ? 0.0 : L[pp]) - lns;
            double hv, ev;
            bulk_h_e1(xx, gl, s * ic[pp], reg ? L[pp] : 0.0, hv, ev);
            const double wv = c_gw[Q][v], fv = c_gx[Q][v];
            tv = fma(wv, hv, tv);
            const double we = wv * ev;
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
        Phi[r].v = sv * s * av;
        if (do_f) {
          Phi[r].f00 = sf * a00;
          Phi[r].f01 = sf * a01;
          Phi[r].f10 = sf * a10;
          Phi[r].f11 = sf * a11;
        }
      }
    }
    if (y > B.b0) {
      const int b = y - 1;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        DMom G{Phi[r + 1].v - Phi[r].v, Phi[r + 1].f00 - Phi[r].f00, Phi[r + 1].f01 - Phi[r].f01,
               Phi[r + 1].f10 - Phi[r].f10, Phi[r + 1].f11 - Phi[r].f11};
        double* M = sm[r][w][lane];
        M[0] = Gp[r].v - G.v;
        M[1] = Gp[r].f00 - G.f00;
        M[2] = Gp[r].f01 - G.f01;
        M[3] = Gp[r].f10 - G.f10;
        M[4] = Gp[r].f11 - G.f11;
        Gp[r] = G;
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int a = r_lo + r;
        if (a < r_hi && a - b >= 2) d_combine_store(B, dual, half, sm[r], L0, K0, a, b, false);
      }
      __syncthreads();
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r)
        Gp[r] = DMom{Phi[r + 1].v - Phi[r].v, Phi[r + 1].f00 - Phi[r].f00, Phi[r + 1].f01 - Phi[r].f01,
                     Phi[r + 1].f10 - Phi[r].f10, Phi[r + 1].f11 - Phi[r].f11};
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
    if (chain_rel(i, j, ng) == 0) val = pair_regular<0>(X, Y, Lg, alpha, near_order(X, Y), 1, 1, 1, 1);
  } else {
    const int jl = (j - 1 + ng) % ng;
    const Seg Yl = seg[jl], Yr = seg[j];
    if (chain_rel(i, jl, ng) == 0 && !collinear(X, Yl))
      val += pair_regular<2>(X, Yl, Lg, alpha, near_order(X, Yl), 1, 1, 0, 1);
    if (chain_rel(i, j, ng) == 0 && !collinear(X, Yr))
      val += pair_regular<2>(X, Yr, Lg, alpha, near_order(X, Yr), 1, 1, 1, 0);
  }
  *entry_ptr(B, a, i, b, j) = val;
}

// D near cells: half-pair threads in the D tile, 5 moments each, smem combine
__global__ void __launch_bounds__(256) k_near_D(BlockArgs B, const Seg* __restrict__ half,
                                                const Dual* __restrict__ dual,
                                                const double* __restrict__ t, double alpha) {
  __shared__ double sm[DWARPS][32][5];
  const int ng = B.ng, nh = 2 * ng;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int K0 = blockIdx.x * DTK, L0 = blockIdx.y * DTL;
  const int cell = blockIdx.z;
  const int a = B.a0 + cell / 2, b = a - (cell % 2);
  if (a >= B.a1 || b < B.b0 || b >= B.b1) return;
  const int p = ((2 * L0 - 1 + w) % nh + nh) % nh;
  const int q = ((2 * K0 - 1 + lane) % nh + nh) % nh;
  const Seg X = half[p], Y = half[q];
  const Lags Lg = make_lags(t, a, b);
  double* M = sm[w][lane];
  M[0] = M[1] = M[2] = M[3] = M[4] = 0.0;
  if (chain_rel(p, q, nh) == 0) {
    const int qo = near_order(X, Y);
    M[0] = pair_regular<0>(X, Y, Lg, alpha, qo, 1, 1, 1, 1);
    if ((X.nx * Y.nx + X.ny * Y.ny) != 0.0) {
      M[1] = pair_regular<1>(X, Y, Lg, alpha, qo, 1, 0, 1, 0);
      M[2] = pair_regular<1>(X, Y, Lg, alpha, qo, 1, 0, 0, 1);
      M[3] = pair_regular<1>(X, Y, Lg, alpha, qo, 0, 1, 1, 0);
      M[4] = pair_regular<1>(X, Y, Lg, alpha, qo, 0, 1, 0, 1);
    }
  }
  __syncthreads();
  d_combine_store(B, dual, half, sm, L0, K0, a, b, false);
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
  constexpr int R = 4;
  if (kind == STB_V) {
    dim3 grid((ng + 31) / 32, (ng + 3) / 4, nband);
    k_bulk_V<Q, R><<<grid, 128, 0, st>>>(BA, m->d_seg, m->d_t, m->alpha, nband);
  } else if (kind == STB_K) {
    dim3 grid((ng + 30) / 31, (ng + 3) / 4, nband);
    k_bulk_K<Q, R><<<grid, 128, 0, st>>>(BA, m->d_seg, m->d_t, m->alpha, nband);
  } else {
    dim3 grid((ng + DTK - 1) / DTK, (ng + DTL - 1) / DTL, nband);
    k_bulk_D<Q, 2><<<grid, 32 * DWARPS, 0, st>>>(BA, m->d_half, m->d_dual, m->d_t, m->alpha, nband);
  }
  count_launch();
}

bem_status launch_assembly(int kind, const bem_mesh* m, bem_matrix* A, int q_bulk, int q_sing,
                           cudaStream_t st) {
  const int ng = m->ng;
  long long* d_poff = nullptr;
  cudaError_t e = cudaMalloc(&d_poff, sizeof(long long) * std::max<size_t>(1, A->poff.size()));
  if (e != cudaSuccess) return cuda_fail(e, "assemble/poff");
  e = cudaMemcpyAsync(d_poff, A->poff.data(), sizeof(long long) * A->poff.size(), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) { cudaFree(d_poff); return cuda_fail(e, "assemble/poff copy"); }
  for (size_t bi = 0; bi < m->blocks.size(); ++bi) {
    const Block& blk = m->blocks[bi];
    BlockArgs BA;
    BA.out = A->data;
    BA.poff = d_poff + A->poff_base[bi];
    BA.a0 = blk.a0; BA.a1 = blk.a1; BA.b0 = blk.b0; BA.b1 = blk.b1;
    BA.ng = ng;
    // bulk: cells d >= 2 exist if a1 - 1 - (b0) >= 2
    const int R = (kind == STB_D) ? 2 : 4;
    const int nband = (blk.a1 - blk.a0 + R - 1) / R;
    if (blk.a1 - 1 - blk.b0 >= 2) {
      switch (q_bulk) {
        case 3: launch_bulk_q<3>(kind, BA, m, st, nband); break;
        case 4: launch_bulk_q<4>(kind, BA, m, st, nband); break;
        case 5: launch_bulk_q<5>(kind, BA, m, st, nband); break;
        case 6: launch_bulk_q<6>(kind, BA, m, st, nband); break;
        default: launch_bulk_q<8>(kind, BA, m, st, nband); break;
      }
    }
    // near cells (d <= 1) and touching pairs, only where such cells exist in this block
    const bool has_near = blk.b1 - 1 >= blk.a0 - 1 && blk.b0 <= blk.a1 - 1;
    if (has_near) {
      const int ncell = 2 * (blk.a1 - blk.a0);
      if (kind == STB_D) {
        dim3 grid((ng + DTK - 1) / DTK, (ng + DTL - 1) / DTL, ncell);
        k_near_D<<<grid, 32 * DWARPS, 0, st>>>(BA, m->d_half, m->d_dual, m->d_t, m->alpha);
      } else {
        dim3 grid((ng + 31) / 32, (ng + 3) / 4, ncell);
        if (kind == STB_V) k_near_VK<STB_V><<<grid, 128, 0, st>>>(BA, m->d_seg, m->d_t, m->alpha);
        else k_near_VK<STB_K><<<grid, 128, 0, st>>>(BA, m->d_seg, m->d_t, m->alpha);
      }
      count_launch();
      const int per_row = kind == STB_V ? 3 : (kind == STB_K ? 4 : 5);
      const long long nwarps = (long long)ncell * ng * per_row;
      const unsigned nblk = (unsigned)((nwarps + 3) / 4);
      if (kind == STB_V) k_sing<STB_V><<<nblk, 128, 0, st>>>(BA, m->d_seg, m->d_half, m->d_dual, m->d_t, m->alpha, q_sing, nwarps);
      else if (kind == STB_K) k_sing<STB_K><<<nblk, 128, 0, st>>>(BA, m->d_seg, m->d_half, m->d_dual, m->d_t, m->alpha, q_sing, nwarps);
      else k_sing<STB_D><<<nblk, 128, 0, st>>>(BA, m->d_seg, m->d_half, m->d_dual, m->d_t, m->alpha, q_sing, nwarps);
      count_launch();
    }
  }
  e = cudaGetLastError();
  cudaStreamSynchronize(st);
  cudaFree(d_poff);
  if (e != cudaSuccess) return cuda_fail(e, "assemble/launch");
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "assemble/kernels");
  return BEM_OK;
}

}  // namespace stb
