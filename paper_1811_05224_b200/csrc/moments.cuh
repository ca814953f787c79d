// moments.cuh — separable (moment) evaluation of the regular-pair space-time integrals,
// included by assemble.cu (one translation unit: the Gauss tables live in __constant__ there).
//
// An entry of time cell (a,b) is the four-lag second difference of node values
//   Phi(x, y) = sum_p W_p G(t_x - t_y; c_p),   c_p = alpha r_p^2 / 4
// over the quadrature points p of the (half-)segment pairs that make up one matrix entry, with
// G the double (V, D curl: H) or single (D normal: F; K: Q) time antiderivative.  G depends on
// the point only through c and on the node only through s = t_x - t_y.  Terms of G that are
// affine in s with point-only coefficients cancel in every second difference whose four lags are
// positive (sum eps_m s_m = 0, sum eps_m = 0), so the bulk evaluates the regularised
//   H~ = s h(x) + (s+c)(gamma + ln c)      = s GH(x) + (s+c) ln s          (x = c/s)
//   F~ = E1(x) + gamma + ln c              = Ein(x) + ln s
//   Q~ = e^{-x}/x - E1(x) - s/c - gamma - ln c = PSI(x) - ln s
// (GH, Ein, PSI entire).  Three regimes per (entry, node), chosen per lane:
//   A  x_max = c_max/s < 8 in the bulk cells (< 4 in the near cells and touching records): the
//      polynomials of moment_coeffs.h in x (degree 20 on [0, 8]), so the sum over points is
//      sum_k f_k s^{-k} M_k with time-independent moments M_k = sum_p W_p c_p^k: one Horner
//      chain in u = 1/s per kernel family, independent of the number of quadrature points.
//   B  the points are clustered, rho = (c_max - c0)/c0 <= 0.5: Taylor expansion in c around c0
//      with shifted moments m_k = sum_p W_p (c_p - c0)^k; the node-dependent Taylor
//      coefficients of E1 / (1+x)E1 - e^{-x} / e^{-x}/x - E1 come from the recurrence for
//      e^{-x}/x (x f = e^{-x}).  The remainder is bounded by rho^K (the pole of E1' at c = 0)
//      and e^{-x0} (rho x0)^K / K! <= rho^K / sqrt(2 pi K) (the exponential), so the order per
//      pair is K = min(56, ceil(ln 1e-17 / ln rho)) (relative error ~1e-17..1e-16 sum |W|).
//   Z  x_min >= 50: the E1 / exp parts are below 1e-23; only the affine constants remain.
//   C  otherwise: the point-by-point sum (same quadrature), dealt over the 32 lanes of the warp.
// The records (moments and constants) depend on the spatial pair only: built once per
// assembly by k_records, reused by every block, band and time node.
#pragma once
#include <type_traits>

#include "moment_coeffs.h"

namespace stb {

constexpr int MKA = 20;          // regime-A polynomial degree (MGH, MEIN, MPSI on [0, 8])
constexpr int MKB = 56;          // regime-B maximum Taylor order
constexpr double MRHO = 0.5;     // regime-B cluster bound (c_max - c0 <= MRHO c0)
constexpr double MXZ = 50.0;     // regime Z threshold on x_min
// record layout (field-major, stride npairs): common fields, then one block per family
enum { RF_CMAX = 0, RF_CMIN = 1, RF_C0 = 2, RF_KB = 3, RF_IC0 = 4, RF_COMMON = 5 };
// per family: A[0..MKA] = poly_k M_k, M0, M1, the regime-B arrays B1, B2 (scaled shifted
// moments, see phi_bz), the affine constants C0, C1
enum { FA = 0, FM0 = MKA + 1, FM1 = MKA + 2, FB1 = MKA + 3, FB2 = FB1 + MKB + 1, FC0 = FB2 + MKB + 1,
       FC1 = FC0 + 1, FAMSZ = FC1 + 1 };
enum { FAM_H = 0, FAM_F = 1, FAM_Q = 2 };

template <int KIND> struct Fams;
template <> struct Fams<STB_V> { static constexpr int n = 1, f0 = FAM_H, f1 = -1; };
template <> struct Fams<STB_K> { static constexpr int n = 1, f0 = FAM_Q, f1 = -1; };
template <> struct Fams<STB_D> { static constexpr int n = 2, f0 = FAM_H, f1 = FAM_F; };
template <int KIND> constexpr int rec_fields() { return RF_COMMON + Fams<KIND>::n * FAMSZ; }
// near records append a second regime-B cluster (regime B2): c0, 1/c0, order and
// split point c_s of the cluster c > c_s, then per family its two coefficient arrays (m_0 and m_1
// in their last slots, as for the first cluster)
enum { R2_C0 = 0, R2_IC0 = 1, R2_KB = 2, R2_CS = 3, R2_FAM = 4, R2_FAMSZ = 2 * (MKB + 1) };
template <int KIND> constexpr int rec2_base() { return rec_fields<KIND>(); }
template <int KIND> constexpr int rec_fields_near() { return rec_fields<KIND>() + R2_FAM + Fams<KIND>::n * R2_FAMSZ; }

static __device__ __constant__ const double STB_INV[MKB + 2] = {
    0.0, 1.0, 1.0 / 2, 1.0 / 3, 1.0 / 4, 1.0 / 5, 1.0 / 6, 1.0 / 7,
    1.0 / 8, 1.0 / 9, 1.0 / 10, 1.0 / 11, 1.0 / 12, 1.0 / 13, 1.0 / 14, 1.0 / 15,
    1.0 / 16, 1.0 / 17, 1.0 / 18, 1.0 / 19, 1.0 / 20, 1.0 / 21, 1.0 / 22, 1.0 / 23,
    1.0 / 24, 1.0 / 25, 1.0 / 26, 1.0 / 27, 1.0 / 28, 1.0 / 29, 1.0 / 30, 1.0 / 31,
    1.0 / 32, 1.0 / 33, 1.0 / 34, 1.0 / 35, 1.0 / 36, 1.0 / 37, 1.0 / 38, 1.0 / 39,
    1.0 / 40, 1.0 / 41, 1.0 / 42, 1.0 / 43, 1.0 / 44, 1.0 / 45, 1.0 / 46, 1.0 / 47,
    1.0 / 48, 1.0 / 49, 1.0 / 50, 1.0 / 51, 1.0 / 52, 1.0 / 53, 1.0 / 54, 1.0 / 55,
    1.0 / 56, 1.0 / 57};

#define STB_INV_H STB_INV

__device__ __forceinline__ double mpoly(int fam, int k) {
  if (fam == FAM_H) return STB_MGH[k];
  if (fam == FAM_F) return STB_MEIN[k];
  return k <= STB_MPSI_DEG ? STB_MPSI[k] : 0.0;
}

struct MomArgs {
  double* rec;            // record storage (rec_fields x npairs)
  long long npairs;       // ng * ng
  const Seg* seg;
  const Seg* half;
  const Dual* dual;
  double alpha;
  int ng;
  int q;                  // bulk Gauss order (bulk records)
  int qfar;               // near-cell order of well-separated pairs (near records)
  unsigned long long* counters;  // node evaluations per regime: A, B, Z, C
  double u_near[2];       // near records: smallest and largest 1/s of the near-cell nodes
  double ell;             // sqrt(4 min h_t / alpha): the length on which U* varies at the
                          // smallest lag; sub-pairs closer than 8 ell get composite rules with
                          // cells of at most ell (no subdivision while kappa <= 1)
  double near_gap;        // near records: distance ratio below which the measured orders apply
  int* list;              // D_h near records: [0] count, [1..] the near_special pairs (k_records appends)
  // records kernels: the pairs (I, J) in chunks of rpc test segments I (cs = rpc N_Gamma pairs),
  // chunk c holding nfc fields of stride cs; one chunk (rpc = N_Gamma, cs = npairs: the layout the
  // bulk and near kernels read) on one rank.  Distributed (G ranks): rank r computes the pairs
  // [p_lo, p_hi) of chunk r into a staging buffer
  long long cs = 0;
  int nfc = 0, rpc = 0;
  long long p_lo = 0, p_hi = 0;
};
// offset of pair (I, J)'s record in the records kernels' layout (32-bit division)
__device__ __forceinline__ long long rec_base(const MomArgs& M, int I, int J) {
  const int c = I / M.rpc, r = I - c * M.rpc;
  return (long long)c * M.nfc * M.cs + (long long)r * M.ng + J;
}

// composite subdivision of a sub-pair: cells per direction.  R24: pairs
// closer than 8 ell with elements longer than ell; R25 (NEAR: the near cells keep the ln c and 1/c
// parts of the kernel): disjoint pairs closer than their length, cells of the distance's size
// vertex pairs at an acute angle (cos > 1/2): the Duffy integrand's A(eta) = |x - y|^2 / rho^2 dips
// to sin^2 of the angle, with complex zeros that close distance from [0,1]: cells in eta of about
// sin(theta) / 1.5 (reading R25); right and obtuse angles keep one cell
__host__ __device__ inline int acute_cells(double cth) {
  if (!(cth > 0.5)) return 1;
  const int ne = (int)ceil(1.5 / sqrt(fmax(1e-12, 1.0 - cth * cth)));
  return ne > 16 ? 16 : ne;
}
template <bool NEAR>
__device__ __forceinline__ int composite_cells(const Seg& X, const Seg& Y, double ell) {
  const double hm = fmax(X.h, Y.h);
  int ns = 1;
  if (ell > 0.0 && hm > ell) {
    const double d = seg_dist(X, Y);
    if (d < 8.0 * ell) ns = min(24, (int)ceil(hm / ell));
  }
  if (NEAR) {
    const double d = seg_dist(X, Y);
    if (d < hm) ns = max(ns, min(16, (int)ceil(2.0 * hm / d)));
  }
  return ns;
}

// ------------------------------------------------------------- point enumeration
// Visits every quadrature point of the (half-)segment pairs that make up entry (I, J) with its
// weights for the kernel families of KIND: vis(c, w_first_family, w_second_family).
//   V: (seg I, seg J), H weight h_X h_Y w_u w_v / 4pi
//   K: entry (i, n) of the primal hat phi_n: (seg i, seg n-1) rising, (seg i, seg n) falling;
//      Q weight alpha h_X h_Y w_u w_v ((x - y).n_y) phi_n(y) / 8pi; collinear pairs are 0
//   D: dual hats psi_l, psi_k on their 4 half segments each (R6, R7): curl weight
//      h_X h_Y w_u w_v psi_l' psi_k' / 4pi (H), normal weight alpha h_X h_Y w_u w_v
//      (n_x.n_y) psi_l psi_k / 4pi (F)
// NEAR: touching sub-pairs are skipped (k_sing adds them) and the order follows the distance.
struct SubPair {
  Seg X, Y;
  int pi, qi, nchain;       // element indices of X and Y in their closed chain of nchain elements
  int q;
  int ns;                   // composite cells per direction (1 = plain tensor Gauss)
  int side;                 // K: 0 = gamma_{n-1} (hat rising), 1 = gamma_n (falling)
  double sa, sb;            // weight scales of the two families
  double l0, l1, k0, k1;    // D: psi_l on X and psi_k on Y, linear from (l0 / k0) to (l1 / k1)
};

template <int KIND, bool NEAR, class Fn>
__device__ __forceinline__ void for_subpairs(const MomArgs& M, int I, int J, Fn&& fn) {
  const int ng = M.ng;
  SubPair sp;
  if (KIND == STB_V) {
    if (NEAR && chain_rel(I, J, ng)) return;
    sp.X = M.seg[I];
    sp.Y = M.seg[J];
    sp.pi = I;
    sp.qi = J;
    sp.nchain = ng;
    sp.q = NEAR ? near_order(sp.X, sp.Y, M.qfar, M.near_gap) : M.q;
    sp.ns = composite_cells<NEAR>(sp.X, sp.Y, M.ell);
    sp.sa = sp.X.h * sp.Y.h / (4.0 * STB_PI);
    sp.sb = 0.0;
    fn(sp);
  } else if (KIND == STB_K) {
    sp.X = M.seg[I];
#pragma unroll 1
    for (int side = 0; side < 2; ++side) {
      const int j = side == 0 ? (J - 1 + ng) % ng : J;
      sp.Y = M.seg[j];
      sp.pi = I;
      sp.qi = j;
      sp.nchain = ng;
      if (collinear(sp.X, sp.Y)) continue;
      if (NEAR && chain_rel(I, j, ng)) continue;
      sp.q = NEAR ? near_order(sp.X, sp.Y, M.qfar, M.near_gap) : M.q;
      sp.ns = composite_cells<NEAR>(sp.X, sp.Y, M.ell);
      sp.side = side;
      sp.sa = M.alpha / (8.0 * STB_PI) * sp.X.h * sp.Y.h;
      sp.sb = 0.0;
      fn(sp);
    }
  } else {
    const int nh = 2 * ng;
    const Dual dl = M.dual[I], dk = M.dual[J];
#pragma unroll 1
    for (int m = 0; m < 4; ++m) {
      const int p = (2 * I - 1 + m + nh) % nh;
      sp.X = M.half[p];
      const double dvl = m < 2 ? 1.0 / dl.Lm : -1.0 / dl.Lp;
      sp.l0 = m == 0 ? 0.0 : (m == 1 ? dl.vm : (m == 2 ? 1.0 : dl.vp));
      sp.l1 = m == 0 ? dl.vm : (m == 1 ? 1.0 : (m == 2 ? dl.vp : 0.0));
#pragma unroll 1
      for (int n = 0; n < 4; ++n) {
        const int qh = (2 * J - 1 + n + nh) % nh;
        if (NEAR && chain_rel(p, qh, nh)) continue;
        sp.Y = M.half[qh];
        sp.pi = p;
        sp.qi = qh;
        sp.nchain = nh;
        sp.q = NEAR ? near_order(sp.X, sp.Y, M.qfar, M.near_gap) : M.q;
        sp.ns = composite_cells<NEAR>(sp.X, sp.Y, M.ell);
        const double dvk = n < 2 ? 1.0 / dk.Lm : -1.0 / dk.Lp;
        sp.k0 = n == 0 ? 0.0 : (n == 1 ? dk.vm : (n == 2 ? 1.0 : dk.vp));
        sp.k1 = n == 0 ? dk.vm : (n == 1 ? 1.0 : (n == 2 ? dk.vp : 0.0));
        const double hh = sp.X.h * sp.Y.h / (4.0 * STB_PI);
        sp.sa = hh * dvl * dvk;
        sp.sb = M.alpha * hh * (sp.X.nx * sp.Y.nx + sp.X.ny * sp.Y.ny);
        fn(sp);
      }
    }
  }
}

// quadrature point (u, v) of a sub-pair: c = alpha r^2 / 4 and the two family weights
// (composite cell cu, node uu) x (cell cv, node vv); cells of width 1 / ns on [0, 1]
template <int KIND>
__device__ __forceinline__ void sub_point(const SubPair& sp, double alpha, int cu, int uu, int cv, int vv,
                                          double& c, double& wa, double& wb) {
  const int q = sp.q;
  const double ins = sp.ns == 1 ? 1.0 : 1.0 / sp.ns;
  const double fu = (cu + c_gx[q][uu]) * ins, fv = (cv + c_gx[q][vv]) * ins;
  const double px = fma(fu, sp.X.bx - sp.X.ax, sp.X.ax), py = fma(fu, sp.X.by - sp.X.ay, sp.X.ay);
  const double qx = fma(fv, sp.Y.bx - sp.Y.ax, sp.Y.ax), qy = fma(fv, sp.Y.by - sp.Y.ay, sp.Y.ay);
  const double dx = px - qx, dy = py - qy;
  c = 0.25 * alpha * (dx * dx + dy * dy);
  const double w = c_gw[q][uu] * c_gw[q][vv] * (ins * ins);
  if (KIND == STB_V) {
    wa = sp.sa * w;
    wb = 0.0;
  } else if (KIND == STB_K) {
    wa = sp.sa * w * (dx * sp.Y.nx + dy * sp.Y.ny) * (sp.side == 0 ? fv : 1.0 - fv);
    wb = 0.0;
  } else {
    wa = sp.sa * w;
    wb = sp.sb * w * fma(sp.l1 - sp.l0, fu, sp.l0) * fma(sp.k1 - sp.k0, fv, sp.k0);
  }
}

template <int KIND, bool NEAR, class Vis>
__device__ __forceinline__ void for_points(const MomArgs& M, int I, int J, Vis&& vis) {
  for_subpairs<KIND, NEAR>(M, I, J, [&](const SubPair& sp) {
    for (int cu = 0; cu < sp.ns; ++cu)
      for (int u = 0; u < sp.q; ++u)
        for (int cv = 0; cv < sp.ns; ++cv)
          for (int v = 0; v < sp.q; ++v) {
            double c, wa, wb;
            sub_point<KIND>(sp, M.alpha, cu, u, cv, v, c, wa, wb);
            vis(c, wa, wb);
          }
  });
}

// the points of entry (I, J) dealt round-robin to the 32 lanes of a warp (lane's share only)
template <int KIND, bool NEAR, class Vis>
__device__ __forceinline__ void for_points_lane(const MomArgs& M, int I, int J, int lane, Vis&& vis) {
  int base = 0;
  for_subpairs<KIND, NEAR>(M, I, J, [&](const SubPair& sp) {
    const int nq = sp.q * sp.ns, n = nq * nq;
    for (int idx = (lane - base) & 31; idx < n; idx += 32) {
      double c, wa, wb;
      const int iu = idx / nq, iv = idx % nq;
      sub_point<KIND>(sp, M.alpha, iu / sp.q, iu % sp.q, iv / sp.q, iv % sp.q, c, wa, wb);
      vis(c, wa, wb);
    }
    base = (base + n) & 31;
  });
}

// ------------------------------------------------------------- records
// One entry-level spatial pair (I, J): c range, regime-A moments premultiplied by the polynomial
// coefficients, regime-B shifted moments, and the affine constants
//   C0 = sum W (gamma + ln c), C1 = sum W c (gamma + ln c)  (H);  C0 (F, Q);  C1 = sum W / c (Q)
// WARP = false: one thread per pair.  WARP = true: one warp per pair, its points dealt round-robin
// to the lanes and the partial sums reduced by xor butterflies (every lane ends with the same
// totals; lane 0 writes the record) -- for the pairs with many points (the near records, whose
// orders 10 / 8 / 6 / q_near differ between neighbouring pairs, and D_h's 16 half-segment
// sub-pairs): thread-per-pair left half of each warp idle on the divergent point counts.
template <bool WARP>
__device__ __forceinline__ double rsum(double v) {
  if (WARP) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  return v;
}
template <int KIND, bool NEAR, bool WARP, class Vis>
__device__ __forceinline__ void rec_points(const MomArgs& M, int I, int J, int lane, Vis&& vis) {
  if (WARP) for_points_lane<KIND, NEAR>(M, I, J, lane, vis);
  else for_points<KIND, NEAR>(M, I, J, vis);
}
template <int KIND, bool NEAR, bool WARP>
__device__ __forceinline__ void records_body(const MomArgs& M, long long pair, int lane) {
  const int I = (int)(pair / M.ng), J = (int)(pair % M.ng);
  double* rec = M.rec + rec_base(M, I, J);
  const long long S = M.cs;
  const bool wr = !WARP || lane == 0;   // the lane that writes the record
  // one pass: c range, regime-A moments M_k = sum W c^k and the affine constants of both
  // families (the constants need c > 0 at every point: dropped at the end if one c is 0)
  constexpr int NF = Fams<KIND>::n;
  double mk[NF][MKA + 1], C0[NF], C1[NF];
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    C0[f] = C1[f] = 0.0;
#pragma unroll
    for (int k = 0; k <= MKA; ++k) mk[f][k] = 0.0;
  }
  double cmin = 1e300, cmax = 0.0;
  int npts = 0;
  rec_points<KIND, NEAR, WARP>(M, I, J, lane, [&](double c, double wa, double wb) {
    cmin = fmin(cmin, c);
    cmax = fmax(cmax, c);
    ++npts;
    const bool pos = c > 0.0;
    const double g = pos ? STB_GAMMA + log(c) : 0.0;
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      const int fam = f == 0 ? Fams<KIND>::f0 : Fams<KIND>::f1;
      const double w = f == 0 ? wa : wb;
      // two independent power chains (even / odd orders)
      const double c2 = c * c;
      double pe = w, po = w * c;
#pragma unroll
      for (int k = 0; k <= MKA; k += 2) {
        mk[f][k] += pe;
        if (k + 1 <= MKA) mk[f][k + 1] += po;
        pe *= c2;
        po *= c2;
      }
      if (pos) {
        C0[f] = fma(w, g, C0[f]);
        C1[f] += fam == FAM_Q ? w / c : w * c * g;
      }
    }
  });
  if (WARP) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      cmin = fmin(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
      cmax = fmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
      npts += __shfl_xor_sync(0xffffffffu, npts, o);
    }
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      C0[f] = rsum<WARP>(C0[f]);
      C1[f] = rsum<WARP>(C1[f]);
#pragma unroll
      for (int k = 0; k <= MKA; ++k) mk[f][k] = rsum<WARP>(mk[f][k]);
    }
  }
  if (npts == 0) cmin = 0.0;
  if (!(cmin > 0.0)) {
#pragma unroll
    for (int f = 0; f < NF; ++f) C0[f] = C1[f] = 0.0;
  }
  double c0m = 0.5 * (cmin + cmax);
  bool okB = cmin > 0.0 && (cmax - c0m) <= MRHO * c0m;
  // near records: a cluster too wide for one Taylor centre (c_max > 3 c_min) but within 9 c_min is
  // split at c_s = sqrt(c_min c_max) into two clusters of ratio <= 3 each (regime B2)
  // (only when a near-cell node can fall between regime A and regime Z for this pair)
  const bool two = NEAR && !okB && cmin > 0.0 && cmax <= 8.99 * cmin && cmax * M.u_near[1] >= STB_MXB &&
                   cmin * M.u_near[0] < MXZ;
  const double cs = two ? sqrt(cmin * cmax) : 0.0;
  if (two) {
    c0m = 0.5 * (cmin + cs);
    okB = true;
  }
  const double c0 = okB ? c0m : 0.0;
  const double cup = two ? cs : cmax;                       // upper end of the first cluster
  const double rho = okB ? (cup - c0m) / c0m : 1.0;
  const int kb = (!okB || rho <= 1e-6) ? 3 : min(MKB, max(3, (int)ceil(log(1e-16) / log(rho))));
  const double c0b = two ? 0.5 * (cs + cmax) : 0.0;
  const double rhob = two ? (cmax - c0b) / c0b : 1.0;
  const int kbb = two ? (rhob <= 1e-6 ? 3 : min(MKB, max(3, (int)ceil(log(1e-16) / log(rhob))))) : 0;
  if (NEAR && wr) {
    double* R2 = rec + (long long)rec2_base<KIND>() * S;
    R2[R2_C0 * S] = c0b;
    R2[R2_IC0 * S] = two ? 1.0 / c0b : 0.0;
    R2[R2_KB * S] = (double)kbb;
    R2[R2_CS * S] = cs;
  }
  if (wr) {
    rec[RF_CMAX * S] = cmax;
    rec[RF_CMIN * S] = cmin;
    rec[RF_C0 * S] = c0;
    rec[RF_KB * S] = (double)kb;
    rec[RF_IC0 * S] = okB ? 1.0 / c0 : 0.0;
  }
  // regime-A fields of both families (static indices: the moments stay in registers)
#pragma unroll
  for (int f = 0; f < NF && wr; ++f) {
    const int fam = f == 0 ? Fams<KIND>::f0 : Fams<KIND>::f1;
    double* R = rec + (RF_COMMON + f * FAMSZ) * S;
#pragma unroll
    for (int k = 0; k <= MKA; ++k) R[(FA + k) * S] = mpoly(fam, k) * mk[f][k];
    R[FM0 * S] = mk[f][0];
    R[FM1 * S] = mk[f][1];
    R[FC0 * S] = C0[f];
    R[FC1 * S] = C1[f];
  }
  // one pass per family and cluster (CL: 0 = c <= c_s or the only cluster, 1 = c > c_s)
  auto bpass = [&](const int slot, auto CLc) {
    constexpr int cl = decltype(CLc)::value;
    const int fam = slot == 0 ? Fams<KIND>::f0 : Fams<KIND>::f1;
    // coefficient arrays: FB1 / FB2 of the family (cluster 0) or of the B2 block (cluster 1)
    double* P1 = cl == 0 ? rec + (RF_COMMON + slot * FAMSZ + FB1) * S
                         : rec + (long long)(rec2_base<KIND>() + R2_FAM + slot * R2_FAMSZ) * S;
    double* P2 = cl == 0 ? rec + (RF_COMMON + slot * FAMSZ + FB2) * S : P1 + (long long)(MKB + 1) * S;
    const double cc0 = cl == 0 ? c0 : c0b;
    const int ckb = cl == 0 ? kb : kbb;
    // regime B: m_k = sum W (c - c0)^k over the cluster's points, only the orders the evaluation
    // reads (k <= kb): chunks of 8 with a per-thread exit, four independent power chains
    double mb[MKB + 1];
#pragma unroll
    for (int k = 0; k <= MKB; ++k) mb[k] = 0.0;
    if (okB) {
      rec_points<KIND, NEAR, WARP>(M, I, J, lane, [&](double c, double wa, double wb) {
        if (cl == 1 ? !(c > cs) : (two && c > cs)) return;
        const double w = slot == 0 ? wa : wb;
        const double d = c - cc0, d2 = d * d, d4 = d2 * d2;
        double p0 = w, p1 = w * d, p2 = w * d2, p3 = p1 * d2;
#pragma unroll
        for (int kc = 0; kc <= MKB / 8; ++kc) {
          if (kc * 8 > ckb) break;
#pragma unroll
          for (int j = 0; j < 8; j += 4) {
            const int k = kc * 8 + j;
            if (k <= MKB) mb[k] += p0;
            if (k + 1 <= MKB) mb[k + 1] += p1;
            if (k + 2 <= MKB) mb[k + 2] += p2;
            if (k + 3 <= MKB) mb[k + 3] += p3;
            p0 *= d4;
            p1 *= d4;
            p2 *= d4;
            p3 *= d4;
          }
        }
      });
      if (WARP) {
#pragma unroll
        for (int kc = 0; kc <= MKB / 8; ++kc) {
          if (kc * 8 > ckb) break;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (kc * 8 + j <= MKB) mb[kc * 8 + j] = rsum<WARP>(mb[kc * 8 + j]);
        }
      }
    }
    if (!wr) return;
    // regime-B polynomial coefficients: every Taylor sum of phi_bz is
    // e^{-x0} sum_i coef_i (-u)^i with per-pair coefficients from backward recurrences over the
    // shifted moments (B1_k = m_k / k, B2_k = m_k / ((k-1) k)):
    //   S1:     G_i = (B1_{i+1} - G_{i+1}) / c0,  G_kb = 0,      coef G_i / i!  -> P1[i], i < kb
    //   S2 (H): H_i = (B2_{i+2} - H_{i+1}) / c0,  H_{kb-1} = 0,  coef H_i / i!  -> P2[i], i < kb
    //   S3 (Q): Q_i = (m_i - Q_{i+1}) / c0 (i >= 1), Q_0 = -Q_1 / c0, Q_{kb+1} = 0  -> P2[i], i <= kb
    //   m_0 -> P1[MKB], m_1 -> P2[MKB] (H)
    {
      const double ic0 = okB ? 1.0 / cc0 : 0.0;
      double G = 0.0, H2 = 0.0, Q3 = 0.0;
#pragma unroll
      for (int i = MKB; i >= 0; --i) {
        if (fam == FAM_Q && i <= ckb) {
          Q3 = ((i >= 1 ? mb[i] : 0.0) - Q3) * ic0;
          P2[i * S] = Q3 * STB_INVFACT[i];
        }
        if (i <= ckb - 1) {
          G = (mb[i + 1 <= MKB ? i + 1 : MKB] * STB_INV_H[i + 1 <= MKB ? i + 1 : MKB] - G) * ic0;
          P1[i * S] = G * STB_INVFACT[i];
          if (fam == FAM_H) {
            if (i <= ckb - 2) {
              const int k2 = i + 2 <= MKB ? i + 2 : MKB;
              H2 = (mb[k2] * STB_INV_H[k2 - 1] * STB_INV_H[k2] - H2) * ic0;
            }
            P2[i * S] = i <= ckb - 2 ? H2 * STB_INVFACT[i] : 0.0;
          }
        }
      }
      P1[MKB * S] = mb[0];
      if (fam == FAM_H) P2[MKB * S] = mb[1];
    }
  };
#pragma unroll 1
  for (int slot = 0; slot < NF; ++slot) bpass(slot, std::integral_constant<int, 0>{});
  if (NEAR && two) {
#pragma unroll 1
    for (int slot = 0; slot < NF; ++slot) bpass(slot, std::integral_constant<int, 1>{});
  }
}
// near records: a pair with a touching sub-pair or one closer than near_gap element lengths takes
// sub-pair orders 10 / 8 / 6 next to q_near and skips its touching sub-pairs -- per lane different
// loop nests, which serialise a thread-per-pair warp several times over; such pairs (a band along
// the chain and the corners) go to the warp-per-pair kernel, the others to thread-per-pair
template <int KIND>
__device__ __forceinline__ bool near_special(const MomArgs& M, int I, int J) {
  bool sp = false;
  for_subpairs<KIND, false>(M, I, J, [&](const SubPair& q) {
    sp |= chain_rel(q.pi, q.qi, q.nchain) != 0 || seg_dist(q.X, q.Y) < M.near_gap * fmax(q.X.h, q.Y.h);
  });
  return sp;
}
// SPLIT: D_h near records: the thread kernel appends the near_special pairs to M.list (in any
// order: each pair's record is computed by exactly one warp, so the results do not depend on it)
// and the persistent warp kernel takes them from the list
template <int KIND, bool NEAR, bool SPLIT = false>
__global__ void __launch_bounds__(128) k_records(MomArgs M) {
  const long long pair = M.p_lo + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (pair >= M.p_hi) return;
  if (SPLIT && near_special<KIND>(M, (int)(pair / M.ng), (int)(pair % M.ng))) {
    M.list[1 + atomicAdd(M.list, 1)] = (int)pair;
    return;
  }
  records_body<KIND, NEAR, false>(M, pair, 0);
}
template <int KIND, bool NEAR>
__global__ void __launch_bounds__(128) k_records_warp(MomArgs M) {
  const int nw = (int)((gridDim.x * blockDim.x) >> 5);
  const int n = *(volatile int*)M.list;
  for (int k = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); k < n; k += nw)   // warp-uniform
    records_body<KIND, NEAR, true>(M, M.list[1 + k], threadIdx.x & 31);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------- node evaluation
// regime A from registers.  The s factor of the H family is folded into the Horner chain:
//   s sum_k P_k u^k = s P_0 + sum_{k>=0} P_{k+1} u^k   (u = 1/s),
// so V_h runs one chain of 17 steps and D_h merges its two families into ONE chain over
//   Pc_k = P^H_{k+1} + P^F_k,   Phi~ = s P^H_0 + sum_k Pc_k u^k + ln s (s M0^H + M1^H + M0^F)
// (the same terms re-associated).
template <int KIND>
struct RegA {
  static constexpr int NC = KIND == STB_K ? MKA + 1 : (KIND == STB_V ? MKA : MKA + 1);
  double P[NC];      // the chain's coefficients (highest degree last)
  double e0;         // V, D: s P^H_0 term; K: unused
  double l0, l1;     // V, D: ln s (s l0 + l1);  K: -ln s l0
  double cmax;
  __device__ __forceinline__ void load(const double* __restrict__ rec, long long S) {
    cmax = rec[RF_CMAX * S];
    const double* R0 = rec + (RF_COMMON + 0 * FAMSZ) * S;
    if (KIND == STB_K) {
#pragma unroll
      for (int k = 0; k <= MKA; ++k) P[k] = R0[(FA + k) * S];
      e0 = 0.0;
      l0 = R0[FM0 * S];
      l1 = 0.0;
    } else if (KIND == STB_V) {
#pragma unroll
      for (int k = 0; k < MKA; ++k) P[k] = R0[(FA + k + 1) * S];
      e0 = R0[FA * S];
      l0 = R0[FM0 * S];
      l1 = R0[FM1 * S];
    } else {
      const double* R1 = rec + (RF_COMMON + 1 * FAMSZ) * S;
#pragma unroll
      for (int k = 0; k <= MKA; ++k) P[k] = (k < MKA ? R0[(FA + k + 1) * S] : 0.0) + R1[(FA + k) * S];
      e0 = R0[FA * S];
      l0 = R0[FM0 * S];
      l1 = R0[FM1 * S] + R1[FM0 * S];
    }
  }
  // Phi~ at the node (s, ln s, u = 1/s): the Horner chain in u, then the s / ln s terms (split so
  // that the bulk kernel holds only u of every node in registers during the chains)
  __device__ __forceinline__ double chain(double u) const {
    double acc = P[NC - 1];
#pragma unroll
    for (int k = NC - 2; k >= 0; --k) acc = fma(acc, u, P[k]);
    return acc;
  }
  __device__ __forceinline__ double finish(double acc, double s, double lns) const {
    if (KIND == STB_K) return fma(-lns, l0, acc);
    return fma(s, fma(lns, l0, e0), fma(lns, l1, acc));
  }
  __device__ __forceinline__ double eval(double s, double lns, double u) const { return finish(chain(u), s, lns); }
};
// RegA::chain with the coefficients in shared memory (this thread's column, entry k at sp[k * 128])
template <int KIND>
__device__ __forceinline__ double chain_s(const double* sp, double u) {
  constexpr int NC = RegA<KIND>::NC;
  double acc = sp[(NC - 1) * 128];
#pragma unroll
  for (int k = NC - 2; k >= 0; --k) acc = fma(acc, u, sp[k * 128]);
  return acc;
}

// point-by-point regularised contributions (regime C), same function as regimes A / B / Z
__device__ __forceinline__ double pt_h(double c, double s, double lns, double u) {
  const double x = c * u;
  if (x < STB_XSPLIT) return fma(s, gh_poly(x), (s + c) * lns);
  const double e = x > STB_XUNDER ? 0.0 : exp(-x);
  const double hf = x > STB_XUNDER ? 0.0 : fma(1.0 + x, e1_large(1.0 / x, e), -e);
  return fma(s, hf, (s + c) * (STB_GAMMA + log(c)));
}
__device__ __forceinline__ double pt_f(double c, double lns, double u) {
  const double x = c * u;
  if (x < STB_XSPLIT) return ein_poly(x) + lns;
  const double e1 = x > STB_XUNDER ? 0.0 : e1_large(1.0 / x, exp(-x));
  return e1 + STB_GAMMA + log(c);
}
__device__ __forceinline__ double pt_q(double c, double s, double lns, double u) {
  const double x = c * u;
  if (x < STB_XSPLIT) return psi_poly(x) - lns;
  const double t = 1.0 / x;
  const double e = x > STB_XUNDER ? 0.0 : exp(-x);
  const double k = x > STB_XUNDER ? 0.0 : e * t - e1_large(t, e);
  return k - s / c - (STB_GAMMA + log(c));
}

// the same point contributions without the affine terms (the true node values of the near
// cells): computing them directly avoids subtracting two large affine sums when c >> s
__device__ __forceinline__ double pt_h_true(double c, double s, double lns, double u) {
  const double x = c * u;
  if (x < STB_XSPLIT) return fma(s, gh_poly(x), (s + c) * (lns - STB_GAMMA - log(c)));
  const double e = x > STB_XUNDER ? 0.0 : exp(-x);
  return x > STB_XUNDER ? 0.0 : s * fma(1.0 + x, e1_large(1.0 / x, e), -e);
}
__device__ __forceinline__ double pt_f_true(double c, double lns, double u) {
  const double x = c * u;
  if (x < STB_XSPLIT) return ein_poly(x) + lns - STB_GAMMA - log(c);
  return x > STB_XUNDER ? 0.0 : e1_large(1.0 / x, exp(-x));
}
__device__ __forceinline__ double pt_q_true(double c, double s, double lns, double u) {
  const double x = c * u;
  if (x < STB_XSPLIT) return psi_poly(x) - lns + s / c + STB_GAMMA + log(c);
  const double t = 1.0 / x;
  const double e = x > STB_XUNDER ? 0.0 : exp(-x);
  return x > STB_XUNDER ? 0.0 : e * t - e1_large(t, e);
}

// regimes B and Z (out of line: rare); *regime = 1 (B), 2 (Z) or 3 (C: not evaluated here).
// Regime B in scaled form (x0 = c0 u): e^_j = u^j e_j = e^{-x0} (-u)^j / j!,
// a^_j = u^{j+1} a_j = (e^_j - a^_{j-1}) / c0 (Taylor coefficients a_j of e^{-x}/x at x0), so that
//   F: sum_k c_k u^k m_k = E1 m_0 - S1
//   H: ... = h(x0) m_0 + E1 u m_1 - S1 - u S2
//   Q: ... = -E1 m_0 + (a^_0 m_0 + S3) / u + S1
// with S1 = sum_{k>=1} a^_{k-1} B1[k], S2 = sum_{k>=2} a^_{k-2} B2[k], S3 = sum_{k>=1} a^_k B2[k]
// (B1[k] = m_k / k; H: B2[k] = m_k / ((k-1) k); Q: B2[k] = m_k): two multiplies for e^, one
// add and one multiply for a^, one FMA per family sum.
// per-lane constants of regimes B and Z, loaded once per thread
template <int KIND>
struct RegBZ {
  double c0, ic0, cmin;
  int kb;
  double m0[Fams<KIND>::n], m1, C0[Fams<KIND>::n], C1[Fams<KIND>::n];
  __device__ __forceinline__ void load(const double* __restrict__ rec, long long S) {
    c0 = rec[RF_C0 * S];
    ic0 = rec[RF_IC0 * S];
    cmin = rec[RF_CMIN * S];
    kb = (int)rec[RF_KB * S];
#pragma unroll
    for (int f = 0; f < Fams<KIND>::n; ++f) {
      const double* R = rec + (RF_COMMON + f * FAMSZ) * S;
      m0[f] = R[(FB1 + MKB) * S];
      C0[f] = R[FC0 * S];
      C1[f] = R[FC1 * S];
    }
    m1 = rec[(RF_COMMON + FB2 + MKB) * S];   // H: m_1
  }
};

// the GB3 coefficients as a (non-const) constant-bank array: read as c[bank][offset] operands of
// the Horner DFMAs instead of being materialised as immediates on every regime-B evaluation
static __device__ __constant__ double STB_GB3_CB[STB_GB3_DEG + 1] = STB_GB3_INIT;
__device__ __forceinline__ double gb3_cb(double t) { return horner<STB_GB3_DEG>(STB_GB3_CB, fma(t, STB_GB3_YS, -1.0)); }

// Regime-B coefficient source.  The Taylor sums are Horner chains over per-pair coefficient arrays
// p1 (S1 of the first family), p2 (S2 of H / S3 of Q) and p3 (S1 of the second family), stored
// field-major in the records (stride S).  The bulk kernel stages the first ns coefficients of its
// pair in shared memory once per thread (sm: [chain][i] with stride BZS_STRIDE between entries), so
// that a node's chains read L2 only for orders >= ns: a chain walked through L2 costs one L2 round
// trip per unrolled step, which made a regime-B node ~25x the cost of a regime-A node.
#ifndef STB_BZ_KBS
#define STB_BZ_KBS 12
#endif
constexpr int BZ_KBS = STB_BZ_KBS;  // staged orders per chain (kb <= 11 for ~90% of the C3 / C5 nodes)
constexpr int BZS_STRIDE = 128;     // threads per bulk CTA: entry i of chain f at sm[(f KBS + i) 128]
struct BzSrc {
  const double* p1;
  const double* p2;
  const double* p3;
  long long S;
  const double* sm;   // this thread's staged coefficients (nullptr: none)
  int ns;             // staged entries per chain (orders 0 .. ns-1; p2 also its top entry kb if kb < ns)
};

// h[c][n] = the chain sums of NN nodes (z_n = -u_n), orders kb-1 .. 0 (+ the Q top entry kb)
template <int KIND, int NN>
__device__ __forceinline__ void bz_chains(const BzSrc& src, int kb, const double (&z)[NN],
                                          double (&h1)[NN], double (&h2)[NN], double (&h3)[NN]) {
  constexpr bool C2 = Fams<KIND>::f0 != FAM_F, C3 = Fams<KIND>::n == 2;
  double top = 0.0;
  if (Fams<KIND>::f0 == FAM_Q) top = kb < src.ns ? src.sm[(BZ_KBS + kb) * BZS_STRIDE] : src.p2[(long long)kb * src.S];
#pragma unroll
  for (int n = 0; n < NN; ++n) h1[n] = h3[n] = 0.0, h2[n] = top;
  int i = kb - 1;
  // orders >= ns from the records (coefficient pointers walked down by the record stride)
  if (i >= src.ns) {
    const long long off = (long long)i * src.S;
    const double* q1 = src.p1 + off;
    const double* q2 = src.p2 + off;
    const double* q3 = src.p3 + off;
#pragma unroll 2
    for (; i >= src.ns; --i) {
      const double c1 = *q1;
#pragma unroll
      for (int n = 0; n < NN; ++n) h1[n] = fma(h1[n], z[n], c1);
      if (C2) {
        const double c2 = *q2;
#pragma unroll
        for (int n = 0; n < NN; ++n) h2[n] = fma(h2[n], z[n], c2);
      }
      if (C3) {
        const double c3 = *q3;
#pragma unroll
        for (int n = 0; n < NN; ++n) h3[n] = fma(h3[n], z[n], c3);
      }
      q1 -= src.S;
      q2 -= src.S;
      q3 -= src.S;
    }
  }
  // staged orders from shared memory
  if (i >= 0) {
    const double* r1 = src.sm + i * BZS_STRIDE;
#pragma unroll 4
    for (; i >= 0; --i) {
      const double c1 = r1[0];
#pragma unroll
      for (int n = 0; n < NN; ++n) h1[n] = fma(h1[n], z[n], c1);
      if (C2) {
        const double c2 = r1[BZ_KBS * BZS_STRIDE];
#pragma unroll
        for (int n = 0; n < NN; ++n) h2[n] = fma(h2[n], z[n], c2);
      }
      if (C3) {
        const double c3 = r1[2 * BZ_KBS * BZS_STRIDE];
#pragma unroll
        for (int n = 0; n < NN; ++n) h3[n] = fma(h3[n], z[n], c3);
      }
      r1 -= BZS_STRIDE;
    }
  }
}

// The Taylor sums of one regime-B cluster (centre c0, order kb, coefficient arrays p1 / p2 of the
// first family and p3 of the second, m_0 / m_1 in their last slots): the non-affine node parts
// T[f].  E1(x0) by the GB3 form for x0 >= 8/3 (every single-cluster node: x0 >= x_max / (1 + MRHO)),
// by the general E1 below (the clusters of regime B2 may sit lower).
template <int KIND>
__device__ __forceinline__ void bz_T(const BzSrc& src, double c0, double ic0, int kb, double s, double u,
                                     double (&T)[2]) {
  const double x0 = c0 * u, ex = exp(-x0);
  const double E1 = x0 >= 8.0 / 3.0 ? ex * (ic0 * s) * gb3_cb(ic0 * s) : dev_e1(x0);
  // the Taylor sums as polynomials in z = -u (coefficients from k_records), Horner from the top
  const double z[1] = {-u};
  double h1[1], h2[1], h3[1];
  bz_chains<KIND, 1>(src, kb, z, h1, h2, h3);
  const double S1a = ex * h1[0], S2a = ex * h2[0], S1b = ex * h3[0];
  const double a0 = ex * ic0;
  const double m0 = src.p1[(long long)MKB * src.S];
  // (the Q form divides by u: multiplied by s = 1 / u instead)
  if (Fams<KIND>::f0 == FAM_H) T[0] = fma(fma(1.0 + x0, E1, -ex), m0, fma(E1 * u, src.p2[(long long)MKB * src.S], -fma(u, S2a, S1a)));
  else T[0] = fma(-E1, m0, fma(fma(a0, m0, S2a), s, S1a));
  if (Fams<KIND>::n == 2) T[1] = fma(E1, src.p3[(long long)MKB * src.S], -S1b);
}

// TRUEV: return the true node value (near cells: without the affine terms, which then need not be
// added here and subtracted again by the caller)
template <int KIND, bool TRUEV = false>
__device__ __forceinline__ double phi_bz(const double* __restrict__ rec, long long S, const RegBZ<KIND>& z,
                                         double s, double u, int* regime, const double* sm = nullptr, int ns = 0) {
  const bool zz = z.cmin > 0.0 && z.cmin * u >= MXZ;
  if (!zz && !(z.c0 > 0.0)) {
    *regime = 3;
    return 0.0;
  }
  double T[2] = {0.0, 0.0};
  if (!zz) {
    const double* R0 = rec + (RF_COMMON + 0 * FAMSZ) * S;
    const double* R1 = rec + (RF_COMMON + 1 * FAMSZ) * S;
    bz_T<KIND>(BzSrc{R0 + FB1 * S, R0 + FB2 * S, R1 + FB1 * S, S, sm, ns}, z.c0, z.ic0, z.kb, s, u, T);
  }
  *regime = zz ? 2 : 1;
  double out = 0.0;
#pragma unroll
  for (int f = 0; f < Fams<KIND>::n; ++f) {
    const int fam = f == 0 ? Fams<KIND>::f0 : Fams<KIND>::f1;
    if (TRUEV) out += fam == FAM_H ? s * T[f] : T[f];
    else if (fam == FAM_H) out += fma(s, T[f] + z.C0[f], z.C1[f]);
    else if (fam == FAM_F) out += T[f] + z.C0[f];
    else out += T[f] - fma(s, z.C1[f], z.C0[f]);
  }
  return out;
}

// regime B2 (near records): the two clusters c <= c_s and c > c_s, each with its own centre and
// its own regime Z test; returns the true node value
struct RegB2 {
  double c0, ic0, cs;
  int kb;
  template <int KIND>
  __device__ __forceinline__ void load(const double* __restrict__ rec, long long S) {
    const double* R2 = rec + (long long)rec2_base<KIND>() * S;
    c0 = R2[R2_C0 * S];
    ic0 = R2[R2_IC0 * S];
    kb = (int)R2[R2_KB * S];
    cs = R2[R2_CS * S];
  }
};
template <int KIND>
__device__ __forceinline__ double phi_b2(const double* __restrict__ rec, long long S, const RegBZ<KIND>& z,
                                         const RegB2& z2, double s, double u, int* regime,
                                         const double* sm = nullptr, int ns = 0) {
  const bool zz1 = z.cmin * u >= MXZ, zz2 = z2.cs * u >= MXZ;
  double T[2] = {0.0, 0.0}, T2[2] = {0.0, 0.0};
  if (!zz1) {
    const double* R0 = rec + (RF_COMMON + 0 * FAMSZ) * S;
    const double* R1 = rec + (RF_COMMON + 1 * FAMSZ) * S;
    bz_T<KIND>(BzSrc{R0 + FB1 * S, R0 + FB2 * S, R1 + FB1 * S, S, sm, ns}, z.c0, z.ic0, z.kb, s, u, T);
  }
  if (!zz2) {
    const double* B = rec + (long long)(rec2_base<KIND>() + R2_FAM) * S;
    bz_T<KIND>(BzSrc{B, B + (long long)(MKB + 1) * S, B + (long long)R2_FAMSZ * S, S, nullptr, 0}, z2.c0, z2.ic0,
               z2.kb, s, u, T2);
  }
  *regime = (zz1 && zz2) ? 2 : 1;
  double out = 0.0;
#pragma unroll
  for (int f = 0; f < Fams<KIND>::n; ++f) {
    const int fam = f == 0 ? Fams<KIND>::f0 : Fams<KIND>::f1;
    out += fam == FAM_H ? s * (T[f] + T2[f]) : T[f] + T2[f];
  }
  return out;
}

// two nodes of the same pair at once (the bulk columns usually hold several regime-B nodes per
// lane): the two Taylor recurrences interleave (ILP 2 on a latency-bound chain) and share the
// moment loads.  reg1 / reg2 as in phi_bz.
template <int KIND, bool TRUEV = false>
__device__ __forceinline__ void phi_bz2(const double* __restrict__ rec, long long S, const RegBZ<KIND>& z,
                                        double s1, double u1, double s2, double u2, double& v1,
                                        double& v2, int* reg1, int* reg2, const double* sm = nullptr, int ns = 0) {
  if (!(z.c0 > 0.0)) {   // no cluster: Z or C per node
    v1 = phi_bz<KIND, TRUEV>(rec, S, z, s1, u1, reg1);
    v2 = phi_bz<KIND, TRUEV>(rec, S, z, s2, u2, reg2);
    return;
  }
  const bool zz1 = z.cmin > 0.0 && z.cmin * u1 >= MXZ, zz2 = z.cmin > 0.0 && z.cmin * u2 >= MXZ;
  const double ic0 = z.ic0;
  const double x01 = z.c0 * u1, x02 = z.c0 * u2;
  const double ex1 = exp(-x01), ex2 = exp(-x02);
  const double E11 = ex1 * (ic0 * s1) * gb3_cb(ic0 * s1), E12 = ex2 * (ic0 * s2) * gb3_cb(ic0 * s2);
  const double* R0 = rec + (RF_COMMON + 0 * FAMSZ) * S;
  const double* R1 = rec + (RF_COMMON + 1 * FAMSZ) * S;
  // both nodes' Taylor sums as polynomials in -u (shared coefficient loads, 2 x 1-3 Horner chains)
  const double zz[2] = {-u1, -u2};
  double h1[2], h2[2], h3[2];
  bz_chains<KIND, 2>(BzSrc{R0 + FB1 * S, R0 + FB2 * S, R1 + FB1 * S, S, sm, ns}, z.kb, zz, h1, h2, h3);
  const double S1a1 = ex1 * h1[0], S2a1 = ex1 * h2[0], S1b1 = ex1 * h3[0];
  const double S1a2 = ex2 * h1[1], S2a2 = ex2 * h2[1], S1b2 = ex2 * h3[1];
  const double a01 = ex1 * ic0, a02 = ex2 * ic0;
  const double m0 = z.m0[0];
  double T1[2], T2[2];
  if (Fams<KIND>::f0 == FAM_H) {
    T1[0] = fma(fma(1.0 + x01, E11, -ex1), m0, fma(E11 * u1, z.m1, -fma(u1, S2a1, S1a1)));
    T2[0] = fma(fma(1.0 + x02, E12, -ex2), m0, fma(E12 * u2, z.m1, -fma(u2, S2a2, S1a2)));
  } else {   // the Q form's division by u as a product with s = 1 / u
    T1[0] = fma(-E11, m0, fma(fma(a01, m0, S2a1), s1, S1a1));
    T2[0] = fma(-E12, m0, fma(fma(a02, m0, S2a2), s2, S1a2));
  }
  if (Fams<KIND>::n == 2) {
    T1[1] = fma(E11, z.m0[1], -S1b1);
    T2[1] = fma(E12, z.m0[1], -S1b2);
  }
  v1 = v2 = 0.0;
#pragma unroll
  for (int f = 0; f < Fams<KIND>::n; ++f) {
    const int fam = f == 0 ? Fams<KIND>::f0 : Fams<KIND>::f1;
    const double t1 = zz1 ? 0.0 : T1[f], t2 = zz2 ? 0.0 : T2[f];
    if (TRUEV) {   // the true node value (near cells): no affine terms
      v1 += fam == FAM_H ? s1 * t1 : t1;
      v2 += fam == FAM_H ? s2 * t2 : t2;
    } else if (fam == FAM_H) {
      v1 += fma(s1, t1 + z.C0[f], z.C1[f]);
      v2 += fma(s2, t2 + z.C0[f], z.C1[f]);
    } else if (fam == FAM_F) {
      v1 += t1 + z.C0[f];
      v2 += t2 + z.C0[f];
    } else {
      v1 += t1 - fma(s1, z.C1[f], z.C0[f]);
      v2 += t2 - fma(s2, z.C1[f], z.C0[f]);
    }
  }
  *reg1 = zz1 ? 2 : 1;
  *reg2 = zz2 ? 2 : 1;
}

// regime C, warp-cooperative: every lane evaluates its round-robin share of the points of
// entry (I, J) at node (s, u) (all lanes pass the same arguments); returns the warp sum
// (NEAR: the true node value, without the affine terms)
template <int KIND, bool NEAR>
__device__ __noinline__ double phi_c_warp(const MomArgs M, int I, int J, double s, double lns, double u) {
  const int lane = threadIdx.x & 31;
  double out = 0.0;
  for_points_lane<KIND, NEAR>(M, I, J, lane, [&](double c, double wa, double wb) {
    if (KIND == STB_V) out = fma(wa, NEAR ? pt_h_true(c, s, lns, u) : pt_h(c, s, lns, u), out);
    else if (KIND == STB_K) out = fma(wa, NEAR ? pt_q_true(c, s, lns, u) : pt_q(c, s, lns, u), out);
    else {
      out = fma(wa, NEAR ? pt_h_true(c, s, lns, u) : pt_h(c, s, lns, u), out);
      if (wb != 0.0) out = fma(wb, NEAR ? pt_f_true(c, lns, u) : pt_f(c, lns, u), out);
    }
  });
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) out += __shfl_xor_sync(0xffffffffu, out, o);
  return out;
}

// true node value for the near cells: Phi = Phi~ - affine part
template <int KIND>
__device__ __forceinline__ double affine_part(const double* __restrict__ rec, long long S, double s) {
  double out = 0.0;
#pragma unroll
  for (int f = 0; f < Fams<KIND>::n; ++f) {
    const int fam = f == 0 ? Fams<KIND>::f0 : Fams<KIND>::f1;
    const double* R = rec + (RF_COMMON + f * FAMSZ) * S;
    const double C0 = R[FC0 * S], C1 = R[FC1 * S];
    if (fam == FAM_H) out += fma(s, C0, C1);
    else if (fam == FAM_F) out += C0;
    else out -= fma(s, C1, C0);
  }
  return out;
}

// counter slots (assemble.cu): bulk [0..4], near [5..9], touching records [10..14], and the bulk
// regime-A nodes summed by the K_h g trial-moment table (k_kg_tab; also counted in slot 0)
constexpr int CTR_TAB = 15, CTR_N = 16;
// warp-aggregated regime counters: [A, B, Z, C, sum of the regime-B Taylor orders]
__device__ __forceinline__ void count_regimes(unsigned long long* ctr, unsigned long long nA,
                                              unsigned long long nB, unsigned long long nZ,
                                              unsigned long long nC, unsigned long long nK) {
  if (!ctr) return;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nA += __shfl_xor_sync(0xffffffffu, nA, o);
    nB += __shfl_xor_sync(0xffffffffu, nB, o);
    nZ += __shfl_xor_sync(0xffffffffu, nZ, o);
    nC += __shfl_xor_sync(0xffffffffu, nC, o);
    nK += __shfl_xor_sync(0xffffffffu, nK, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(ctr + 0, nA);
    if (nB) atomicAdd(ctr + 1, nB);
    if (nZ) atomicAdd(ctr + 2, nZ);
    if (nC) atomicAdd(ctr + 3, nC);
    if (nK) atomicAdd(ctr + 4, nK);
  }
}

// ------------------------------------------------------------- bulk cells (d >= 2)
// thread = entry-level pair (I, J): warp = row I, lane = column J (coalesced stores); band of R
// test steps; the thread sweeps the trial nodes y and evaluates the R+1 nodes (x, y) of the band
// once each (1.125 node evaluations per entry at R = 8).  Column fast path: when the node with
// the smallest lag is in regime A for every lane, all R+1 nodes are (s grows with x), and the
// R+1 Horner chains run unrolled and interleaved.
// The lag-table rows of the band's nodes (shared by the whole CTA) are staged in shared memory
// by cp.async in chunks of LAG_CH columns, double-buffered: the chunk after the current one is in
// flight while the current one is evaluated (a global load per column left every column waiting
// on an L2 round trip: a quarter of the kernel's stall samples).
// PROD (product mode, K_h g without storing K_h): each entry is multiplied by g at its trial
// index and summed over the thread's columns; one warp sum per (test row, trial tile) is written
// to the block's partial buffer (fixed slots: deterministic)
constexpr int LAG_CH = 16;
// the temporal blocks one bulk launch covers (all owned blocks of the rank): per block its panel
// offsets, step ranges and (product mode) partial base
struct BulkBlock {
  const long long* poff;
  int a0, a1, b0, b1;
  long long pbase;
};
// one CTA slab of the near cells: test steps [a_beg, a_end) of an owned block (all blocks in one launch)
struct NearItem {
  BulkBlock blk;
  int a_beg, a_end;
};
struct BulkList {
  const BulkBlock* blk;
  int n;
};
// test steps per band: 7 for V_h and K_h g (their 3-CTA register budget: 8 spilled in the B path,
// C5 V 10.1 -> 9.7 ms, K g 16.5 -> 16.0 ms at 7), 8 for D_h (2 CTAs, 11.6 vs 12.1 ms at 7)
#ifndef STB_BULK_R_D
#define STB_BULK_R_D 8      // band height of the D_h bulk kernel
#endif
#ifndef STB_BULK_MINB_D
#define STB_BULK_MINB_D 2   // CTAs per SM the D_h bulk kernel is register-budgeted for
#endif
template <int KIND>
__host__ __device__ constexpr int bulk_r() { return KIND == STB_D ? STB_BULK_R_D : 7; }
template <int KIND>
__host__ __device__ constexpr int bulk_nch() { return Fams<KIND>::n == 2 ? 3 : 2; }
#ifndef STB_BULK_SMP
#define STB_BULK_SMP 1
#endif
// regime-A chain coefficients of the V_h bulk kernel in shared memory (one column per thread, read
// once per Horner step for all R + 1 chains) instead of registers: no spills at 152 registers, C5
// 9.53 -> 9.25 ms; K_h g measured the same (15.19 / 15.24 ms), and at four CTAs per SM (128
// registers, 8 staged regime-B orders) both were slower (V 9.41, K g 16.06 ms)
#ifndef STB_BULK_SMP_D
#define STB_BULK_SMP_D 0
#endif
template <int KIND>
__host__ __device__ constexpr bool bulk_smp() { return (STB_BULK_SMP && KIND == STB_V) || (STB_BULK_SMP_D && KIND == STB_D); }
// dynamic shared memory of k_bulk_m: staged regime-B coefficients + two lag chunks (+ SMP chains)
template <int KIND, int R>
__host__ __device__ constexpr size_t bulk_smem_bytes() {
  return sizeof(double) * bulk_nch<KIND>() * BZ_KBS * BZS_STRIDE + sizeof(double4) * 2 * LAG_CH * (R + 1) +
         (bulk_smp<KIND>() ? sizeof(double) * RegA<KIND>::NC * 128 : 0);
}
__device__ __forceinline__ void cp_async16_bulk(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(sa), "l"(gmem));
}
#ifndef STB_BULK_MINB_K
#define STB_BULK_MINB_K 3   // CTAs per SM the K_h bulk kernels are register-budgeted for
#endif
// MULTI: the blocks of the list L (a rank's owned blocks); otherwise the one block of B (kernel
// parameters: the loop and the list reads compile away -- the list form costs one GPU's single
// block ~7% in spills, C5 V 9.7 vs 10.4 ms)
#ifndef STB_BULK_LEAD
#define STB_BULK_LEAD 1     // per-chunk regime-A prefix instead of a per-column vote
#endif
#ifndef STB_NEAR_TWO
#define STB_NEAR_TWO 1      // k_near_m: the two nodes of a test step evaluated together
#endif
#ifndef STB_BULK_MINB_V
#define STB_BULK_MINB_V 3   // CTAs per SM the V_h bulk kernel is register-budgeted for
#endif
template <int KIND, int R, bool PROD = false, bool MULTI = false>
__global__ void __launch_bounds__(128, KIND == STB_D ? STB_BULK_MINB_D : (KIND == STB_K ? STB_BULK_MINB_K : STB_BULK_MINB_V)) k_bulk_m(BlockArgs B, BulkList L, MomArgs M) {
  const int ng = B.ng;
  const int lane = threadIdx.x & 31;
  const int J0 = blockIdx.x * 32 + lane;
  const int I0 = blockIdx.y * 4 + (threadIdx.x >> 5);
  const bool valid = I0 < ng && J0 < ng;
  const int I = min(I0, ng - 1), J = min(J0, ng - 1);
  // MULTI: grid z = band x nsub, CTA (band, sub) takes the listed blocks sub, sub + nsub, ... (a
  // rank's many small blocks spread over more CTAs: whole waves instead of a few long CTAs)
  const int nsub = MULTI ? B.nsub : 1;
  const int band = blockIdx.z / nsub, ksub = blockIdx.z % nsub;
  // sym: the CTA's 4 rows lie in tile row (4 blockIdx.y) / 32, its 32 columns in tile column
  // blockIdx.x; tiles below the tile diagonal are the mirror images of stored ones
  const int ti = (blockIdx.y * 4) / SYM_TS, tj = blockIdx.x;
  if (B.sym && ti > tj) return;                   // CTA-uniform
  // does band z of any listed block have bulk cells?  (CTA-uniform)
  const int nlist = MULTI ? L.n : 1;
  auto block_k = [&](int k) -> BulkBlock {
    return MULTI ? L.blk[k] : BulkBlock{B.poff, B.a0, B.a1, B.b0, B.b1, B.pbase};
  };
  {
    bool any = false;
    for (int k = ksub; k < nlist && !any; k += nsub) {
      const BulkBlock Q = block_k(k);
      const int rh = Q.a1 - R * band, rl = max(Q.a0, rh - R);
      any = rh > rl && min(Q.b1 - 1, rh - 3) >= Q.b0;
    }
    if (!any) return;
  }
  const long long pair = (long long)I * ng + J;
  const long long S = M.npairs;
  const double* recp = M.rec + pair;               // the pair's record (field stride S)
  // row offsets of the band rows a = r_lo + r for this warp's row I (panel offset + I * ld, or
  // the tile's offset + (I mod 32) * 32), shared by the warp: a store is one LDS + one address add
  __shared__ long long s_row[4][R];
  __shared__ double s_phi[(R + 1) * 128];       // per-thread node values during the fix-ups
  extern __shared__ __align__(16) double bulk_dyn[];
  constexpr int NCH = bulk_nch<KIND>();
  double* s_bz = bulk_dyn;                                                  // [NCH][KBS][128]
  double4* s_lag = reinterpret_cast<double4*>(bulk_dyn + NCH * BZ_KBS * BZS_STRIDE);   // [2][LAG_CH][R+1]
  constexpr bool SMP = bulk_smp<KIND>();
  // SMP: this thread's chain coefficients, entry k at sPt[k * 128]
  double* sPt = reinterpret_cast<double*>(s_lag + 2 * LAG_CH * (R + 1)) + threadIdx.x;
  long long* srow = s_row[threadIdx.x >> 5];
  const long long cstride = B.sym ? B.blk : (long long)ng;   // per trial step b
  const int jcol = B.sym ? J % SYM_TS : J;
  // stores: diagonal tiles of the symmetric packing keep their upper triangle only
  const bool vst = valid && (!B.sym || ti != tj || jcol >= I % SYM_TS);
  RegA<KIND> A;
  A.load(recp, S);
  if (SMP) {
#pragma unroll
    for (int k = 0; k < RegA<KIND>::NC; ++k) sPt[k * 128] = A.P[k];   // read back by this thread only
  }
  // pairs without quadrature points (K_h on collinear elements: the kernel vanishes) hold
  // only zero entries: a warp of them writes zeros (or, in product mode, nothing) and skips the
  // node evaluations, counted as regime A (warp-uniform; the warp still joins the lag staging)
  const bool zero_warp = __all_sync(0xffffffffu, A.cmax == 0.0 && A.P[0] == 0.0 && A.l0 == 0.0);
  RegBZ<KIND> Z;
  Z.load(recp, S);
  // the pair's regime-B Taylor coefficients, orders < BZ_KBS (and K's top entry), staged once in
  // shared memory: this thread's column of s_bz (only this thread reads it, no barrier needed)
  double* sbz = s_bz + threadIdx.x;
  int nsb = 0;
  if (!zero_warp && Z.c0 > 0.0) {
    const double* R0 = recp + (RF_COMMON + 0 * FAMSZ) * S;
    const double* R1 = recp + (RF_COMMON + 1 * FAMSZ) * S;
    nsb = min(Z.kb + 1, BZ_KBS);
    for (int i = 0; i < nsb; ++i) {
      sbz[i * BZS_STRIDE] = R0[(FB1 + i) * S];
      if (Fams<KIND>::f0 != FAM_F) sbz[(BZ_KBS + i) * BZS_STRIDE] = R0[(FB2 + i) * S];
      if (NCH == 3) sbz[(2 * BZ_KBS + i) * BZS_STRIDE] = R1[(FB1 + i) * S];
    }
  }
  unsigned long long nA = 0, nB = 0, nZ = 0, nC = 0, nK = 0, nT = 0;
  // the listed blocks one after the other (a rank's owned blocks of the cyclic plan; one block on one
  // GPU): the per-pair setup above is paid once per CTA, not once per block
  for (int kb_ = ksub; kb_ < nlist; kb_ += nsub) {
  const BulkBlock Bk = block_k(kb_);
  const int r_hi = Bk.a1 - R * band;
  const int r_lo = max(Bk.a0, r_hi - R);
  if (r_hi <= r_lo) continue;                     // CTA-uniform
  const int bmax = min(Bk.b1 - 1, r_hi - 1 - 2);
  if (bmax < Bk.b0) continue;                     // CTA-uniform
  if (MULTI) __syncthreads();                     // the previous block's lag chunks and row offsets are no longer read
  // lag chunk c: columns y = b0 + c LAG_CH + k, nodes x = min(r_lo + r, r_hi) (2 x 16 B per entry)
  const int ncols = bmax + 2 - Bk.b0;
  auto stage = [&](int c) {
    double4* dst = s_lag + (c & 1) * (LAG_CH * (R + 1));
    for (int e = threadIdx.x; e < 2 * LAG_CH * (R + 1); e += blockDim.x) {
      const int ent = e >> 1, k = ent / (R + 1), r = ent % (R + 1);
      const int y = Bk.b0 + c * LAG_CH + k;
      if (c * LAG_CH + k < ncols) {
        const double* src = reinterpret_cast<const double*>(B.lag + (long long)min(r_lo + r, r_hi) * B.ldlag + y);
        cp_async16_bulk(reinterpret_cast<double*>(dst + ent) + 2 * (e & 1), src + 2 * (e & 1));
      }
    }
    asm volatile("cp.async.commit_group;");
  };
  // K_h g with the table: the leading columns whose nodes are all regime A for every lane of the
  // CTA are the table's entirely (A at the band's first node x = r_lo implies A at every node: u
  // falls with x, and rises with y) -- the loop starts at the first chunk holding a column where a
  // lane leaves regime A (binary search along the lag row of x = r_lo, CTA minimum)
  int ystart = Bk.b0;
  if (PROD && B.kgtab) {
    __shared__ int s_ys[4];
    const int yhi = min(bmax + 1, r_lo - 2);          // the table columns are y <= r_lo - 3
    int lo = Bk.b0, hi = max(Bk.b0, yhi);
    if (valid && !zero_warp) {
      const double4* lrow = B.lag + (long long)r_lo * B.ldlag;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (A.cmax * lrow[mid].z < STB_MXB) lo = mid + 1;
        else hi = mid;
      }
    } else {
      lo = max(Bk.b0, yhi);
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    if (lane == 0) s_ys[threadIdx.x >> 5] = lo;
    __syncthreads();
    ystart = min(min(s_ys[0], s_ys[1]), min(s_ys[2], s_ys[3]));
    ystart = Bk.b0 + ((ystart - Bk.b0) / LAG_CH) * LAG_CH;   // a chunk boundary
    const unsigned long long skipped = (unsigned long long)(ystart - Bk.b0) * (r_hi - r_lo + 1);
    nA += skipped;
    nT += skipped;
  }
  stage((ystart - Bk.b0) / LAG_CH);
  if (!PROD && lane < R) {
    const int a = min(r_lo + lane, r_hi - 1);
    srow[lane] = Bk.poff[a - Bk.a0] + (B.sym ? sym_tile_offset(ti, tj, B.nt) + sym_row_base(I % SYM_TS, ti == tj)
                                             : (long long)I * pad4((long long)panel_nb(a, Bk.b0, Bk.b1) * ng));
  }
  __syncwarp();
  double accp[R];
#pragma unroll
  for (int r = 0; r < R; ++r) accp[r] = 0.0;
  double Gp[PROD ? 1 : R];   // stored mode: the previous column's node differences
#pragma unroll
  for (int r = 0; r < (PROD ? 1 : R); ++r) Gp[r] = 0.0;
  double gprev = 0.0;        // product mode: g of the previous trial step (0 before b0)
  bool gp_ok = ystart == Bk.b0;   // gprev holds it (else loaded when the next column is used)
  int ylead = ystart;        // columns y < ylead: regime A at the smallest-lag node for the whole warp
  for (int y = ystart; y <= bmax + 1; ++y) {
    const int kc = y - Bk.b0;
    if (kc % LAG_CH == 0) {                          // CTA-uniform: chunk kc / LAG_CH is needed
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();                               // visible to all; the other buffer is free
      if (kc + LAG_CH < ncols) stage(kc / LAG_CH + 1);
      if (STB_BULK_LEAD) {
        // the chunk's leading columns whose smallest-lag node (x = r_lo) is in regime A for every
        // lane of the warp (u grows with y, so a prefix): one batch of independent shared loads per
        // chunk instead of a load -> compare -> vote chain per column
        const double4* c0p = s_lag + ((kc / LAG_CH) & 1) * (LAG_CH * (R + 1));
        unsigned m = 0;
#pragma unroll
        for (int k = 0; k < LAG_CH; ++k) m |= (unsigned)(A.cmax * c0p[k * (R + 1)].z < STB_MXB) << k;
        ylead = y + __reduce_min_sync(0xffffffffu, (unsigned)(__ffs(~m) - 1));
      }
    }
    const double4* ndc = s_lag + ((kc / LAG_CH) & 1) * (LAG_CH * (R + 1)) + (kc % LAG_CH) * (R + 1);
    // every node of the column by the regime-A form, branch-free (clamped into the lag table,
    // invalid nodes zeroed) so that the R+1 Horner chains interleave; then the nodes of lanes
    // outside regime A are overwritten (B / Z per lane, C warp-cooperatively)
    // only u = 1/s of the column's nodes is held in registers through the Horner chains; s and
    // ln s are read from shared memory again for the closing terms
    const double* ndd = reinterpret_cast<const double*>(ndc);
    double phi[R + 1];
    unsigned bmask = 0;
    // full columns (every band node above the trial node) whose smallest-lag node is in regime A
    // for every lane: all nodes are (s grows with x), no masks or regime tests per node
    const bool full = r_lo > y && r_hi - r_lo == R;       // CTA-uniform
    // K_h g with the trial-moment sums (k_kg_tab): the regime-A nodes (x, y) with y <= x - 3 are
    // summed over the trial index there; a column whose nodes all satisfy y <= x - 3 leaves only
    // this lane's nodes outside regime A (B / Z / C) to evaluate here -- no Horner chains
    const bool tabcol = PROD && B.kgtab && y <= r_lo - 3;  // CTA-uniform
    if (tabcol) {
#pragma unroll
      for (int r = 0; r <= R; ++r) {
        const bool ok = r_lo + r <= r_hi;
        const bool inA = A.cmax * ndd[4 * r + 2] < STB_MXB;
        phi[r] = 0.0;
        nA += ok && inA;
        nT += ok && inA;
        if (ok && !inA && !zero_warp) bmask |= 1u << r;
      }
      if (!__any_sync(0xffffffffu, bmask != 0)) {   // the table's column entirely
        gp_ok = false;
        continue;
      }
    } else if (zero_warp) {
#pragma unroll
      for (int r = 0; r <= R; ++r) {
        phi[r] = 0.0;
        nA += r_lo + r <= r_hi && r_lo + r > y;
      }
    } else if (full && (STB_BULK_LEAD ? y < ylead : __all_sync(0xffffffffu, A.cmax * ndd[2] < STB_MXB))) {
#pragma unroll
      for (int r = 0; r <= R; ++r) phi[r] = SMP ? chain_s<KIND>(sPt, ndd[4 * r + 2]) : A.chain(ndd[4 * r + 2]);
#pragma unroll
      for (int r = 0; r <= R; ++r) phi[r] = A.finish(phi[r], ndd[4 * r], ndd[4 * r + 1]);
      nA += R + 1;
      if (PROD && B.kgtab) {   // nodes y <= x - 3 are the table's (regime A here)
#pragma unroll
        for (int r = 0; r <= R; ++r)
          if (y <= r_lo + r - 3) {
            phi[r] = 0.0;
            ++nT;
          }
      }
    } else {
#pragma unroll
      for (int r = 0; r <= R; ++r) phi[r] = SMP ? chain_s<KIND>(sPt, ndd[4 * r + 2]) : A.chain(ndd[4 * r + 2]);
#pragma unroll
      for (int r = 0; r <= R; ++r) {
        const int x = r_lo + r;
        const double v = A.finish(phi[r], ndd[4 * r], ndd[4 * r + 1]);
        const bool ok = x <= r_hi && x > y;
        const bool inA = A.cmax * ndd[4 * r + 2] < STB_MXB;
        const bool tab = PROD && B.kgtab && inA && y <= x - 3;   // the table's node
        phi[r] = ok && !tab ? v : 0.0;
        nA += ok && inA;
        nT += ok && tab;
        if (ok && !inA) bmask |= 1u << r;
      }
    }
    if (__any_sync(0xffffffffu, bmask != 0)) {
      // the node values pass through shared memory while lanes overwrite their B / Z / C nodes
      // (dynamic node index without register-array selects)
      double* sp = s_phi + threadIdx.x;
#pragma unroll
      for (int r = 0; r <= R; ++r) sp[r * 128] = phi[r];
      unsigned cmask = 0;   // nodes r of this lane left to regime C
      // two nodes per pass (the Taylor chains interleave and share the coefficient loads); an odd
      // last node is evaluated as a pair with itself, so that every lane runs the same code path
      while (bmask) {
        const int r = __ffs(bmask) - 1;
        bmask &= bmask - 1;
        const int r2 = bmask ? __ffs(bmask) - 1 : r;
        bmask &= bmask - 1;
        const double4 q = ndc[r], q2 = ndc[r2];
        int reg = 0, reg2 = 0;
        double v = 0.0, v2 = 0.0;
        phi_bz2<KIND>(recp, S, Z, q.x, q.z, q2.x, q2.z, v, v2, &reg, &reg2, sbz, nsb);
        if (r2 == r) reg2 = 0;
        nB += (reg == 1) + (reg2 == 1);
        nK += (reg == 1 ? Z.kb : 0) + (reg2 == 1 ? Z.kb : 0);
        nZ += (reg == 2) + (reg2 == 2);
        if (reg == 3) {
          cmask |= 1u << r;
          ++nC;
        }
        if (reg2 == 3) {
          cmask |= 1u << r2;
          ++nC;
        }
        sp[r * 128] = v;
        if (r2 != r) sp[r2 * 128] = v2;
      }
      unsigned lanes = __ballot_sync(0xffffffffu, cmask != 0);
      while (lanes) {                                   // warp-uniform
        const int src = __ffs(lanes) - 1;
        lanes &= lanes - 1;
        unsigned cm = __shfl_sync(0xffffffffu, cmask, src);
        const int Is = __shfl_sync(0xffffffffu, I, src), Js = __shfl_sync(0xffffffffu, J, src);
        while (cm) {
          const int r = __ffs(cm) - 1;
          cm &= cm - 1;
          const double4 q = ndc[r];
          const double v = phi_c_warp<KIND, false>(M, Is, Js, q.x, q.y, q.z);
          if (lane == src) sp[r * 128] = v;
        }
      }
#pragma unroll
      for (int r = 0; r <= R; ++r) phi[r] = sp[r * 128];
    }
    if (PROD) {
      // K_h g by summation by parts over the trial steps: with G_y = phi_y[r] - phi_y[r-1] the
      // row's entries are E_b = G_b - G_{b+1}, and sum_b E_b g_b = sum_y G_y (g~_y - g~_{y-1}),
      // g~_y = g_y on the row's bulk columns b0 <= y <= min(bmax, a - 2), 0 elsewhere (the same
      // sum, re-associated: no previous-column G per row is kept)
      const double gv = (valid && y <= bmax) ? B.g[(long long)y * ng + J] : 0.0;
      if (!gp_ok) gprev = (valid && y - 1 >= Bk.b0 && y - 1 <= bmax) ? B.g[(long long)(y - 1) * ng + J] : 0.0;
      if (y <= r_lo - 2 && r_hi - r_lo == R) {      // interior column: g~ = g for every row
        const double dg = gv - gprev;
#pragma unroll
        for (int r = 1; r <= R; ++r) accp[r - 1] = fma(phi[r] - phi[r - 1], dg, accp[r - 1]);
      } else {
#pragma unroll
        for (int r = 1; r <= R; ++r) {
          const int a = r_lo + r - 1;
          const double dg = (y <= a - 2 ? gv : 0.0) - (y - 1 <= a - 2 ? gprev : 0.0);
          if (a < r_hi) accp[r - 1] = fma(phi[r] - phi[r - 1], dg, accp[r - 1]);
        }
      }
      gprev = gv;
      gp_ok = true;
    } else if (y > Bk.b0) {
      const int b = y - 1;
      // interior column: every band row is a full bulk cell (no per-row conditions)
      const bool interior = b <= r_lo - 2 && r_hi - r_lo == R;
      double* col = B.out + ((long long)(b - Bk.b0) * cstride + jcol);
      if (interior && vst) {
#pragma unroll
        for (int r = 1; r <= R; ++r) {
          const double G = phi[r] - phi[r - 1];
          col[srow[r - 1]] = Gp[r - 1] - G;
          Gp[r - 1] = G;
        }
      } else {
#pragma unroll
        for (int r = 1; r <= R; ++r) {
          const int a = r_lo + r - 1;
          const double G = phi[r] - phi[r - 1];
          if (vst && a < r_hi && a - b >= 2) col[srow[r - 1]] = Gp[r - 1] - G;
          Gp[r - 1] = G;
        }
      }
    } else {
#pragma unroll
      for (int r = 1; r <= R; ++r) Gp[r - 1] = phi[r] - phi[r - 1];
    }
  }
  if (PROD) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double sum = warp_sum(accp[r]);
      const int a = r_lo + r;
      if (lane == 0 && a < r_hi && I0 < ng)
        B.part[Bk.pbase + ((long long)(a - Bk.a0) * ng + I) * B.pslots + blockIdx.x] = sum;
    }
  }
  }   // listed blocks
  if (!valid) nA = nB = nZ = nC = nK = nT = 0;
  count_regimes(M.counters, nA, nB, nZ, nC, nK);
  if (PROD && M.counters) {   // regime-A nodes left to the trial-moment table (counted in A above)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nT += __shfl_xor_sync(0xffffffffu, nT, o);
    if (lane == 0 && nT) atomicAdd(M.counters + CTR_TAB, nT);
  }
}

// ------------------------------------------------------------- K_h g: regime-A trial-moment sums
// In the regime-A form a node value of pair (i, n) is linear in the pair's fields,
//   Phi~_n(x, y) = sum_k P_k(i, n) u^k - ln s P_21(i, n)     (RegA<K>: P_k = poly_k M_k, P_21 = M_0),
// so over the pairs n of test segment i that are in regime A at the node (c_max(i, n) u < 8: a
// prefix of the pairs sorted by c_max) the trial sum is one Horner chain on prefix sums:
//   sum_{n in A} Phi~_n(x, y) dg_y(n) = sum_k u^k T_k[m] - ln s T_21[m],
//   T_f[m] = sum_{m' < m} P_f(i, ord[m']) dg_y(ord[m']),   m = #{n : c_max(i, n) u < 8}.
// The same quadrature and regime forms as pair by pair, re-associated over n.
// Covered: the nodes (x, y) with y <= x - 3, b0 <= y <= b1, a0 <= x <= a1 of a listed block, whose
// weight in every row that uses them is dg_y = g~_y - g~_{y-1} (g~ = g on the block's trial steps);
// the per-pair kernel (kgtab) skips exactly these (same predicate on the same lag-table u).  Row a
// receives S(a+1) - S(a), S(x) = sum_y of the node sums, in its own partial slot (2 ntile + 5).
// CTA = (test segment i, listed block), thread = (field f, chunk c of the sorted pairs): warp f,
// lane c -- the 32 chunks of one field per warp, the chunk's fields in registers.  Per trial step
// y: the chunk total, its exclusive prefix over the chunks by a warp shuffle scan,
// the chunk's scan again from that offset into the prefix table; then thread t takes the test
// nodes x = a0 + t (+ KGT_THREADS), whose sums S(x) and cutoffs m stay in registers (m only falls
// as y grows at fixed x: a walk down the sorted c_max instead of a search).  The prefix table and
// the weights are double-buffered, so one barrier per trial step separates the scans of y from
// the node reads of y (and, one step later, from the scans of y + 2 into the same buffer).
// Storage of the pairs in chunks of ch with one padding slot per chunk (stride ch + 1, odd for
// the even chunk lengths): the 32 lanes of a field read and write 32 different banks.
constexpr int KGT_NF = MKA + 2;
constexpr int KGT_CH = 32;
constexpr int KGT_THREADS = KGT_NF * KGT_CH;   // 704
__host__ __device__ inline int kg_ch(int ng) { return (ng + KGT_CH - 1) / KGT_CH; }
__host__ __device__ inline int kg_pch(int ng) { return kg_ch(ng) + 1 - (kg_ch(ng) & 1); }   // odd, > ch - 1
__host__ __device__ inline int kg_ld_t(int ng) { return (KGT_CH * kg_pch(ng) + 1) | 1; }
__host__ __device__ inline size_t kg_tab_smem(int ng, int nxmax) {
  return sizeof(double) * (2 * (size_t)KGT_NF * kg_ld_t(ng) + 2 * ((size_t)KGT_CH * kg_pch(ng) + 40) + (size_t)ng + nxmax) +
         sizeof(int) * (2 * (size_t)ng + 1 + 3 * (size_t)nxmax);
}
constexpr int KGT_NODE = KGT_THREADS / 2;   // threads [0, 352) evaluate the nodes, [352, 704) find their cutoffs
// pairs per chunk the register arrays hold (template instances 12: N_Gamma <= 384, 20: <= 640)
__host__ __device__ inline int kg_chm(int ng) { return kg_ch(ng) <= 12 ? 12 : 20; }
template <int CHM>
__global__ void __launch_bounds__(KGT_THREADS, 1) k_kg_tab(BlockArgs B, BulkList L, MomArgs M, int nxmax,
                                                            const int* __restrict__ gs) {
  extern __shared__ __align__(16) double kgt[];
  const int ng = B.ng, i = blockIdx.x, t = threadIdx.x;
  // CTA = (test segment i, group of listed blocks with one trial range [b0, b1]): the sort, the field
  // loads and the prefix scans of a trial step depend on the trial range only, so the blocks of one
  // trial slice (a rank's owned blocks (I, J) of one J) share them; their test nodes are concatenated
  const int k0 = gs[blockIdx.y], k1 = gs[blockIdx.y + 1];
  const BulkBlock Bk = L.blk[k0];                             // b0, b1 of the group
  int a1max = Bk.a1, nxt = 0;
  for (int k = k0; k < k1; ++k) {
    a1max = max(a1max, L.blk[k].a1);
    nxt += L.blk[k].a1 - L.blk[k].a0 + 1;
  }
  const int ymax = min(Bk.b1, a1max - 3);
  if (ymax < Bk.b0) return;                                   // CTA-uniform: no covered node
  const long long S = M.npairs;
  // ldw: one weight buffer, its last chunk followed by CHM zeros (the scans read CHM entries per chunk)
  const int ch = kg_ch(ng), pch = kg_pch(ng), ldt = kg_ld_t(ng), ldw = KGT_CH * pch + CHM;
  double* T = kgt;                                            // [2][KGT_NF][ldt] prefix sums
  double* w = T + 2 * (size_t)KGT_NF * ldt;                   // [2][ldw] dg_y, padded sorted order
  double* cmx = w + 2 * (size_t)ldw;                          // [ng] sorted c_max
  double* Sx = cmx + ng;                                      // [nx] node sums S(x) (end)
  int* ord = reinterpret_cast<int*>(Sx + nxmax);              // [ng] pair of sorted index m
  int* pos = ord + ng;                                        // [ng + 1] table slot of prefix m
  int* mcut = pos + ng + 1;                                   // [3][nxmax] cutoffs m(x, y), y mod 3
  const double* rec = M.rec + (long long)i * ng;
  auto padm = [&](int m) { return (m / ch) * pch + m % ch; };
  // sort the row's pairs by c_max (rank = #smaller, ties by index): the scratch is T's space
  for (int n = t; n < ng; n += KGT_THREADS) T[n] = rec[RF_CMAX * S + n];
  for (int e = t; e < 2 * ldw; e += KGT_THREADS) w[e] = 0.0;   // padding slots stay 0
  for (int m = t; m <= ng; m += KGT_THREADS) pos[m] = m == 0 ? 0 : 1 + padm(m - 1);
  __syncthreads();
  for (int n = t; n < ng; n += KGT_THREADS) {
    const double c = T[n];
    int rk = 0;
    for (int n2 = 0; n2 < ng; ++n2) {
      const double c2 = T[n2];
      rk += c2 < c || (c2 == c && n2 < n);
    }
    ord[rk] = n;
    cmx[rk] = c;
  }
  __syncthreads();
  // this thread's fields in sorted order (registers)
  const int f = t / KGT_CH, c = t % KGT_CH;
  const int m0 = min(ng, c * ch), nm = min(ng, m0 + ch) - m0;
  const double* Rf = rec + (long long)(RF_COMMON + (f < MKA + 1 ? FA + f : FM0)) * S;
  double cs[CHM];
#pragma unroll
  for (int j = 0; j < CHM; ++j) cs[j] = j < nm ? Rf[ord[m0 + j]] : 0.0;
  if (c == 0) T[(size_t)f * ldt] = T[((size_t)KGT_NF + f) * ldt] = 0.0;   // prefix m = 0
  auto gt = [&](int yy, int n) -> double {   // g~ on the block's trial steps
    return (yy >= Bk.b0 && yy < Bk.b1) ? B.g[(long long)yy * ng + n] : 0.0;
  };
  // node x = a0 + t (threads t < KGT_NODE: its sum S(x)); cutoff thread t' = t - KGT_NODE finds
  // m(x', y + 1) for node x' = a0 + t' during step y (galloping down from m(x', y): the cutoff only
  // falls as y grows), triple-buffered by y mod 3 so that one barrier per step orders it
  const bool nodet = t < KGT_NODE;
  const int jn = nodet ? t : t - KGT_NODE;                    // this thread's node in the group
  int xk = 0, xa1 = -1;                                       // its test node x and its block's a1
  {
    int cum = 0;
    for (int k = k0; k < k1; ++k) {
      const int nx = L.blk[k].a1 - L.blk[k].a0 + 1;
      if (jn >= cum && jn < cum + nx) {
        xk = L.blk[k].a0 + jn - cum;
        xa1 = L.blk[k].a1;
      }
      cum += nx;
    }
  }
  const int nxk = nxt;
  double sx = 0.0;
  int mprev = ng;
  auto cutoff = [&](double u, int H) {          // #{m : c_max[m] u < 8} given it is <= H
    int L = -1, step = 1;
    while (true) {
      const int k = H - step;
      if (k < 0) break;
      if (cmx[k] * u < STB_MXB) { L = k; break; }
      H = k;
      step <<= 1;
    }
    while (H - L > 1) {
      const int mid = (L + H) >> 1;
      if (cmx[mid] * u < STB_MXB) L = mid;
      else H = mid;
    }
    return H;
  };
  const int wslot = padm(min(ng - 1, t));
  const int nt_ = t < ng ? ord[t] : 0;
  for (int m = t; m < ng; m += KGT_THREADS) w[padm(m)] = gt(Bk.b0, ord[m]) - gt(Bk.b0 - 1, ord[m]);
  // global loads one trial step ahead (L2 latency off the step's critical path): the lag entry
  // (u, ln s) of this thread's node (node threads: step y + 1; cutoff threads: step y + 2) and g
  // of the weights stored during the step
  auto ldq = [&](int yy) -> double2 {
    if (yy > ymax || xk > xa1 || xk < yy + 3) return make_double2(0.0, 0.0);
    const double4 q = B.lag[(long long)xk * B.ldlag + yy];
    return make_double2(q.z, q.y);
  };
  if (!nodet && xk <= xa1 && xk >= Bk.b0 + 3) {            // cutoff of step b0
    mprev = cutoff(ldq(Bk.b0).x, ng);
    mcut[jn] = mprev;
  }
  double2 qc = ldq(nodet ? Bk.b0 : Bk.b0 + 1);
  double ga = (t < ng && Bk.b0 < ymax) ? gt(Bk.b0 + 1, nt_) : 0.0;   // weights of step b0 + 1
  double gb = (t < ng && Bk.b0 < ymax) ? gt(Bk.b0, nt_) : 0.0;
  __syncthreads();
  for (int y = Bk.b0; y <= ymax; ++y) {
    const int par = (y - Bk.b0) & 1;
    const double* wy = w + (size_t)par * ldw + c * pch;
    double* wn = w + (size_t)(par ^ 1) * ldw;
    double* Ty = T + (size_t)par * KGT_NF * ldt;
    const double2 qn = ldq(nodet ? y + 1 : y + 2);
    const double gan = (t < ng && y + 1 < ymax) ? gt(y + 2, nt_) : 0.0;
    const double gbn = (t < ng && y + 1 < ymax) ? gt(y + 1, nt_) : 0.0;
    // prefix sums of the 22 fields weighted by dg_y: the chunk total, its exclusive prefix over the
    // field's 32 chunks (the lanes of its warp), the chunk's scan again from there
    double tot = 0.0;
#pragma unroll
    for (int j = 0; j < CHM; ++j) tot = fma(cs[j], wy[j], tot);   // (past the chunk: cs = 0, wy finite)
    // (exclusive scan of the totals shifted by one lane: inc - tot would cancel the small prefix
    // against the large totals of the last chunks, whose c_max^k moments dominate the high fields)
    double run = __shfl_up_sync(0xffffffffu, tot, 1);
    if (c == 0) run = 0.0;
#pragma unroll
    for (int d = 1; d < KGT_CH; d <<= 1) {
      const double v = __shfl_up_sync(0xffffffffu, run, d);
      if (c >= d) run += v;
    }
    double* Tc = Ty + (size_t)f * ldt + 1 + c * pch;
    if (nm == CHM) {   // full chunks (every chunk when CHM = ch and 32 | N_Gamma): no store predicates
#pragma unroll
      for (int j = 0; j < CHM; ++j) {
        run = fma(cs[j], wy[j], run);
        Tc[j] = run;
      }
    } else {
#pragma unroll
      for (int j = 0; j < CHM; ++j) {
        run = fma(cs[j], wy[j], run);
        if (j < nm) Tc[j] = run;
      }
    }
    if (t < ng && y < ymax) wn[wslot] = ga - gb;
    // cutoff threads: m(x', y + 1) into buffer (y + 1) mod 3
    if (!nodet && xk <= xa1 && xk >= y + 4 && y < ymax) {
      mprev = cutoff(qc.x, mprev);
      mcut[((y + 1 - Bk.b0) % 3) * nxk + jn] = mprev;
    }
    __syncthreads();
    // the covered node of trial step y (lag table: s, ln s, u)
    if (nodet && xk <= xa1 && xk >= y + 3) {
      const double u = qc.x;
      const double* Tm = Ty + pos[mcut[((y - Bk.b0) % 3) * nxk + jn]];
      double acc = Tm[(size_t)MKA * ldt];
#pragma unroll
      for (int kk = MKA - 1; kk >= 0; --kk) acc = fma(acc, u, Tm[(size_t)kk * ldt]);
      sx += fma(-qc.y, Tm[(size_t)(MKA + 1) * ldt], acc);
    }
    qc = qn;
    ga = gan;
    gb = gbn;
  }
  if (nodet && xk <= xa1) Sx[jn] = sx;
  __syncthreads();
  for (int k = k0, cum = 0; k < k1; ++k) {
    const BulkBlock Q = L.blk[k];
    for (int a = Q.a0 + t; a < Q.a1; a += KGT_THREADS)
      B.part[Q.pbase + ((long long)(a - Q.a0) * ng + i) * B.pslots + 2 * B.ntile + 5] = Sx[cum + a + 1 - Q.a0] - Sx[cum + a - Q.a0];
    cum += Q.a1 - Q.a0 + 1;
  }
}

// ------------------------------------------------------------- near cells (d <= 1)
// thread = entry-level pair; it walks the test steps a of its chunk: entry (a, a) = Phi(a+1, a),
// entry (a, a-1) = Phi(a+1, a-1) - Phi(a, a-1) - Phi(a+1, a) (Phi(a, a) = 0: G vanishes at s = 0),
// with the true node values Phi = Phi~ - affine part (the affine terms do not cancel here).
// Touching sub-pairs are excluded from the near records; k_sing adds them afterwards.
template <int KIND, bool PROD = false>
__global__ void __launch_bounds__(128) k_near_m(BlockArgs B0, MomArgs M, int chunk, const NearItem* __restrict__ items) {
  // items: grid z enumerates (owned block, chunk of its test steps) of every block with near cells
  // (one launch for a rank's blocks); nullptr: the one block of B0, chunk z
  BlockArgs B = B0;
  int a_beg, a_end;
  if (items) {
    const NearItem it = items[blockIdx.z];
    B.poff = it.blk.poff;
    B.a0 = it.blk.a0;
    B.a1 = it.blk.a1;
    B.b0 = it.blk.b0;
    B.b1 = it.blk.b1;
    B.pbase = it.blk.pbase;
    a_beg = it.a_beg;
    a_end = it.a_end;
  } else {
    a_beg = B.a0 + blockIdx.z * chunk;
    a_end = min(B.a1, a_beg + chunk);
  }
  const int ng = B.ng;
  const int lane = threadIdx.x & 31;
  const int J0 = blockIdx.x * 32 + lane;
  const int I0 = blockIdx.y * 4 + (threadIdx.x >> 5);
  const bool valid = I0 < ng && J0 < ng;
  const int I = min(I0, ng - 1), J = min(J0, ng - 1);
  if (B.sym && (int)(blockIdx.y * 4) / SYM_TS > (int)blockIdx.x) return;   // CTA-uniform (mirror tiles)
  const long long pair = (long long)I * ng + J;
  const long long S = M.npairs;
  const double* rec = M.rec + pair;
  RegA<KIND> A;
  A.load(rec, S);
  RegBZ<KIND> Z;
  Z.load(rec, S);
  RegB2 Z2;
  Z2.load<KIND>(rec, S);
  // D_h: the first cluster's regime-B Taylor coefficients staged in shared memory as in k_bulk_m
  // (about half of its near-cell nodes are in regime B, three chains each walked through L2: C5
  // 1.70 -> 1.58 ms); V_h and K_h measured faster without (the 24 KB cost them occupancy)
  constexpr bool STAGE = KIND == STB_D;
  constexpr int NCH = bulk_nch<KIND>();
  __shared__ double s_bzn[STAGE ? NCH * BZ_KBS * BZS_STRIDE : 1];
  double* sbz = s_bzn + (STAGE ? threadIdx.x : 0);
  int nsb = 0;
  if (STAGE && Z.c0 > 0.0) {
    const double* R0 = rec + (RF_COMMON + 0 * FAMSZ) * S;
    const double* R1 = rec + (RF_COMMON + 1 * FAMSZ) * S;
    nsb = min(Z.kb + 1, BZ_KBS);
    for (int i = 0; i < nsb; ++i) {
      sbz[i * BZS_STRIDE] = R0[(FB1 + i) * S];
      if (Fams<KIND>::f0 != FAM_F) sbz[(BZ_KBS + i) * BZS_STRIDE] = R0[(FB2 + i) * S];
      if (NCH == 3) sbz[(2 * BZ_KBS + i) * BZS_STRIDE] = R1[(FB1 + i) * S];
    }
  }
  unsigned long long nA = 0, nB = 0, nZ = 0, nC = 0, nK = 0;
  // node value without regime C (per lane): inA -> the regularised regime-A value, else the true
  // value of regimes B / B2 / Z; needC -> regime C, left to the warp-cooperative pass
  auto node_nc = [&](const double4& nd, bool& inA, bool& needC) -> double {
    needC = false;
    inA = A.cmax * nd.z < STB_MXB;
    if (inA) {
      ++nA;
      return A.eval(nd.x, nd.y, nd.z);
    }
    int reg = 0;
    const double v = Z2.kb > 0 ? phi_b2<KIND>(rec, S, Z, Z2, nd.x, nd.z, &reg, STAGE ? sbz : nullptr, STAGE ? nsb : 0)
                               : phi_bz<KIND, true>(rec, S, Z, nd.x, nd.z, &reg, STAGE ? sbz : nullptr, STAGE ? nsb : 0);
    nB += reg == 1;
    nK += reg == 1 ? Z.kb + Z2.kb : 0;
    nZ += reg == 2;
    if (reg == 3) {
      needC = true;
      ++nC;
    }
    return v;
  };
  // regime C of the lanes that need it at node nd (warp-uniform call)
  auto pass_c = [&](const double4& nd, bool needC, double& v) {
    unsigned lanes = __ballot_sync(0xffffffffu, needC);
    while (lanes) {
      const int src = __ffs(lanes) - 1;
      lanes &= lanes - 1;
      const int Is = __shfl_sync(0xffffffffu, I, src), Js = __shfl_sync(0xffffffffu, J, src);
      const double c = phi_c_warp<KIND, true>(M, Is, Js, nd.x, nd.y, nd.z);
      if (lane == src) v = c;
    }
  };
  // node value for every lane (warp-uniform call: regime C is computed cooperatively)
  auto node = [&](int x, int y) -> double {
    const double4 nd = B.lag[x * B.ldlag + y];
    bool inA, needC;
    double v = node_nc(nd, inA, needC);
    pass_c(nd, needC, v);
    // regime A gives the regularised value; B, Z and C return the true value directly
    return inA ? v - affine_part<KIND>(rec, S, nd.x) : v;
  };
  // two nodes of the same pair at once (Phi(a+1, a) and Phi(a+1, a-1)), warp-uniform call: both
  // regime-A chains in one block, or both single-cluster regime-B Taylor sums interleaved by
  // phi_bz2 (ILP 2, shared coefficient loads); per lane, the C pass after it for the whole warp
  auto node2 = [&](int x1, int y1, int x2, int y2, double& o1, double& o2) {
    if (!STB_NEAR_TWO) {
      o1 = node(x1, y1);
      o2 = node(x2, y2);
      return;
    }
    const double4 n1 = B.lag[x1 * B.ldlag + y1], n2 = B.lag[x2 * B.ldlag + y2];
    const bool a1 = A.cmax * n1.z < STB_MXB, a2 = A.cmax * n2.z < STB_MXB;
    double v1 = 0.0, v2 = 0.0;
    bool i1 = a1, i2 = a2, c1 = false, c2 = false;
    if (a1 && a2) {
      v1 = A.eval(n1.x, n1.y, n1.z);
      v2 = A.eval(n2.x, n2.y, n2.z);
      nA += 2;
    } else if (!a1 && !a2 && Z2.kb == 0) {
      int r1 = 0, r2 = 0;
      phi_bz2<KIND, true>(rec, S, Z, n1.x, n1.z, n2.x, n2.z, v1, v2, &r1, &r2, STAGE ? sbz : nullptr,
                          STAGE ? nsb : 0);
      nB += (r1 == 1) + (r2 == 1);
      nK += (r1 == 1 ? Z.kb : 0) + (r2 == 1 ? Z.kb : 0);
      nZ += (r1 == 2) + (r2 == 2);
      c1 = r1 == 3;
      c2 = r2 == 3;
      nC += c1 + c2;
    } else {
      v1 = node_nc(n1, i1, c1);
      v2 = node_nc(n2, i2, c2);
    }
    pass_c(n1, c1, v1);
    pass_c(n2, c2, v2);
    o1 = i1 ? v1 - affine_part<KIND>(rec, S, n1.x) : v1;
    o2 = i2 ? v2 - affine_part<KIND>(rec, S, n2.x) : v2;
  };
  double prev = 0.0;  // Phi(a, a-1)
  if (a_beg < a_end && a_beg >= 1 && a_beg - 1 >= B.b0 && a_beg - 1 < B.b1) prev = node(a_beg, a_beg - 1);
#pragma unroll 1
  for (int a = a_beg; a < a_end; ++a) {
    const bool d0 = a >= B.b0 && a < B.b1, d1 = a - 1 >= B.b0 && a - 1 < B.b1;
    double p10 = 0.0, p20 = 0.0;
    if (d1) node2(a + 1, a, a + 1, a - 1, p10, p20);   // CTA-uniform conditions
    else if (d0) p10 = node(a + 1, a);
    if (PROD) {
      double c = 0.0;
      if (d0 && valid) c = p10 * B.g[(long long)a * ng + J];
      if (d1) {
        if (valid) c = fma(p20 - prev - p10, B.g[(long long)(a - 1) * ng + J], c);
      }
      c = warp_sum(c);
      if (lane == 0 && (d0 || d1) && I0 < ng)
        B.part[B.pbase + ((long long)(a - B.a0) * ng + I) * B.pslots + B.ntile + blockIdx.x] = c;
    } else {
      const bool vst = valid && (!B.sym || sym_stored(I, J));
      if (d0 && vst) *entry_ptr(B, a, I, a, J) = p10;
      if (d1 && vst) *entry_ptr(B, a, I, a - 1, J) = p20 - prev - p10;
    }
    prev = p10;
  }
  if (!valid) nA = nB = nZ = nC = nK = 0;
  count_regimes(M.counters, nA, nB, nZ, nC, nK);
}

// ------------------------------------------------------------- touching sub-pairs (d <= 1)
// The touching (identical or vertex-sharing) sub-pairs of entry (I, J) with the singular rules
// of order n: identical elements by the 1-D reduction
// int int f(|x - y|) = int_0^h f(w) G(w) dw, vertex pairs by the Duffy map at the shared vertex,
// the logarithm split as ln c = lnA + 2 ln rho with the ln rho part on log-weighted Gauss rules:
//   int W F(c)       = sum wa F(c)
//   int W F(c) ln c  = sum [wa lnA + 2 wla] F(c)
// vis(c, lnA, wa, wb, wla, wlb) for the two families (weights include the kernel prefactors).
__device__ __forceinline__ double lin1(double v0, double v1, double f) { return fma(v1 - v0, f, v0); }

template <int KIND, class Vis>
__device__ __forceinline__ void for_touch_points(const MomArgs& M, int I, int J, int n, int lane, int nl,
                                                 Vis&& vis) {
  const double alpha = M.alpha;
  for_subpairs<KIND, false>(M, I, J, [&](const SubPair& sp) {
    const int rel = chain_rel(sp.pi, sp.qi, sp.nchain);
    if (!rel) return;
    const Seg &X = sp.X, &Y = sp.Y;
    const double hh = X.h * Y.h;
    const double wsa = sp.sa / hh, wsb = sp.sb / hh;
    // shapes on X and Y of family a (K: the primal hat on Y) and family b (D normal: psi_l, psi_k)
    const double ax0 = 1.0, ax1 = 1.0;
    const double ay0 = KIND == STB_K ? (sp.side == 0 ? 0.0 : 1.0) : 1.0;
    const double ay1 = KIND == STB_K ? (sp.side == 0 ? 1.0 : 0.0) : 1.0;
    const double bx0 = sp.l0, bx1 = sp.l1, by0 = sp.k0, by1 = sp.k1;
    if (rel == 1) {
      if (KIND == STB_K) return;  // dot = 0 on a straight element
      const double h = X.h;
      const double L0 = log(0.25 * alpha) + 2.0 * log(h);
      for (int k = lane; k < n; k += nl) {
        const double rho = c_gx[n][k], w = h * rho, len = h - w;
        // G(w) = int_0^{h-w} [Sx(v+w) Sy(v) + Sx(v) Sy(v+w)] dv (quadratic: 2-point Gauss exact)
        double Ga = 0.0, Gb = 0.0;
        for (int r = 0; r < 2; ++r) {
          const double v = len * c_gx[2][r];
          Ga += c_gw[2][r] * (lin1(ax0, ax1, (v + w) / h) * lin1(ay0, ay1, v / h) +
                              lin1(ax0, ax1, v / h) * lin1(ay0, ay1, (v + w) / h));
          if (KIND == STB_D)
            Gb += c_gw[2][r] * (lin1(bx0, bx1, (v + w) / h) * lin1(by0, by1, v / h) +
                                lin1(bx0, bx1, v / h) * lin1(by0, by1, (v + w) / h));
        }
        Ga *= len * h * wsa;
        Gb *= len * h * wsb;
        vis(0.25 * alpha * w * w, L0, Ga * c_gw[n][k], Gb * c_gw[n][k], Ga * c_glw[n][k], Gb * c_glw[n][k]);
      }
    } else {
      const double h1 = X.h, h2 = Y.h;
      double e1x, e1y, e2x, e2y;
      double axV, axF, ayV, ayF, bxV, bxF, byV, byF;
      if (rel == 2) {   // X.end == Y.start
        e1x = -X.tx; e1y = -X.ty; e2x = Y.tx; e2y = Y.ty;
        axV = ax1; axF = ax0; ayV = ay0; ayF = ay1;
        bxV = bx1; bxF = bx0; byV = by0; byF = by1;
      } else {          // X.start == Y.end
        e1x = X.tx; e1y = X.ty; e2x = -Y.tx; e2y = -Y.ty;
        axV = ax0; axF = ax1; ayV = ay1; ayF = ay0;
        bxV = bx0; bxF = bx1; byV = by1; byF = by0;
      }
      const double cth = e1x * e2x + e1y * e2y;
      const double e1n = e1x * Y.nx + e1y * Y.ny;
      const int ne = acute_cells(cth);                  // eta cells (reading R25)
      const double ine = 1.0 / ne;
      for (int idx = lane; idx < 2 * ne * n * n; idx += nl) {
            const int tri = idx / (ne * n * n), ie = (idx / n) % (ne * n), ir = idx % n;
            const double eta = (ie / n + c_gx[n][ie % n]) * ine, rho = c_gx[n][ir];
            const double A = tri == 0 ? (h1 * h1 + h2 * h2 * eta * eta - 2.0 * h1 * h2 * eta * cth)
                                      : (h1 * h1 * eta * eta + h2 * h2 - 2.0 * h1 * h2 * eta * cth);
            const double u = tri == 0 ? h1 * rho : h1 * rho * eta;
            const double v = tri == 0 ? h2 * rho * eta : h2 * rho;
            const double jac = h1 * h2 * rho;
            double fa = lin1(axV, axF, u / h1) * lin1(ayV, ayF, v / h2) * jac * wsa;
            if (KIND == STB_K) fa *= u * e1n;   // (x - y).n_y = u e1.n_y at the shared vertex
            const double fb = KIND == STB_D ? lin1(bxV, bxF, u / h1) * lin1(byV, byF, v / h2) * jac * wsb : 0.0;
            const double we = c_gw[n][ie % n] * ine;
            const double wr = we * c_gw[n][ir], wl = we * c_glw[n][ir];
            vis(0.25 * alpha * rho * rho * A, log(0.25 * alpha * A), fa * wr, fb * wr, fa * wl, fb * wl);
          }
    }
  });
}

// sing records: entry-level pairs (I, J = I + jo - 2), jo = 0..4, with touching sub-pairs; the
// touching parts only, regime-A data and the affine constants (same layout as the pair records)
template <int KIND>
__global__ void __launch_bounds__(128) k_sing_records(MomArgs M, int nsing) {
  const long long rid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;   // warp per record
  if (rid >= M.npairs) return;                    // warp-uniform
  const int lane = threadIdx.x & 31;
  const int I = (int)(rid / 5), jo = (int)(rid % 5);
  const int J = (I + jo - 2 + M.ng) % M.ng;
  double* rec = M.rec + rid;
  const long long S = M.npairs;
  double cmax = 0.0;
  for_touch_points<KIND>(M, I, J, nsing, lane, 32, [&](double c, double, double, double, double, double) {
    cmax = fmax(cmax, c);
  });
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cmax = fmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
  if (lane == 0) {
    rec[RF_CMAX * S] = cmax;
    rec[RF_CMIN * S] = 0.0;
    rec[RF_C0 * S] = 0.0;
    rec[RF_KB * S] = 0.0;
    rec[RF_IC0 * S] = 0.0;
  }
#pragma unroll 1
  for (int slot = 0; slot < Fams<KIND>::n; ++slot) {
    const int fam = slot == 0 ? Fams<KIND>::f0 : Fams<KIND>::f1;
    double* R = rec + (RF_COMMON + slot * FAMSZ) * S;
    double mk[MKA + 1];
#pragma unroll
    for (int k = 0; k <= MKA; ++k) mk[k] = 0.0;
    double C0 = 0.0, C1 = 0.0;
    for_touch_points<KIND>(M, I, J, nsing, lane, 32, [&](double c, double lnA, double wa, double wb, double wla, double wlb) {
      const double w = slot == 0 ? wa : wb, wl = slot == 0 ? wla : wlb;
      double pw = w;
#pragma unroll
      for (int k = 0; k <= MKA; ++k) {
        mk[k] += pw;
        pw *= c;
      }
      // int W (gamma + ln c) and int W c (gamma + ln c); Q: int W / c (regular after Duffy)
      const double wlog = fma(w, STB_GAMMA + lnA, 2.0 * wl);
      C0 += wlog;
      C1 += fam == FAM_Q ? w / c : wlog * c;
    });
#pragma unroll
    for (int k = 0; k <= MKA; ++k) mk[k] = warp_sum(mk[k]);
    C0 = warp_sum(C0);
    C1 = warp_sum(C1);
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k <= MKA; ++k) R[(FA + k) * S] = mpoly(fam, k) * mk[k];
      R[FM0 * S] = mk[0];
      R[FM1 * S] = mk[1];
#pragma unroll
      for (int k = 0; k <= MKB; ++k) R[(FB1 + k) * S] = R[(FB2 + k) * S] = 0.0;
      R[FC0 * S] = C0;
      R[FC1 * S] = C1;
    }
  }
}

// touching contributions to the near cells, added onto the near-kernel values: thread = (sing
// record, chunk of test steps); regime A only (the host checks c_max / min lag < 4 before it
// chooses this path; a violation is counted in counters[3] and fails the assembly)
template <int KIND, bool PROD = false>
__global__ void __launch_bounds__(128) k_sing_m(BlockArgs B, MomArgs M, int chunk) {
  const long long rid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (rid >= M.npairs) return;
  const int I = (int)(rid / 5), jo = (int)(rid % 5);
  if ((KIND == STB_V && (jo == 0 || jo == 4)) || (KIND == STB_K && jo == 0)) return;
  const int J = (I + jo - 2 + M.ng) % M.ng;
  if (B.sym && !sym_stored(I, J)) return;   // mirror of the stored entry (J, I)
  const int a_beg = B.a0 + blockIdx.y * chunk;
  const int a_end = min(B.a1, a_beg + chunk);
  const long long S = M.npairs;
  const double* rec = M.rec + rid;
  RegA<KIND> A;
  A.load(rec, S);
  unsigned long long bad = 0;
  auto node = [&](int x, int y) -> double {
    const double4 nd = B.lag[x * B.ldlag + y];
    bad += !(A.cmax * nd.z < STB_MXA);
    return A.eval(nd.x, nd.y, nd.z) - affine_part<KIND>(rec, S, nd.x);
  };
  double prev = 0.0;
  if (a_beg < a_end && a_beg >= 1 && a_beg - 1 >= B.b0 && a_beg - 1 < B.b1) prev = node(a_beg, a_beg - 1);
#pragma unroll 1
  for (int a = a_beg; a < a_end; ++a) {
    const bool d0 = a >= B.b0 && a < B.b1, d1 = a - 1 >= B.b0 && a - 1 < B.b1;
    double p10 = 0.0;
    if (d0 || d1) p10 = node(a + 1, a);
    if (PROD) {
      double c = 0.0;
      if (d0) c = p10 * B.g[(long long)a * M.ng + J];
      if (d1) c = fma(node(a + 1, a - 1) - prev - p10, B.g[(long long)(a - 1) * M.ng + J], c);
      if (d0 || d1) B.part[B.pbase + ((long long)(a - B.a0) * M.ng + I) * B.pslots + 2 * B.ntile + jo] = c;
    } else {
      if (d0) *entry_ptr(B, a, I, a, J) += p10;
      if (d1) *entry_ptr(B, a, I, a - 1, J) += node(a + 1, a - 1) - prev - p10;
    }
    prev = p10;
  }
  if (bad && M.counters) atomicAdd(M.counters + 3, bad);   // regime C slot of the sing counters
}

}  // namespace stb
