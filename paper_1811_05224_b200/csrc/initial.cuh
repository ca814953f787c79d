// initial.cuh — the initial potential term M_h^0 u0 of eq. (4),
// included by assemble.cu (Gauss tables in its __constant__ memory).  For the test function
// phi^0_(a,i) and u0_h in S_h^1(Omega_h):
//   f[(a,i)] = int_{t_a}^{t_{a+1}} int_{gamma_i} int_Omega U*(x-y,t) u0_h(y) dy ds_x dt
//            = (alpha/4pi) [N_i(t_{a+1}) - N_i(t_a)],  N_i(t) = int_{gamma_i} int_Omega E1(c/t) u0_h dy ds_x
// (exact time integral, c = alpha |x-y|^2 / 4, N_i(0) = 0).  Space: qx Gauss points on gamma_i,
// the collapsed (Duffy) tensor Gauss rule on each triangle (qt_near^2 points when the distance from
// gamma_i to the centroid is below 2 max(h_i, longest edge), else qt_far^2); the first step
// (a = 0: E1(c/t_1) alone is log singular at y = x) uses on the near triangles the apex-split rule
// at each x point: the three sub-triangles (x, V_k, V_k+1) with signed areas, radial coordinate on a
// geometric composite Gauss rule (ratio 0.15, 10 levels x 16 points: on a level [0.15 r, r] the log
// singularity sits 0.18 of its length away, Bernstein ratio 2.26, 2.26^-32 = 5e-12), angular
// 12-point Gauss
// (reading R22).  Node values from the moments of each warp's 32-triangle point cluster
// (initial_warp); per-warp partial rows, k_initial_finish sums them in fixed order.
#pragma once

namespace stb {

// x points of the first step on gamma_i (parameter f in [0, 1] and weight): 2 x 16 Gauss points on
// the halves of the element; a half that ends at a corner of Gamma (tangent change) gets geometric
// levels toward it instead (ratio 0.15, 8 levels x 8 points): the log kernel's potential over the
// domain is singular in x at a corner (reading R22)
struct XRule {
  int n0, n1, qx;
  bool plain;                                       // no corner: Gauss qx on the element
  __device__ __forceinline__ XRule(bool c0, bool c1, int q) : n0(c0 ? 64 : 16), n1(c1 ? 64 : 16), qx(q), plain(!c0 && !c1) {}
  __device__ __forceinline__ int n() const { return plain ? qx : n0 + n1; }
  __device__ __forceinline__ void point(int k, double& f, double& w) const {
    if (plain) {
      f = c_gx[qx][k];
      w = c_gw[qx][k];
      return;
    }
    const bool h1 = k >= n0;
    const int kk = h1 ? k - n0 : k, nh = h1 ? n1 : n0;
    double g, wg;                                   // position from the half's outer end, in [0, 1/2]
    if (nh == 16) {
      g = 0.5 * c_gx[16][kk];
      wg = 0.5 * c_gw[16][kk];
    } else {
      const int lev = kk >> 3, r = kk & 7;
      double hi = 0.5;
      for (int l = 0; l < lev; ++l) hi *= 0.15;
      const double lo = lev < 7 ? hi * 0.15 : 0.0;
      g = fma(hi - lo, c_gx[8][r], lo);
      wg = (hi - lo) * c_gw[8][r];
    }
    f = h1 ? 1.0 - g : g;
    w = wg;
  }
};

// one geometric xi level lev (0..10) of the sub-triangle (p, v_s, v_s+1) of the apex split
__device__ double apex_level(double px, double py, const double (&V)[6], const double (&uv)[3],
                             double u_apex, double alpha, double t1, int s, int lev) {
  double acc = 0.0;
  {
    const double e1x = V[2 * s] - px, e1y = V[2 * s + 1] - py;
    const double e2x = V[2 * ((s + 1) % 3)] - px, e2y = V[2 * ((s + 1) % 3) + 1] - py;
    const double area2 = e1x * e2y - e1y * e2x;      // signed
    if (fabs(area2) < 1e-300) return 0.0;
    const double u1 = uv[s], u2 = uv[(s + 1) % 3];
    // eta along the far side: the xi-integrated kernel ~ log rho(eta) is near-singular at a side end
    // the apex sits close to (x near a triangle vertex): geometric levels (ratio 0.15, 8 Gauss points
    // each) toward that end down to |p - v| / side, else 12 Gauss points (reading R22)
    const double l1 = sqrt(e1x * e1x + e1y * e1y), l2 = sqrt(e2x * e2x + e2y * e2y);
    const double sx = e2x - e1x, sy = e2y - e1y, ls = sqrt(sx * sx + sy * sy);
    const double dm = fmin(l1, l2);
    const bool grade = dm < 0.15 * ls, at0 = l1 < l2;
    const int nlev = grade ? min(14, (int)ceil(log(dm / ls) * (1.0 / log(0.15))) + 1) : 0;
    const int ne = grade ? 8 * nlev : 12;
    double hi = 1.0;
    for (int l = 0; l < lev; ++l) hi *= 0.15;
    {
      const double lo = lev < 10 ? hi * 0.15 : 0.0;
      for (int r = 0; r < 16; ++r) {
        const double xi = fma(hi - lo, c_gx[16][r], lo), wxi = (hi - lo) * c_gw[16][r];
        double part = 0.0, etop = 1.0;
        for (int e = 0; e < ne; ++e) {
          double eta, we;
          if (grade) {
            const int q = e & 7;
            const double ebot = (e >> 3) == nlev - 1 ? 0.0 : 0.15 * etop;
            const double d = fma(etop - ebot, c_gx[8][q], ebot);
            eta = at0 ? d : 1.0 - d;
            we = (etop - ebot) * c_gw[8][q];
            if (q == 7) etop = ebot;
          } else {
            eta = c_gx[12][e];
            we = c_gw[12][e];
          }
          const double dx = xi * fma(eta, sx, e1x), dy = xi * fma(eta, sy, e1y);
          const double uh = fma(xi, fma(eta, u2 - u1, u1) - u_apex, u_apex);
          const double c = 0.25 * alpha * (dx * dx + dy * dy);
          part = fma(we * uh, dev_e1(c / t1), part);
        }
        acc = fma(area2 * xi * wxi, part, acc);
      }
    }
  }
  return acc;
}

// the quadrature points of (gamma_i x triangle): x Gauss on gamma_i, the collapsed Duffy rule on the
// triangle; vis(c, W) with c = alpha |x - y|^2 / 4 and the full weight W (h area2 xi w w u0_h(y))
template <class F>
__device__ __forceinline__ void for_tri_points(const Seg& S, const double (&V)[6], const double (&uv)[3],
                                               int qx, int qt, double alpha, F&& vis) {
  const double e1x = V[2] - V[0], e1y = V[3] - V[1], e2x = V[4] - V[0], e2y = V[5] - V[1];
  const double area2 = fabs(e1x * e2y - e1y * e2x);
  for (int p = 0; p < qx; ++p) {
    const double xx = fma(c_gx[qx][p], S.bx - S.ax, S.ax), xy = fma(c_gx[qx][p], S.by - S.ay, S.ay);
    const double wp = c_gw[qx][p] * S.h * area2;
    for (int a1 = 0; a1 < qt; ++a1) {
      const double xi = c_gx[qt][a1];
      for (int a2 = 0; a2 < qt; ++a2) {
        const double eta = c_gx[qt][a2];
        const double u = xi * (1.0 - eta), v = xi * eta;
        const double yx = V[0] + u * e1x + v * e2x, yy = V[1] + u * e1y + v * e2y;
        const double uh = (1.0 - u - v) * uv[0] + u * uv[1] + v * uv[2];
        const double dx = xx - yx, dy = xy - yy;
        vis(0.25 * alpha * (dx * dx + dy * dy), wp * xi * c_gw[qt][a1] * c_gw[qt][a2] * uh);
      }
    }
  }
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// One warp = 32 triangles of a batch against element i.  The node values
//   N(t_n) = sum_{p in the warp's points} W_p E1(c_p / t_n)
// are evaluated on the moments of the WARP's joint point cluster (row f1):
//   regime A (c_max u < 4):  sum_k MEIN_k u^k M_k - gamma M_0 - L_0 - ln(u) M_0,
//                            M_k = sum W c^k, L_0 = sum W ln c           (E1 = Ein - gamma - ln x)
//   regime B (rho <= 1/2):   E1(x0) m_0 - sum_k a_{k-1} m_k / k, m_k = sum W (c - c0)^k (as phi_bz)
// -- algebraic identities of the point sum of each triangle's own rule (qt_far^2 or qt_near^2
// points), so the moments are summed over the 32 lanes once and each lane then evaluates its own
// nodes n = 1 + lane, 1 + lane + 32, ...  Nodes in neither regime (a prefix n < n_A of small t,
// only when the cluster is wide) take the per-lane point sum.  Step 0 (the log-singular E1(c/t_1)
// alone): the apex-split rule on near triangles, the regular rule on far ones.
// acc: this warp's row of nt + 2 node accumulators (shared or global), owned by the warp;
// sm: the warp's moment slots in shared memory (MKA + MKB + 2 doubles).
__device__ __forceinline__ void initial_warp(const Seg& S, const double* __restrict__ tg, int k, int nt,
                                             double alpha, const double* __restrict__ nodes,
                                             const int* __restrict__ tris, int ntri,
                                             const double* __restrict__ u0, int qx, int qtf, int qtn,
                                             int use_moments, double* acc, double* sm, bool cor0, bool cor1) {
  const int lane = threadIdx.x & 31;
  const XRule xr(cor0, cor1, qx);
  const bool valid = k < ntri;
  double V[6] = {0, 0, 0, 0, 0, 0}, uv[3] = {0, 0, 0};
  bool near = false;
  if (valid) {
#pragma unroll
    for (int v = 0; v < 3; ++v) {
      const int id = tris[3 * k + v];
      V[2 * v] = nodes[2 * id];
      V[2 * v + 1] = nodes[2 * id + 1];
      uv[v] = u0[id];
    }
    const double gx = (V[0] + V[2] + V[4]) / 3.0, gy = (V[1] + V[3] + V[5]) / 3.0;
    double le = 0.0;
#pragma unroll
    for (int v = 0; v < 3; ++v) {
      const double ex = V[2 * ((v + 1) % 3)] - V[2 * v], ey = V[2 * ((v + 1) % 3) + 1] - V[2 * v + 1];
      le = fmax(le, sqrt(ex * ex + ey * ey));
    }
    double f0 = (gx - S.ax) * S.tx + (gy - S.ay) * S.ty;
    f0 = fmin(fmax(f0, 0.0), S.h);
    const double qx0 = S.ax + f0 * S.tx - gx, qy0 = S.ay + f0 * S.ty - gy;
    near = sqrt(qx0 * qx0 + qy0 * qy0) < 2.0 * fmax(S.h, le);
  }
  const int qt = near ? qtn : qtf;
  // step 0.  Near triangles: the apex-split rule, work items (x point, sub-triangle, xi level) spread
  // over the warp one near triangle at a time (a corner row's graded x rule makes them heavy)
  double first = 0.0;
  unsigned nmask = __ballot_sync(0xffffffffu, valid && near);
  while (nmask) {
    const int src = __ffs(nmask) - 1;
    nmask &= nmask - 1;
    double Vs[6], us[3];
#pragma unroll
    for (int v = 0; v < 6; ++v) Vs[v] = __shfl_sync(0xffffffffu, V[v], src);
#pragma unroll
    for (int v = 0; v < 3; ++v) us[v] = __shfl_sync(0xffffffffu, uv[v], src);
    const double e1x = Vs[2] - Vs[0], e1y = Vs[3] - Vs[1], e2x = Vs[4] - Vs[0], e2y = Vs[5] - Vs[1];
    const double det = e1x * e2y - e1y * e2x;
    const int nitem = xr.n() * 33;
    for (int w = lane; w < nitem; w += 32) {
      const int p = w / 33, sl = w - 33 * p;
      double fp, wp;
      xr.point(p, fp, wp);
      const double xx = fma(fp, S.bx - S.ax, S.ax), xy = fma(fp, S.by - S.ay, S.ay);
      const double uu = ((xx - Vs[0]) * e2y - (xy - Vs[1]) * e2x) / det;
      const double vv = ((xy - Vs[1]) * e1x - (xx - Vs[0]) * e1y) / det;
      const double ua = (1.0 - uu - vv) * us[0] + uu * us[1] + vv * us[2];
      first = fma(wp * S.h, apex_level(xx, xy, Vs, us, ua, alpha, tg[1], sl / 11, sl % 11), first);
    }
  }
  if (valid && !near) {
    // step 0 alone on a far triangle: E1(c / t_1) varies on ell_1 = sqrt(4 t_1 / alpha); composite
    // collapsed rule of ceil(2 l / ell_1) cells per direction (reading R24)
    const double it = 1.0 / tg[1];
    const double e1x = V[2] - V[0], e1y = V[3] - V[1], e2x = V[4] - V[0], e2y = V[5] - V[1];
    const double l = sqrt(fmax(fmax(e1x * e1x + e1y * e1y, e2x * e2x + e2y * e2y),
                               (e2x - e1x) * (e2x - e1x) + (e2y - e1y) * (e2y - e1y)));
    const int ns = min(24, max(1, (int)ceil(2.0 * l / sqrt(4.0 * tg[1] / alpha))));
    const double ins = 1.0 / ns, area2 = fabs(e1x * e2y - e1y * e2x);
    // a triangle whose every point is beyond x = c/t_1 = 50 from gamma_i adds below e^{-50}/50
    const double gx = V[0] + (e1x + e2x) / 3.0, gy = V[1] + (e1y + e2y) / 3.0;
    double f0 = (gx - S.ax) * S.tx + (gy - S.ay) * S.ty;
    f0 = fmin(fmax(f0, 0.0), S.h);
    const double qx0 = S.ax + f0 * S.tx - gx, qy0 = S.ay + f0 * S.ty - gy;
    const double dmin = fmax(0.0, sqrt(qx0 * qx0 + qy0 * qy0) - l);
    // (smooth in x: Gauss qx on gamma_i also at a corner element)
    const int np = 0.25 * alpha * dmin * dmin * it > 50.0 ? 0 : qx;
    for (int p = 0; p < np; ++p) {
      const double fp = c_gx[qx][p], wp = c_gw[qx][p];
      const double xx = fma(fp, S.bx - S.ax, S.ax), xy = fma(fp, S.by - S.ay, S.ay);
      double sp = 0.0;
      for (int a1 = 0; a1 < qt * ns; ++a1) {
        const double xi = (a1 / qt + c_gx[qt][a1 % qt]) * ins;
        for (int a2 = 0; a2 < qt * ns; ++a2) {
          const double eta = (a2 / qt + c_gx[qt][a2 % qt]) * ins;
          const double u = xi * (1.0 - eta), v = xi * eta;
          const double dx = xx - (V[0] + u * e1x + v * e2x), dy = xy - (V[1] + u * e1y + v * e2y);
          const double uh = (1.0 - u - v) * uv[0] + u * uv[1] + v * uv[2];
          sp = fma(xi * c_gw[qt][a1 % qt] * c_gw[qt][a2 % qt] * uh, dev_e1(0.25 * alpha * (dx * dx + dy * dy) * it), sp);
        }
      }
      first = fma(wp * S.h * area2 * ins * ins, sp, first);
    }
  }
  first = warp_sum(first);
  if (lane == 0) acc[0] += first;

  // the warp's joint moments (all lanes hold the sums)
  double P[MKA + 1], mb[MKB + 1];
#pragma unroll
  for (int q = 0; q <= MKA; ++q) P[q] = 0.0;
#pragma unroll
  for (int q = 0; q <= MKB; ++q) mb[q] = 0.0;
  double L0 = 0.0, cmn = 1e300, cmx = 0.0;
  if (valid && use_moments)
    for_tri_points(S, V, uv, qx, qt, alpha, [&](double c, double W) {
      cmn = fmin(cmn, c);
      cmx = fmax(cmx, c);
      L0 = fma(W, log(c), L0);
      double pw = W;
#pragma unroll
      for (int q = 0; q <= MKA; ++q) {
        P[q] += pw;
        pw *= c;
      }
    });
  const double cmin = warp_min(valid ? cmn : 1e300), cmax = warp_max(valid ? cmx : 0.0);
  const double c0 = 0.5 * (cmin + cmax);
  const bool okB = use_moments && cmin > 0.0 && cmin < 1e300 && (cmax - c0) <= MRHO * c0;
  const double ic0 = okB ? 1.0 / c0 : 0.0;
  int kb = 0;
  if (okB) {
    const double rho = (cmax - c0) / c0;
    kb = rho <= 1e-6 ? 3 : min(MKB, max(3, (int)ceil(log(1e-16) / log(rho))));
    if (valid)
      for_tri_points(S, V, uv, qx, qt, alpha, [&](double c, double W) {
        const double d = c - c0;
        double pw = W;
#pragma unroll
        for (int q = 0; q <= MKB; ++q) {
          mb[q] += pw;
          pw *= d;
        }
      });
#pragma unroll
    for (int q = 0; q <= MKB; ++q)
      if (q <= kb) {                                      // kb warp-uniform
        const double v = warp_sum(mb[q]);
        if (lane == 0) sm[MKA + 1 + q] = q == 0 ? v : v * STB_INV[q];
      }
  }
  if (use_moments) {
    L0 = warp_sum(L0);
#pragma unroll
    for (int q = 0; q <= MKA; ++q) P[q] = warp_sum(P[q]);
    if (lane == 0) {
      sm[0] = P[0];
#pragma unroll
      for (int q = 1; q <= MKA; ++q) sm[q] = P[q] * STB_MEIN[q];
    }
    L0 = fma(STB_GAMMA, P[0], L0);                         // gamma M_0 + L_0
  }
  __syncwarp();
  const double* Pm = sm;                                   // joint moments, broadcast reads
  const double* mbm = sm + MKA + 1;
  // joint regimes; n_A = first node in regime A (t grows with n)
  int nA = nt + 1;
  if (use_moments) {
    for (int n = 1; n <= nt; ++n)
      if (cmax < 4.0 * tg[n]) {
        nA = n;
        break;
      }
  }
  const int nlane = use_moments && okB ? 1 : nA;          // nodes [1, nlane) take per-lane point sums
  for (int n = 1 + lane; n <= nt; n += 32) {
    if (n < nlane) continue;
    const double it = 1.0 / tg[n];
    double s = 0.0;
    if (cmin * it > STB_XUNDER) {
      s = 0.0;
    } else if (n >= nA) {
      double h = Pm[MKA];
#pragma unroll
      for (int q = MKA - 1; q >= 1; --q) h = fma(h, it, Pm[q]);
      s = fma(h, it, -fma(log(it), Pm[0], L0));
    } else {
      const double x0 = c0 * it, ex = exp(-x0), tt = ic0 * tg[n];
      const double E1 = ex * tt * gb3_cb(tt);
      double e = ex, ap = ex * ic0, S1 = 0.0;
      for (int q = 1; q <= kb; ++q) {
        e = -e * (it * STB_INV[q]);
        S1 = fma(ap, mbm[q], S1);
        ap = (e - ap) * ic0;
      }
      s = fma(E1, mbm[0], -S1);
    }
    acc[n] += s;
  }
  for (int n = 1; n < nlane; ++n) {                       // per-lane point sums (rare with moments)
    const double it = 1.0 / tg[n];
    double s = 0.0;
    if (valid)
      for_tri_points(S, V, uv, qx, qt, alpha, [&](double c, double W) {
        if (c * it <= STB_XUNDER) s = fma(W, dev_e1(c * it), s);
      });
    s = warp_sum(s);
    if (lane == 0) acc[n] += s;
  }
}

// CTA = (element i, chunk), 8 warps: the chunk's triangle batches k = (bt * nch + chunk) * 256 + tid
// are interleaved over the chunks (balance of the near triangles); every warp accumulates its node
// values into its own row (shared memory when 8 (nt + 2) doubles fit, else its global partial row)
// in batch order; k_initial_finish sums the rows in fixed order (deterministic).
__global__ void __launch_bounds__(256) k_initial(const Seg* __restrict__ seg, const double* __restrict__ tg,
                                                int ng, int nt, double alpha,
                                                const double* __restrict__ nodes, const int* __restrict__ tris,
                                                int ntri, const double* __restrict__ u0, int qx, int qtf, int qtn,
                                                int use_moments, int nbatch, int use_smem,
                                                double* __restrict__ part) {
  extern __shared__ double acc_s[];
  __shared__ double msh[8][MKA + MKB + 2];               // each warp's joint moments
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long row = (((long long)blockIdx.x * gridDim.y + blockIdx.y) * 8 + warp) * (nt + 2);
  double* acc = use_smem ? acc_s + warp * (nt + 2) : part + row;
  for (int r = lane; r < nt + 2; r += 32) acc[r] = 0.0;
  __syncwarp();
  const Seg S = seg[blockIdx.x];
  const Seg Sp = seg[(blockIdx.x + ng - 1) % ng], Sn = seg[(blockIdx.x + 1) % ng];
  const bool cor0 = S.tx * Sp.tx + S.ty * Sp.ty < 1.0 - 1e-12, cor1 = S.tx * Sn.tx + S.ty * Sn.ty < 1.0 - 1e-12;
  for (int bt = 0; bt < nbatch; ++bt) {
    const int k0 = (bt * gridDim.y + blockIdx.y) * 256;
    if (k0 >= ntri) break;                                // CTA-uniform
    initial_warp(S, tg, k0 + threadIdx.x, nt, alpha, nodes, tris, ntri, u0, qx, qtf, qtn, use_moments, acc,
                 msh[warp], cor0, cor1);
    __syncwarp();
  }
  if (use_smem) {
    __syncwarp();
    for (int r = lane; r < nt + 2; r += 32) part[row + r] = acc[r];
  }
}

__global__ void k_initial_finish(const double* __restrict__ part, int ng, int nt, int nch, double alpha,
                                 double* __restrict__ b) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (long long)ng * nt) return;
  const int a = (int)(r / ng), i = (int)(r % ng);
  double v = 0.0;
  for (int row = 0; row < nch * 8; ++row) {       // chunk-major, warp-minor: fixed order
    const double* p = part + ((long long)i * nch * 8 + row) * (nt + 2);
    v += a == 0 ? p[0] : p[a + 1] - p[a];
  }
  b[r] -= alpha / (4.0 * STB_PI) * v;    // b <- b - M_h^0 u0 (eq. 4)
}

}  // namespace stb
