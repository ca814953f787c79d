// potential.cuh — representation formula in Q (eq. 2), included by
// assemble.cu (the Gauss tables live in its __constant__ memory).  With u0 = 0:
//   u(x,t) = (Vt w)(x,t) - (W g)(x,t)
//   (Vt w)(x,t) = sum_{b,j} w_bj h_j int_0^1 (1/(4 pi)) [E1(c/s_hi) - E1(c/s_lo)] df
//   (W g)(x,t)  = sum_{b,j} h_j int_0^1 g_b(y(f)) ((x - y).n_j / (2 pi r^2)) [e^{-c/s_hi} - e^{-c/s_lo}] df
// with the exact time integrals of (1/alpha) U* and (1/alpha) d_ny U* over step b (s = t - tau,
// s_hi = t - t_b, s_lo = max(0, t - t_{b+1})), c = alpha r^2 / 4, w piecewise constant and g the
// nodal hat interpolant (constant in time per step).  Gauss order per element from the distance
// ratio rho = dist / h: 16 (rho < 2), 12 (rho < 6), 8 (Bernstein-ellipse error below 1e-19 for
// rho >= 1); points closer than h_max to Gamma are rejected.  One warp per point, lanes over the
// elements, each time node evaluated once per Gauss point, a warp sum per point (deterministic).
#pragma once

namespace stb {

template <int Q>
__device__ __forceinline__ void pot_element(const Seg& S, double x1, double x2, double t, double alpha,
                                            const double* __restrict__ tg, int nb, int ng, int j,
                                            const double* __restrict__ w, const double* __restrict__ g,
                                            double& sv, double& sw) {
  double c[Q], kw[Q], pv[Q], pw[Q], Fn[Q], En[Q];
#pragma unroll
  for (int u = 0; u < Q; ++u) {
    const double f = c_gx[Q][u];
    const double d1 = x1 - fma(f, S.bx - S.ax, S.ax), d2 = x2 - fma(f, S.by - S.ay, S.ay);
    const double r2 = d1 * d1 + d2 * d2;
    c[u] = 0.25 * alpha * r2;
    kw[u] = (d1 * S.nx + d2 * S.ny) / r2;
    pv[u] = pw[u] = Fn[u] = En[u] = 0.0;   // node nb: s <= 0, the antiderivatives vanish
  }
  const int j1 = (j + 1) % ng;
  for (int b = nb - 1; b >= 0; --b) {
    const double is = 1.0 / (t - tg[b]);
    const long long o = (long long)b * ng;
    const double wb = w[o + j], g0 = g[o + j], dg = g[o + j1] - g0;
#pragma unroll
    for (int u = 0; u < Q; ++u) {
      const double x = c[u] * is;
      const double Fb = dev_e1(x), Eb = exp(-x);
      pv[u] = fma(wb, Fb - Fn[u], pv[u]);
      pw[u] = fma(fma(c_gx[Q][u], dg, g0), Eb - En[u], pw[u]);
      Fn[u] = Fb;
      En[u] = Eb;
    }
  }
#pragma unroll
  for (int u = 0; u < Q; ++u) {
    sv = fma(c_gw[Q][u], pv[u], sv);
    sw = fma(c_gw[Q][u] * kw[u], pw[u], sw);
  }
}

__global__ void __launch_bounds__(128) k_potential(const Seg* __restrict__ seg, const double* __restrict__ tg,
                                                  int ng, int nt, double alpha, double hmin_dist,
                                                  const double* __restrict__ w, const double* __restrict__ g,
                                                  long long npts, const double* __restrict__ pts,
                                                  double* __restrict__ out, int* __restrict__ bad) {
  const long long k = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (k >= npts) return;   // warp-uniform
  const int lane = threadIdx.x & 31;
  const double x1 = pts[3 * k], x2 = pts[3 * k + 1], t = pts[3 * k + 2];
  int nb = 0;               // steps with t_b < t
  while (nb < nt && tg[nb] < t) ++nb;
  double vw = 0.0, wg = 0.0;
  bool near = false;
  // lanes over the elements j; the time steps are swept from the last one down so that each time
  // node t_b is evaluated once per Gauss point (E1 and e^{-x} at s = t - t_b serve steps b-1, b),
  // the Q Gauss points of an element advance together (independent chains, one load of w, g per step)
  for (int j = lane; j < ng; j += 32) {
    const Seg S = seg[j];
    double f0 = (x1 - S.ax) * S.tx + (x2 - S.ay) * S.ty;
    f0 = fmin(fmax(f0, 0.0), S.h);
    const double qx = S.ax + f0 * S.tx - x1, qy = S.ay + f0 * S.ty - x2;
    const double dist = sqrt(qx * qx + qy * qy);
    near |= dist < hmin_dist;
    const double rho = dist / S.h;
    double sv = 0.0, sw = 0.0;
    if (rho < 2.0) pot_element<16>(S, x1, x2, t, alpha, tg, nb, ng, j, w, g, sv, sw);
    else if (rho < 6.0) pot_element<12>(S, x1, x2, t, alpha, tg, nb, ng, j, w, g, sv, sw);
    else pot_element<8>(S, x1, x2, t, alpha, tg, nb, ng, j, w, g, sv, sw);
    vw = fma(S.h, sv, vw);
    wg = fma(S.h, sw, wg);
  }
  vw = warp_sum(vw) / (4.0 * STB_PI);
  wg = warp_sum(wg) / (2.0 * STB_PI);
  if (__any_sync(0xffffffffu, near) && lane == 0) atomicOr(bad, 1);
  if (lane == 0) out[k] = vw - wg;
}

// Initial potential of the representation formula (eq. 2; row f2 with u0 != 0):
//   u(x,t) += (M~_0 u0)(x,t) = int_Omega U*(x - y, t) u0_h(y) dy,  U*(z,t) = alpha/(4 pi t) e^{-alpha |z|^2/(4t)}.
// Warp per point, lanes over the triangles.  Each triangle by the collapsed Gauss rule of order 6 on
// ns x ns cells, ns = ceil(l / ell), ell = sqrt(4 t / alpha) the Gaussian's width (reading R24);
// triangles whose distance from x exceeds 7 ell are skipped (their integrand is below
// e^{-49} = 5e-22 of the peak).  Points with t <= 0 set *bad.
__global__ void __launch_bounds__(128) k_potential_initial(const double* __restrict__ nodes,
                                                          const int* __restrict__ tris, int ntri,
                                                          const double* __restrict__ u0, double alpha,
                                                          long long npts, const double* __restrict__ pts,
                                                          double* __restrict__ out, int* bad) {
  const long long p = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= npts) return;                                  // warp-uniform
  const double x1 = pts[3 * p], x2 = pts[3 * p + 1], t = pts[3 * p + 2];
  if (!(t > 0.0)) {
    if (lane == 0) atomicExch(bad, 1);
    return;
  }
  constexpr int Q = 6;
  const double ell = sqrt(4.0 * t / alpha), ia = alpha / (4.0 * t);
  double acc = 0.0;
  for (int e = lane; e < ntri; e += 32) {
    const int i0 = tris[3 * e], i1 = tris[3 * e + 1], i2 = tris[3 * e + 2];
    const double ax = nodes[2 * i0], ay = nodes[2 * i0 + 1];
    const double e1x = nodes[2 * i1] - ax, e1y = nodes[2 * i1 + 1] - ay;
    const double e2x = nodes[2 * i2] - ax, e2y = nodes[2 * i2 + 1] - ay;
    const double l = sqrt(fmax(fmax(e1x * e1x + e1y * e1y, e2x * e2x + e2y * e2y),
                               (e2x - e1x) * (e2x - e1x) + (e2y - e1y) * (e2y - e1y)));
    // distance from x to the triangle >= distance to the centroid - circumradius bound (l)
    const double gx = ax + (e1x + e2x) / 3.0 - x1, gy = ay + (e1y + e2y) / 3.0 - x2;
    if (sqrt(gx * gx + gy * gy) - l > 7.0 * ell) continue;
    const double u0a = u0[i0], u0b = u0[i1], u0c = u0[i2];
    const int ns = min(64, max(1, (int)ceil(l / ell)));
    const double ins = 1.0 / ns;
    double ts = 0.0;
    for (int cx = 0; cx < ns; ++cx)
#pragma unroll
      for (int a1 = 0; a1 < Q; ++a1) {
        const double xi = (cx + c_gx[Q][a1]) * ins, wx = c_gw[Q][a1] * xi;
        double row = 0.0;
        for (int cy = 0; cy < ns; ++cy)
#pragma unroll
          for (int a2 = 0; a2 < Q; ++a2) {
            const double eta = (cy + c_gx[Q][a2]) * ins;
            const double u = xi * (1.0 - eta), v = xi * eta;
            const double dx = x1 - (ax + u * e1x + v * e2x), dy = x2 - (ay + u * e1y + v * e2y);
            const double uh = fma(u, u0b - u0a, fma(v, u0c - u0a, u0a));
            row = fma(c_gw[Q][a2] * uh, exp(-ia * (dx * dx + dy * dy)), row);
          }
        ts = fma(wx, row, ts);
      }
    acc = fma(fabs(e1x * e2y - e1y * e2x) * ins * ins, ts, acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) out[p] += alpha / (4.0 * STB_PI * t) * acc;
}

}  // namespace stb
