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

}  // namespace stb
