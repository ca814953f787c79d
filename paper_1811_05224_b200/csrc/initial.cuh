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
// geometric composite Gauss rule (ratio 0.15, 10 levels x 8 points), angular 12-point Gauss
// (reading R22).  CTA = (element i, chunk of 256 triangles), thread = triangle, one block
// sum per time node into fixed partial slots, k_initial_finish sums the chunks in fixed order.
#pragma once

namespace stb {

__device__ __forceinline__ double block_sum256(double v, double* red) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += red[k];
  return s;
}

__device__ double apex_split(double px, double py, const double (&V)[6], const double (&uv)[3],
                             double u_apex, double alpha, double t1) {
  double acc = 0.0;
  for (int s = 0; s < 3; ++s) {
    const double e1x = V[2 * s] - px, e1y = V[2 * s + 1] - py;
    const double e2x = V[2 * ((s + 1) % 3)] - px, e2y = V[2 * ((s + 1) % 3) + 1] - py;
    const double area2 = e1x * e2y - e1y * e2x;      // signed
    if (fabs(area2) < 1e-300) continue;
    const double u1 = uv[s], u2 = uv[(s + 1) % 3];
    double hi = 1.0;
    for (int lev = 0; lev <= 10; ++lev) {
      const double lo = lev < 10 ? hi * 0.15 : 0.0;
      for (int r = 0; r < 8; ++r) {
        const double xi = fma(hi - lo, c_gx[8][r], lo), wxi = (hi - lo) * c_gw[8][r];
        double part = 0.0;
        for (int e = 0; e < 12; ++e) {
          const double eta = c_gx[12][e];
          const double dx = xi * fma(eta, e2x - e1x, e1x), dy = xi * fma(eta, e2y - e1y, e1y);
          const double uh = fma(xi, fma(eta, u2 - u1, u1) - u_apex, u_apex);
          const double c = 0.25 * alpha * (dx * dx + dy * dy);
          part = fma(c_gw[12][e] * uh, dev_e1(c / t1), part);
        }
        acc = fma(area2 * xi * wxi, part, acc);
      }
      hi = lo;
    }
  }
  return acc;
}

__global__ void __launch_bounds__(256) k_initial(const Seg* __restrict__ seg, const double* __restrict__ tg,
                                                int ng, int nt, double alpha,
                                                const double* __restrict__ nodes, const int* __restrict__ tris,
                                                int ntri, const double* __restrict__ u0, int qx, int qtf, int qtn,
                                                double* __restrict__ part) {
  __shared__ double red[8];
  const int i = blockIdx.x, k = blockIdx.y * 256 + threadIdx.x;
  const bool valid = k < ntri;
  const Seg S = seg[i];
  double V[6] = {0, 0, 0, 0, 0, 0}, uv[3] = {0, 0, 0};
  bool near = false;
  double cmin = 1e300;
  if (valid) {
#pragma unroll
    for (int v = 0; v < 3; ++v) {
      const int id = tris[3 * k + v];
      V[2 * v] = nodes[2 * id];
      V[2 * v + 1] = nodes[2 * id + 1];
      uv[v] = u0[id];
    }
    const double gx = (V[0] + V[2] + V[4]) / 3.0, gy = (V[1] + V[3] + V[5]) / 3.0;
    double le = 0.0, rad = 0.0;
#pragma unroll
    for (int v = 0; v < 3; ++v) {
      const double ex = V[2 * ((v + 1) % 3)] - V[2 * v], ey = V[2 * ((v + 1) % 3) + 1] - V[2 * v + 1];
      le = fmax(le, sqrt(ex * ex + ey * ey));
      rad = fmax(rad, sqrt((V[2 * v] - gx) * (V[2 * v] - gx) + (V[2 * v + 1] - gy) * (V[2 * v + 1] - gy)));
    }
    double f0 = (gx - S.ax) * S.tx + (gy - S.ay) * S.ty;
    f0 = fmin(fmax(f0, 0.0), S.h);
    const double qx0 = S.ax + f0 * S.tx - gx, qy0 = S.ay + f0 * S.ty - gy;
    const double dist = sqrt(qx0 * qx0 + qy0 * qy0);
    near = dist < 2.0 * fmax(S.h, le);
    const double dmin = fmax(0.0, dist - rad);
    cmin = 0.25 * alpha * dmin * dmin;    // lower bound of c over the triangle x gamma_i
  }
  const double e1x = V[2] - V[0], e1y = V[3] - V[1], e2x = V[4] - V[0], e2y = V[5] - V[1];
  const double area2 = fabs(e1x * e2y - e1y * e2x);
  const int qt = near ? qtn : qtf;
  double first = 0.0;
  if (valid && near) {
    // step 0 on a near triangle: the apex-split rule at every x point
    const double det = e1x * e2y - e1y * e2x;
    for (int p = 0; p < qx; ++p) {
      const double xx = fma(c_gx[qx][p], S.bx - S.ax, S.ax), xy = fma(c_gx[qx][p], S.by - S.ay, S.ay);
      const double uu = ((xx - V[0]) * e2y - (xy - V[1]) * e2x) / det;
      const double vv = ((xy - V[1]) * e1x - (xx - V[0]) * e1y) / det;
      const double ua = (1.0 - uu - vv) * uv[0] + uu * uv[1] + vv * uv[2];
      first = fma(c_gw[qx][p] * S.h, apex_split(xx, xy, V, uv, ua, alpha, tg[1]), first);
    }
  }
  const long long base = ((long long)blockIdx.x * gridDim.y + blockIdx.y) * (nt + 2);
  for (int n = 1; n <= nt; ++n) {
    const double it = 1.0 / tg[n];
    double s = 0.0;
    if (valid && cmin * it <= STB_XUNDER) {
      for (int p = 0; p < qx; ++p) {
        const double xx = fma(c_gx[qx][p], S.bx - S.ax, S.ax), xy = fma(c_gx[qx][p], S.by - S.ay, S.ay);
        double sp = 0.0;
        for (int a1 = 0; a1 < qt; ++a1) {
          const double xi = c_gx[qt][a1];
          for (int a2 = 0; a2 < qt; ++a2) {
            const double eta = c_gx[qt][a2];
            const double u = xi * (1.0 - eta), v = xi * eta;
            const double yx = V[0] + u * e1x + v * e2x, yy = V[1] + u * e1y + v * e2y;
            const double uh = (1.0 - u - v) * uv[0] + u * uv[1] + v * uv[2];
            const double dx = xx - yx, dy = xy - yy;
            const double c = 0.25 * alpha * (dx * dx + dy * dy);
            sp = fma(xi * c_gw[qt][a1] * c_gw[qt][a2] * uh, dev_e1(c * it), sp);
          }
        }
        s = fma(c_gw[qx][p] * S.h * area2, sp, s);
      }
    }
    if (n == 1 && !near) first += s;         // far triangles: the regular rule serves step 0 too
    const double tot = block_sum256(s, red);
    if (threadIdx.x == 0) part[base + n] = tot;
  }
  const double tf = block_sum256(first, red);
  if (threadIdx.x == 0) part[base] = tf;
}

__global__ void k_initial_finish(const double* __restrict__ part, int ng, int nt, int nch, double alpha,
                                 double* __restrict__ b) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (long long)ng * nt) return;
  const int a = (int)(r / ng), i = (int)(r % ng);
  double v = 0.0;
  for (int ch = 0; ch < nch; ++ch) {
    const double* p = part + ((long long)i * nch + ch) * (nt + 2);
    v += a == 0 ? p[0] : p[a + 1] - p[a];
  }
  b[r] -= alpha / (4.0 * STB_PI) * v;    // b <- b - M_h^0 u0 (eq. 4)
}

}  // namespace stb
