/*
 * stbem_oracle.c — CPU ORACLE for the space-time Galerkin BEM of
 * Dohr, Merta, Of, Steinbach, Zapletal (arXiv:1811.05224).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_1811_05224_b200/csrc) and neither side includes the other.
 *
 * What it computes (PAPER.md = P:<line>):
 *   V_h[(a,i),(b,j)] = <V phi^0_(b,j), phi^0_(a,i)>        P:86  (eq. 4 defs)
 *   K_h[(a,i),(b,n)] = <K phi^10_(b,n), phi^0_(a,i)>
 *   D_h[(a,l),(b,k)] = <D psi_(b,k), psi_(a,l)>             P:108 (Thm 1)
 * with the fundamental solution U* of P:47-54, the 1/alpha prefactors of the
 * boundary potentials, D = -d_n W in the integration-by-parts
 * form cited at P:129 (derived in DESIGN.md, reading R7), and the dual space
 * Y_h = X^{1,0}(dual mesh) of P:133 (dual nodes = primal midpoints, R6).
 *
 * Method (step by step, in the paper's notation; every choice the paper leaves
 * open is a DESIGN.md reading):
 *   1. time integrals are exact: the double antiderivatives
 *        H(s) = [(s+c)E1(c/s) - s e^{-c/s}]/(4 pi)          for (1/alpha) U*
 *        Q(s) = (alpha/(8 pi)) [e^{-x}/x - E1(x)], x=c/s    for (1/alpha) d_ny U* / dot
 *      and the first antiderivative F(s) = alpha E1(c/s)/(4 pi) of U*, c = alpha r^2/4,
 *      combined by the four-lag second difference sum_m eps_m G(s_m),
 *      s = (t_{a+1}-t_b, t_a-t_b, t_{a+1}-t_{b+1}, t_a-t_{b+1}), eps = (+,-,-,+).
 *   2. space integrals: tensor Gauss-Legendre on segment pairs that do not touch;
 *      segment pairs that touch (identical or sharing a vertex) are split as
 *      kernel = R(c) + P(c) ln c, R smooth, P a polynomial; R by Gauss after
 *      the 1-D reduction (identical) or the Duffy map at the shared vertex,
 *      the ln part by the exact identity  int_0^1 g(r) ln r dr = -int_0^1 int_0^1 g(r t) dr dt.
 *   3. E1 by its power series (x <= 1) and continued fraction (x > 1).
 *
 * Pins (tests/test_oracle_pins.py): closed forms of U*, mpmath values of E1,
 * H/F/Q against numerical time quadrature, brute-force mpmath integrals of
 * singular entries, the K row-sum "1/2 I jump" identity, the D normal-term
 * row-sum identity, Laplace steady limits, mass-matrix closed forms.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORA_PI 3.14159265358979323846264338327950288
#define ORA_EULER 0.57721566490153286060651209008240243

/* ------------------------------------------------------------------ E1 --- */
/* Ein(x) = sum_{k>=1} (-1)^{k+1} x^k / (k k!)   (entire part of E1) */
static double ora_ein_series(double x) {
  double term = x, sum = x;
  for (int k = 2; k < 200; ++k) {
    term *= -x / k;               /* term = (-1)^{k+1} x^k / k! */
    double add = term / k;
    sum += add;
    if (fabs(add) < 1e-18 * fabs(sum)) break;
  }
  return sum;
}

/* E1(x) = int_x^inf e^{-t}/t dt, x > 0 */
double ora_e1(double x) {
  if (!(x > 0.0)) return INFINITY;
  if (x <= 1.0) return -ORA_EULER - log(x) + ora_ein_series(x);
  if (x > 745.0) return 0.0;
  /* continued fraction E1(x) = e^{-x} / (x+1 - 1^2/(x+3 - 2^2/(x+5 - ...))),
     evaluated by the modified Lentz method */
  const double tiny = 1e-300;
  double b = x + 1.0, c = 1.0 / tiny, d = 1.0 / b, h = d;
  for (int i = 1; i < 100000; ++i) {
    double an = -(double)i * i;
    b += 2.0;
    d = 1.0 / (an * d + b);
    c = b + an / c;
    double del = c * d;
    h *= del;
    if (fabs(del - 1.0) < 1e-17) break;
  }
  return h * exp(-x);
}

/* Ein(x) = E1(x) + gamma + ln x, accurate for all x >= 0 */
double ora_ein(double x) {
  if (x <= 2.0) return ora_ein_series(x);
  return ora_e1(x) + ORA_EULER + log(x);
}

/* -------------------------------------------------------------- kernels --- */
/* U*(z,s) and (1/alpha) d_{n_y} U*, for pins only */
double ora_ustar(double alpha, double r2, double s) {
  if (!(s > 0.0)) return 0.0;
  return alpha / (4.0 * ORA_PI * s) * exp(-alpha * r2 / (4.0 * s));
}
double ora_ustar_dny(double alpha, double dot, double r2, double s) {
  /* d/dn_y U*(x-y,s) = alpha^2 ((x-y).n_y) / (8 pi s^2) exp(-alpha r^2/(4s)) */
  if (!(s > 0.0)) return 0.0;
  return alpha * alpha * dot / (8.0 * ORA_PI * s * s) * exp(-alpha * r2 / (4.0 * s));
}
/* single-lag antiderivatives (exposed for the d/ds pins) */
double ora_H(double alpha, double r2, double s) {
  if (!(s > 0.0)) return 0.0;
  double c = alpha * r2 / 4.0, x = c / s;
  return ((s + c) * ora_e1(x) - s * exp(-x)) / (4.0 * ORA_PI);
}
double ora_F(double alpha, double r2, double s) {
  if (!(s > 0.0)) return 0.0;
  double c = alpha * r2 / 4.0;
  return alpha * ora_e1(c / s) / (4.0 * ORA_PI);
}
double ora_Q(double alpha, double r2, double s) {
  if (!(s > 0.0)) return 0.0;
  double c = alpha * r2 / 4.0, x = c / s;
  return alpha / (8.0 * ORA_PI) * (exp(-x) / x - ora_e1(x));
}

/* lag set of the time-cell (a,b): the four-lag second difference */
typedef struct {
  int n;
  double s[4], e[4];
  double S;      /* sum eps_m s_m over positive lags: h_a for d=0, exactly 0 for d>=1 */
  int d;
} ora_lags;

static ora_lags make_lags(const double* t, int a, int b) {
  ora_lags L;
  L.n = 0;
  L.d = a - b;
  double s[4] = {t[a + 1] - t[b], t[a] - t[b], t[a + 1] - t[b + 1], t[a] - t[b + 1]};
  double e[4] = {1.0, -1.0, -1.0, 1.0};
  for (int m = 0; m < 4; ++m)
    if (s[m] > 0.0) { L.s[L.n] = s[m]; L.e[L.n] = e[m]; L.n++; }
  L.S = (L.d == 0) ? (t[a + 1] - t[a]) : 0.0;
  return L;
}

enum { KER_H = 0, KER_F = 1, KER_Q = 2 };

/* direct kernel sum at a point pair with c > 0 (non-touching pairs) */
static double ker_direct(int ker, const ora_lags* L, double alpha, double c) {
  double acc = 0.0;
  if (ker == KER_H) {
    for (int m = 0; m < L->n; ++m) {
      double s = L->s[m], x = c / s;
      acc += L->e[m] * s * ((1.0 + x) * ora_e1(x) - exp(-x));
    }
    return acc / (4.0 * ORA_PI);
  } else if (ker == KER_F) {
    for (int m = 0; m < L->n; ++m) acc += L->e[m] * ora_e1(c / L->s[m]);
    return alpha * acc / (4.0 * ORA_PI);
  } else {
    /* sum eps Q = (alpha/8pi) [ S/c + sum eps psi(x) ], psi(x) = e^{-x}/x - 1/x - E1(x) */
    for (int m = 0; m < L->n; ++m) {
      double x = c / L->s[m], psi;
      if (x < 2.0) psi = expm1(-x) / x + ORA_EULER + log(x) - ora_ein(x);
      else psi = exp(-x) / x - 1.0 / x - ora_e1(x);
      acc += L->e[m] * psi;
    }
    return alpha / (8.0 * ORA_PI) * (L->S / c + acc);
  }
}

/* split form kernel = R(c) + P(c) ln c (touching pairs); R finite at c = 0 */
static void ker_split(int ker, const ora_lags* L, double alpha, double c, double* R, double* P) {
  double r = 0.0, p = 0.0;
  if (ker == KER_H) {
    for (int m = 0; m < L->n; ++m) {
      double s = L->s[m], x = c / s;
      r += L->e[m] * ((s + c) * (-ORA_EULER + log(s) + ora_ein(x)) - s * exp(-x));
      p += L->e[m] * (s + c);
    }
    *R = r / (4.0 * ORA_PI);
    *P = -p / (4.0 * ORA_PI);
  } else if (ker == KER_F) {
    for (int m = 0; m < L->n; ++m) {
      double s = L->s[m], x = c / s;
      r += L->e[m] * (-ORA_EULER + log(s) + ora_ein(x));
      p += L->e[m];
    }
    *R = alpha * r / (4.0 * ORA_PI);
    *P = -alpha * p / (4.0 * ORA_PI);
  } else {
    /* without the dot factor; the S/c term is returned inside R (caller guarantees c>0
       whenever S != 0, i.e. only vertex-sharing pairs at d = 0) */
    for (int m = 0; m < L->n; ++m) {
      double s = L->s[m], x = c / s;
      double em1 = (x > 0.0) ? expm1(-x) / x : -1.0;
      r += L->e[m] * (em1 + ORA_EULER - log(s) - ora_ein(x));
      p += L->e[m];
    }
    *R = alpha / (8.0 * ORA_PI) * ((L->S != 0.0 ? L->S / c : 0.0) + r);
    *P = alpha / (8.0 * ORA_PI) * p;
  }
}

/* ------------------------------------------------------- Gauss-Legendre --- */
/* n-point Gauss-Legendre rule on [0,1]: Newton iteration on P_n */
static void gauss01(int n, double* x, double* w) {
  for (int i = 0; i < n; ++i) {
    double z = cos(ORA_PI * (i + 0.75) / (n + 0.5)), pp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p1 = 1.0, p2 = 0.0;
      for (int k = 1; k <= n; ++k) {
        double p3 = p2;
        p2 = p1;
        p1 = ((2.0 * k - 1.0) * z * p2 - (k - 1.0) * p3) / k;
      }
      pp = n * (z * p1 - p2) / (z * z - 1.0);
      double dz = p1 / pp;
      z -= dz;
      if (fabs(dz) < 1e-16) break;
    }
    /* recompute derivative at the converged root */
    {
      double p1 = 1.0, p2 = 0.0;
      for (int k = 1; k <= n; ++k) {
        double p3 = p2;
        p2 = p1;
        p1 = ((2.0 * k - 1.0) * z * p2 - (k - 1.0) * p3) / k;
      }
      pp = n * (z * p1 - p2) / (z * z - 1.0);
    }
    x[i] = 0.5 * (1.0 - z);
    w[i] = 1.0 / ((1.0 - z * z) * pp * pp);   /* = (2/((1-z^2)P'^2)) / 2 */
  }
}

#define ORA_QMAX 32
typedef struct { int n; double x[ORA_QMAX], w[ORA_QMAX]; } ora_rule;
static ora_rule RULES[ORA_QMAX + 1];
static int rules_ready = 0;
static void init_rules(void) {
  if (rules_ready) return;
  for (int n = 1; n <= ORA_QMAX; ++n) { RULES[n].n = n; gauss01(n, RULES[n].x, RULES[n].w); }
  rules_ready = 1;
}

/* ----------------------------------------------------------------- mesh --- */
typedef struct {
  double ax, ay, bx, by;   /* endpoints */
  double h;                /* length */
  double tx, ty;           /* unit tangent */
  double nx, ny;           /* outward unit normal */
} ora_seg;

typedef struct {
  int ng, nt;              /* N_Gamma, N_I */
  double alpha;
  double* t;               /* nt+1 */
  ora_seg* seg;            /* ng primal segments */
  ora_seg* half;           /* 2 ng half segments: 2i=[x_i,m_i], 2i+1=[m_i,x_{i+1}] */
  int q_far, q_near, q_sing, q_log;
  double ell;              /* sqrt(4 min h_t / alpha) (reading R24) */
} ora_mesh;

static ora_seg make_seg(double ax, double ay, double bx, double by) {
  ora_seg s;
  s.ax = ax; s.ay = ay; s.bx = bx; s.by = by;
  double dx = bx - ax, dy = by - ay;
  s.h = sqrt(dx * dx + dy * dy);
  s.tx = dx / s.h; s.ty = dy / s.h;
  s.nx = s.ty; s.ny = -s.tx;     /* CCW polygon: outward normal = tangent rotated clockwise */
  return s;
}

/* vertices: nv CCW polygon corners; segs_per_side[nv]; t: nt+1 breakpoints */
ora_mesh* ora_mesh_new(int nv, const double* vxy, const int* segs_per_side, int nt,
                       const double* t, double alpha) {
  init_rules();
  int ng = 0;
  for (int s = 0; s < nv; ++s) ng += segs_per_side[s];
  ora_mesh* m = (ora_mesh*)calloc(1, sizeof(ora_mesh));
  m->ng = ng; m->nt = nt; m->alpha = alpha;
  m->t = (double*)malloc(sizeof(double) * (nt + 1));
  memcpy(m->t, t, sizeof(double) * (nt + 1));
  double* nodes = (double*)malloc(sizeof(double) * 2 * ng);
  int k = 0;
  for (int s = 0; s < nv; ++s) {
    double x0 = vxy[2 * s], y0 = vxy[2 * s + 1];
    double x1 = vxy[2 * ((s + 1) % nv)], y1 = vxy[2 * ((s + 1) % nv) + 1];
    for (int j = 0; j < segs_per_side[s]; ++j) {
      double f = (double)j / segs_per_side[s];
      nodes[2 * k] = x0 + f * (x1 - x0);
      nodes[2 * k + 1] = y0 + f * (y1 - y0);
      ++k;
    }
  }
  m->seg = (ora_seg*)malloc(sizeof(ora_seg) * ng);
  m->half = (ora_seg*)malloc(sizeof(ora_seg) * 2 * ng);
  for (int i = 0; i < ng; ++i) {
    int i1 = (i + 1) % ng;
    double ax = nodes[2 * i], ay = nodes[2 * i + 1], bx = nodes[2 * i1], by = nodes[2 * i1 + 1];
    m->seg[i] = make_seg(ax, ay, bx, by);
    double mx = 0.5 * (ax + bx), my = 0.5 * (ay + by);
    m->half[2 * i] = make_seg(ax, ay, mx, my);
    m->half[2 * i + 1] = make_seg(mx, my, bx, by);
    /* the half segments inherit the exact normal of their parent */
    m->half[2 * i].nx = m->half[2 * i + 1].nx = m->seg[i].nx;
    m->half[2 * i].ny = m->half[2 * i + 1].ny = m->seg[i].ny;
  }
  free(nodes);
  m->q_far = 10; m->q_near = 16; m->q_sing = 16; m->q_log = 8;
  double htmin = t[1] - t[0];
  for (int a = 1; a < nt; ++a) if (t[a + 1] - t[a] < htmin) htmin = t[a + 1] - t[a];
  m->ell = sqrt(4.0 * htmin / alpha);
  return m;
}

void ora_mesh_free(ora_mesh* m) {
  if (!m) return;
  free(m->t); free(m->seg); free(m->half); free(m);
}

void ora_set_orders(ora_mesh* m, int q_far, int q_near, int q_sing, int q_log) {
  if (q_far >= 1 && q_far <= ORA_QMAX) m->q_far = q_far;
  if (q_near >= 1 && q_near <= ORA_QMAX) m->q_near = q_near;
  if (q_sing >= 1 && q_sing <= ORA_QMAX) m->q_sing = q_sing;
  if (q_log >= 1 && q_log <= ORA_QMAX) m->q_log = q_log;
}

int ora_mesh_ng(const ora_mesh* m) { return m->ng; }
/* segments: out[ng*8] = ax ay bx by h nx ny 0 */
void ora_mesh_segments(const ora_mesh* m, double* out) {
  for (int i = 0; i < m->ng; ++i) {
    const ora_seg* s = &m->seg[i];
    double v[8] = {s->ax, s->ay, s->bx, s->by, s->h, s->nx, s->ny, 0.0};
    memcpy(out + 8 * i, v, sizeof(v));
  }
}

/* ------------------------------------------------- segment-pair integral --- */
/* Integral over X x Y of Sx(x) Sy(y) * kernel, where the shape functions are
 * linear: Sx = sx0 at X's start, sx1 at X's end (same for Y).
 * rel: 0 = disjoint, 1 = identical, 2 = X.end == Y.start, 3 = X.start == Y.end. */
typedef struct { double sx0, sx1, sy0, sy1; } ora_shape;

static double lin(double v0, double v1, double f) { return v0 + (v1 - v0) * f; }

/* Composite rules (reading R24): U* varies on the length ell = sqrt(4 min h_t / alpha)
 * at the smallest lag; elements longer than ell are integrated with ns = ceil(h / ell) equal cells
 * per direction (a Gauss rule of the given order in each cell). */
static double pt_seg_dist(double px, double py, const ora_seg* S) {
  double dx = S->bx - S->ax, dy = S->by - S->ay;
  double f = ((px - S->ax) * dx + (py - S->ay) * dy) / (dx * dx + dy * dy);
  if (f < 0.0) f = 0.0;
  if (f > 1.0) f = 1.0;
  double qx = S->ax + f * dx - px, qy = S->ay + f * dy - py;
  return sqrt(qx * qx + qy * qy);
}
/* distance of two non-crossing segments: the smallest endpoint-to-segment distance */
static double seg_seg_dist(const ora_seg* X, const ora_seg* Y) {
  double d = pt_seg_dist(X->ax, X->ay, Y), e;
  if ((e = pt_seg_dist(X->bx, X->by, Y)) < d) d = e;
  if ((e = pt_seg_dist(Y->ax, Y->ay, X)) < d) d = e;
  if ((e = pt_seg_dist(Y->bx, Y->by, X)) < d) d = e;
  return d;
}
/* pairs farther apart than 8 ell keep the plain rule: U* there is below e^{-64} of its peak at
 * the smallest lag and varies on the scale of its distance at the larger ones */
static int ora_cells(const ora_mesh* m, const ora_seg* X, const ora_seg* Y) {
  double hm = X->h > Y->h ? X->h : Y->h;
  if (!(m->ell > 0.0) || hm <= m->ell || seg_seg_dist(X, Y) >= 8.0 * m->ell) return 1;
  int ns = (int)ceil(hm / m->ell);
  return ns > 24 ? 24 : ns;
}

/* near cells (d <= 1) of disjoint pairs closer than their length (reading R25): the true kernel
 * keeps its ln c and 1/c parts, which vary on the scale of the distance -- cells of that size */
static int ora_near_cells(const ora_seg* X, const ora_seg* Y) {
  double hm = X->h > Y->h ? X->h : Y->h, d = seg_seg_dist(X, Y);
  if (d >= hm) return 1;
  int ns = (int)ceil(2.0 * hm / d);
  return ns > 16 ? 16 : ns;
}

static double pair_disjoint(const ora_mesh* m, int ker, const ora_lags* L, const ora_seg* X,
                            const ora_seg* Y, const ora_shape* sh, int q) {
  const ora_rule* R = &RULES[q];
  int ns = ora_cells(m, X, Y);
  if (L->d <= 1) {
    int nn = ora_near_cells(X, Y);
    if (nn > ns) ns = nn;
  }
  double acc = 0.0;
  for (int p = 0; p < q * ns; ++p) {
    double fu = (p / q + R->x[p % q]) / ns, wu = R->w[p % q] / ns;
    double x0 = X->ax + fu * (X->bx - X->ax), x1 = X->ay + fu * (X->by - X->ay);
    double su = lin(sh->sx0, sh->sx1, fu);
    double inner = 0.0;
    for (int r = 0; r < q * ns; ++r) {
      double fv = (r / q + R->x[r % q]) / ns, wv = R->w[r % q] / ns;
      double y0 = Y->ax + fv * (Y->bx - Y->ax), y1 = Y->ay + fv * (Y->by - Y->ay);
      double dx = x0 - y0, dy = x1 - y1;
      double c = m->alpha * (dx * dx + dy * dy) / 4.0;
      double k = ker_direct(ker, L, m->alpha, c);
      if (ker == KER_Q) k *= dx * Y->nx + dy * Y->ny;
      inner += wv * lin(sh->sy0, sh->sy1, fv) * k;
    }
    acc += wu * su * inner;
  }
  return acc * X->h * Y->h;
}

/* identical segments: 1-D reduction in w = |u - v| */
static double pair_identical(const ora_mesh* m, int ker, const ora_lags* L, const ora_seg* X,
                             const ora_shape* sh) {
  if (ker == KER_Q) return 0.0;            /* (x-y).n_y = 0 on a straight segment */
  const double h = X->h, alpha = m->alpha;
  const ora_rule* Rr = &RULES[m->q_sing];
  const ora_rule* Rl = &RULES[m->q_log];
  const ora_rule* Rv = &RULES[4];
  /* G(w) = int_0^{h-w} [Sx(v+w) Sy(v) + Sx(v) Sy(v+w)] dv, shapes in arc length */
#define SHX(u) lin(sh->sx0, sh->sx1, (u) / h)
#define SHY(u) lin(sh->sy0, sh->sy1, (u) / h)
  /* composite in rho = w / h (R24): cell 0 = [0, 1/ns] with the split treatment below (rho = t/ns,
   * ln rho = ln t - ln ns), cells k >= 1 by plain Gauss with ln c evaluated */
  const int ns = ora_cells(m, X, X);
  const double lns = log((double)ns);
  double acc_reg = 0.0, acc_log = 0.0, acc_out = 0.0;
  for (int cell = 1; cell < ns; ++cell)
    for (int p = 0; p < Rr->n; ++p) {
      double w = h * (cell + Rr->x[p]) / ns, len = h - w, G = 0.0;
      for (int r = 0; r < Rv->n; ++r) {
        double v = len * Rv->x[r];
        G += Rv->w[r] * (SHX(v + w) * SHY(v) + SHX(v) * SHY(v + w));
      }
      G *= len;
      double c = alpha * w * w / 4.0, Rk, Pk;
      ker_split(ker, L, alpha, c, &Rk, &Pk);
      acc_out += Rr->w[p] / ns * G * (Rk + Pk * log(c));
    }
  for (int p = 0; p < Rr->n; ++p) {
    double w = h * Rr->x[p] / ns, len = h - w, G = 0.0;
    for (int r = 0; r < Rv->n; ++r) {
      double v = len * Rv->x[r];
      G += Rv->w[r] * (SHX(v + w) * SHY(v) + SHX(v) * SHY(v + w));
    }
    G *= len;
    double c = alpha * w * w / 4.0, Rk, Pk;
    ker_split(ker, L, alpha, c, &Rk, &Pk);
    acc_reg += Rr->w[p] / ns * G * (Rk + Pk * (log(alpha / 4.0) + 2.0 * log(h) - 2.0 * lns));
  }
  /* 2 int_0^1 P(c(h t/ns)) G(h t/ns) ln t dt / ns = -2 int int P G (h t tau / ns) / ns */
  for (int p = 0; p < Rl->n; ++p)
    for (int q = 0; q < Rl->n; ++q) {
      double w = h * Rl->x[p] * Rl->x[q] / ns, len = h - w, G = 0.0;
      for (int r = 0; r < Rv->n; ++r) {
        double v = len * Rv->x[r];
        G += Rv->w[r] * (SHX(v + w) * SHY(v) + SHX(v) * SHY(v + w));
      }
      G *= len;
      double c = alpha * w * w / 4.0, Rk, Pk;
      ker_split(ker, L, alpha, c, &Rk, &Pk);
      acc_log += Rl->w[p] * Rl->w[q] / ns * Pk * G;
    }
#undef SHX
#undef SHY
  return h * (acc_reg - 2.0 * acc_log + acc_out);
}

/* segments sharing one vertex V: x = V + u e1 (u in [0,h1]), y = V + v e2 (v in [0,h2]);
 * Duffy map on the two triangles of [0,1]^2 in (u/h1, v/h2). */
static double pair_vertex(const ora_mesh* m, int ker, const ora_lags* L, const ora_seg* X,
                          const ora_seg* Y, const ora_shape* sh, int rel) {
  const double alpha = m->alpha, h1 = X->h, h2 = Y->h;
  double e1x, e1y, e2x, e2y;
  /* shape values as functions of the distance from V */
  double sxV, sxF, syV, syF;   /* value at V and at the far end */
  if (rel == 2) {                /* X.end == Y.start == V */
    e1x = -X->tx; e1y = -X->ty; sxV = sh->sx1; sxF = sh->sx0;
    e2x = Y->tx; e2y = Y->ty; syV = sh->sy0; syF = sh->sy1;
  } else {                       /* X.start == Y.end == V */
    e1x = X->tx; e1y = X->ty; sxV = sh->sx0; sxF = sh->sx1;
    e2x = -Y->tx; e2y = -Y->ty; syV = sh->sy1; syF = sh->sy0;
  }
  double cth = e1x * e2x + e1y * e2y;
  double e1n = e1x * Y->nx + e1y * Y->ny;      /* (x-y).n_y = u e1.n_y  (e2 . n_y = 0) */
  if (ker == KER_Q && fabs(e1n) < 1e-14) return 0.0;   /* collinear: exactly 0 */
  const ora_rule* Rr = &RULES[m->q_sing];
  const ora_rule* Rl = &RULES[m->q_log];
  /* composite (R24): eta by plain Gauss in ns cells; rho in ns cells, cell 0 with the split
   * treatment (rho = t/ns), cells k >= 1 by plain Gauss with ln c evaluated */
  const int ns = ora_cells(m, X, Y);
  const double lns = log((double)ns);
  /* acute angle (cos > 1/2, reading R25): A(eta) dips to sin^2(theta) h^2 near eta* = cos(theta)
   * h1/h2 and its complex zeros approach [0,1]: eta in cells of width about sin(theta)/1.5 */
  int nea = 1;
  if (cth > 0.5) {
    double sth = sqrt(1.0 - cth * cth);
    nea = (int)ceil(1.5 / (sth > 1e-6 ? sth : 1e-6));
    if (nea > 16) nea = 16;
  }
  const int ne = ns * nea;
  double total = 0.0;
  for (int tri = 0; tri < 2; ++tri) {
    for (int ie = 0; ie < Rr->n * ne; ++ie) {
      double eta = (ie / Rr->n + Rr->x[ie % Rr->n]) / ne, weta = Rr->w[ie % Rr->n] / ne;
      /* r^2 = rho^2 A(eta) */
      double A = (tri == 0) ? (h1 * h1 + h2 * h2 * eta * eta - 2.0 * h1 * h2 * eta * cth)
                            : (h1 * h1 * eta * eta + h2 * h2 - 2.0 * h1 * h2 * eta * cth);
      double lnA = log(alpha * A / 4.0);
      double reg = 0.0, lg = 0.0, out = 0.0;
      for (int cell = 1; cell < ns; ++cell)
        for (int ir = 0; ir < Rr->n; ++ir) {
          double rho = (cell + Rr->x[ir]) / ns;
          double u = (tri == 0) ? h1 * rho : h1 * rho * eta;
          double v = (tri == 0) ? h2 * rho * eta : h2 * rho;
          double f = lin(sxV, sxF, u / h1) * lin(syV, syF, v / h2) * h1 * h2 * rho;
          double c = alpha * rho * rho * A / 4.0, Rk, Pk;
          ker_split(ker, L, alpha, c, &Rk, &Pk);
          if (ker == KER_Q) f *= u * e1n;
          out += Rr->w[ir] / ns * f * (Rk + Pk * log(c));
        }
      for (int ir = 0; ir < Rr->n; ++ir) {
        double rho = Rr->x[ir] / ns;
        double u = (tri == 0) ? h1 * rho : h1 * rho * eta;
        double v = (tri == 0) ? h2 * rho * eta : h2 * rho;
        double f = lin(sxV, sxF, u / h1) * lin(syV, syF, v / h2) * h1 * h2 * rho;
        double c = alpha * rho * rho * A / 4.0, Rk, Pk;
        ker_split(ker, L, alpha, c, &Rk, &Pk);
        if (ker == KER_Q) f *= u * e1n;
        reg += Rr->w[ir] / ns * f * (Rk + Pk * (lnA - 2.0 * lns));
      }
      for (int ir = 0; ir < Rl->n; ++ir)
        for (int it = 0; it < Rl->n; ++it) {
          double rho = Rl->x[ir] * Rl->x[it] / ns;
          double u = (tri == 0) ? h1 * rho : h1 * rho * eta;
          double v = (tri == 0) ? h2 * rho * eta : h2 * rho;
          double f = lin(sxV, sxF, u / h1) * lin(syV, syF, v / h2) * h1 * h2 * rho;
          double c = alpha * rho * rho * A / 4.0, Rk, Pk;
          ker_split(ker, L, alpha, c, &Rk, &Pk);
          if (ker == KER_Q) f *= u * e1n;
          lg += Rl->w[ir] * Rl->w[it] / ns * f * Pk;
        }
      total += weta * (reg - 2.0 * lg + out);
    }
  }
  return total;
}

/* relation of elements p, q of a closed chain of n elements */
static int chain_rel(int p, int q, int n) {
  if (p == q) return 1;
  if ((p + 1) % n == q) return 2;
  if ((q + 1) % n == p) return 3;
  return 0;
}

static double pair_integral(const ora_mesh* m, int ker, const ora_lags* L, const ora_seg* X,
                            const ora_seg* Y, const ora_shape* sh, int rel) {
  if (L->n == 0) return 0.0;
  if (rel == 0) return pair_disjoint(m, ker, L, X, Y, sh, (L->d <= 1) ? m->q_near : m->q_far);
  if (rel == 1) return pair_identical(m, ker, L, X, sh);
  return pair_vertex(m, ker, L, X, Y, sh, rel);
}

/* ---------------------------------------------------------------- entries --- */
/* V_h[(a,i),(b,j)], P:86 with the single-layer kernel (1/alpha) U* */
double ora_entry_V(const ora_mesh* m, int a, int i, int b, int j) {
  if (a < b) return 0.0;
  ora_lags L = make_lags(m->t, a, b);
  ora_shape one = {1.0, 1.0, 1.0, 1.0};
  return pair_integral(m, KER_H, &L, &m->seg[i], &m->seg[j], &one, chain_rel(i, j, m->ng));
}

/* K_h[(a,i),(b,n)], P:86 with (1/alpha) d_{n_y} U* (P:44); trial = primal hat at node n */
double ora_entry_K(const ora_mesh* m, int a, int i, int b, int n) {
  if (a < b) return 0.0;
  ora_lags L = make_lags(m->t, a, b);
  int ng = m->ng;
  int jl = (n - 1 + ng) % ng;           /* hat rises on gamma_{n-1}: 0 -> 1 */
  ora_shape up = {1.0, 1.0, 0.0, 1.0}, down = {1.0, 1.0, 1.0, 0.0};
  double v = pair_integral(m, KER_Q, &L, &m->seg[i], &m->seg[jl], &up, chain_rel(i, jl, ng));
  v += pair_integral(m, KER_Q, &L, &m->seg[i], &m->seg[n], &down, chain_rel(i, n, ng));
  return v;
}

/* dual hat psi_l on its four half segments (R6): index, end values, arc derivative */
static void dual_support(const ora_mesh* m, int l, int hp[4], double v0[4], double v1[4],
                         double dv[4]) {
  int ng = m->ng, nh = 2 * ng;
  double hm = m->seg[(l - 1 + ng) % ng].h, h0 = m->seg[l].h, hp1 = m->seg[(l + 1) % ng].h;
  double vm = hm / (hm + h0), vp = hp1 / (h0 + hp1);
  double Lm = 0.5 * (hm + h0), Lp = 0.5 * (h0 + hp1);
  hp[0] = (2 * l - 1 + nh) % nh; v0[0] = 0.0; v1[0] = vm;  dv[0] = 1.0 / Lm;
  hp[1] = 2 * l;                 v0[1] = vm;  v1[1] = 1.0; dv[1] = 1.0 / Lm;
  hp[2] = 2 * l + 1;             v0[2] = 1.0; v1[2] = vp;  dv[2] = -1.0 / Lp;
  hp[3] = (2 * l + 2) % nh;      v0[3] = vp;  v1[3] = 0.0; dv[3] = -1.0 / Lp;
}

/* D_h[(a,l),(b,k)] (Thm 1) in the integration-by-parts form (R7):
 *   int int psi_l'(x) psi_k'(y) sum eps H  +  int int (n_x.n_y) psi_l(x) psi_k(y) sum eps F */
double ora_entry_D(const ora_mesh* m, int a, int l, int b, int k) {
  if (a < b) return 0.0;
  ora_lags L = make_lags(m->t, a, b);
  int hl[4], hk[4];
  double l0[4], l1[4], ld[4], k0[4], k1[4], kd[4];
  dual_support(m, l, hl, l0, l1, ld);
  dual_support(m, k, hk, k0, k1, kd);
  int nh = 2 * m->ng;
  ora_shape one = {1.0, 1.0, 1.0, 1.0};
  double acc = 0.0;
  for (int p = 0; p < 4; ++p)
    for (int q = 0; q < 4; ++q) {
      const ora_seg* X = &m->half[hl[p]];
      const ora_seg* Y = &m->half[hk[q]];
      int rel = chain_rel(hl[p], hk[q], nh);
      double curl = pair_integral(m, KER_H, &L, X, Y, &one, rel);
      ora_shape sh = {l0[p], l1[p], k0[q], k1[q]};
      double nn = X->nx * Y->nx + X->ny * Y->ny;
      double nrm = (nn != 0.0) ? pair_integral(m, KER_F, &L, X, Y, &sh, rel) : 0.0;
      acc += ld[p] * kd[q] * curl + nn * nrm;
    }
  return acc;
}


/* single segment-pair integral, for the brute-force pins:
 * half = 0: primal segments p, q; half = 1: half segments p, q (indices 0..2ng-1);
 * ker 0 = H (V / D-curl), 1 = F (D-normal), 2 = Q (K, dot included);
 * linear shape values (sx0, sx1) on X = p, (sy0, sy1) on Y = q. */
double ora_pair(const ora_mesh* m, int ker, int half, int a, int b, int p, int q, double sx0,
                double sx1, double sy0, double sy1) {
  if (a < b) return 0.0;
  ora_lags L = make_lags(m->t, a, b);
  ora_shape sh = {sx0, sx1, sy0, sy1};
  const ora_seg* S = half ? m->half : m->seg;
  int n = half ? 2 * m->ng : m->ng;
  return pair_integral(m, ker, &L, &S[p], &S[q], &sh, chain_rel(p, q, n));
}

typedef double (*entry_fn)(const ora_mesh*, int, int, int, int);
static entry_fn pick(int kind) {
  return kind == 0 ? ora_entry_V : (kind == 1 ? ora_entry_K : ora_entry_D);
}

/* batch of entries by global (time-major) indices row = a*ng+i, col = b*ng+j */
void ora_entries(const ora_mesh* m, int kind, long long cnt, const long long* row,
                 const long long* col, double* out) {
  entry_fn f = pick(kind);
  int ng = m->ng;
#pragma omp parallel for schedule(dynamic, 16)
  for (long long e = 0; e < cnt; ++e)
    out[e] = f(m, (int)(row[e] / ng), (int)(row[e] % ng), (int)(col[e] / ng), (int)(col[e] % ng));
}

/* dense N x N (row-major), N = ng*nt */
void ora_dense(const ora_mesh* m, int kind, double* out) {
  entry_fn f = pick(kind);
  int ng = m->ng, nt = m->nt;
  long long N = (long long)ng * nt;
#pragma omp parallel for schedule(dynamic, 1)
  for (long long r = 0; r < N; ++r) {
    int a = (int)(r / ng), i = (int)(r % ng);
    for (long long cc = 0; cc < N; ++cc) {
      int b = (int)(cc / ng), j = (int)(cc % ng);
      out[r * N + cc] = (b <= a) ? f(m, a, i, b, j) : 0.0;
    }
  }
}

/* rows [r0, r0+nr) of the dense matrix, columns [0, N) */
void ora_dense_rows(const ora_mesh* m, int kind, long long r0, long long nr, double* out) {
  entry_fn f = pick(kind);
  int ng = m->ng, nt = m->nt;
  long long N = (long long)ng * nt;
#pragma omp parallel for schedule(dynamic, 1)
  for (long long rr = 0; rr < nr; ++rr) {
    long long r = r0 + rr;
    int a = (int)(r / ng), i = (int)(r % ng);
    for (long long cc = 0; cc < N; ++cc) {
      int b = (int)(cc / ng), j = (int)(cc % ng);
      out[rr * N + cc] = (b <= a) ? f(m, a, i, b, j) : 0.0;
    }
  }
}

int ora_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------ representation formula --- */
/* Row f2: the solution in Q by the representation formula (eq. 2) with
 * u0 = 0:   u(x,t) = (Vt w)(x,t) - (W g)(x,t)
 *   (Vt w)(x,t) = (1/alpha) int_Sigma U*(x-y, t-tau) w(y,tau) ds_y dtau
 *   (W g)(x,t)  = (1/alpha) int_Sigma d_{n_y} U*(x-y, t-tau) g(y,tau) ds_y dtau
 * w piecewise constant (element j, step b: w[b*ng + j]); g piecewise linear in space (nodal
 * values, hat phi_n) and constant in time on each step (g[b*ng + n]) -- the discrete spaces of
 * eq. (4).  Time integrals exact (U* of P:48-54, s = t - tau):
 *   int (1/alpha) U* dtau       = (1/(4 pi)) [E1(c/s_hi) - E1(c/s_lo)]
 *   int (1/alpha) d_ny U* dtau  = ((x-y).n_y / (2 pi r^2)) [exp(-c/s_hi) - exp(-c/s_lo)]
 * with c = alpha r^2/4, s_hi = t - t_b, s_lo = max(0, t - t_{b+1}) (terms with s_lo = 0 vanish).
 * Space: Gauss-Legendre with q points per element (the caller keeps the points away from Gamma).
 * pts[3k] = (x1, x2, t).  OpenMP over points. */
void ora_potential(const ora_mesh* m, const double* w, const double* g, long long npts,
                   const double* pts, int q, double* out) {
  init_rules();
  const ora_rule* R = &RULES[q];
  const int ng = m->ng, nt = m->nt;
  const double alpha = m->alpha;
#pragma omp parallel for schedule(dynamic, 1)
  for (long long k = 0; k < npts; ++k) {
    const double x1 = pts[3 * k], x2 = pts[3 * k + 1], t = pts[3 * k + 2];
    double vw = 0.0, wg = 0.0;
    for (int b = 0; b < nt && m->t[b] < t; ++b) {
      const double s_hi = t - m->t[b];
      const double s_lo = t - m->t[b + 1] > 0.0 ? t - m->t[b + 1] : 0.0;
      for (int j = 0; j < ng; ++j) {
        const ora_seg* S = &m->seg[j];
        const double g0 = g[(long long)b * ng + j], g1 = g[(long long)b * ng + (j + 1) % ng];
        double sv = 0.0, sw = 0.0;
        for (int u = 0; u < q; ++u) {
          const double f = R->x[u];
          const double y1 = S->ax + f * (S->bx - S->ax), y2 = S->ay + f * (S->by - S->ay);
          const double d1 = x1 - y1, d2 = x2 - y2;
          const double r2 = d1 * d1 + d2 * d2;
          const double c = 0.25 * alpha * r2;
          const double ev = ora_e1(c / s_hi) - (s_lo > 0.0 ? ora_e1(c / s_lo) : 0.0);
          const double ex = exp(-c / s_hi) - (s_lo > 0.0 ? exp(-c / s_lo) : 0.0);
          sv += R->w[u] * ev;
          sw += R->w[u] * (d1 * S->nx + d2 * S->ny) / r2 * ex * (g0 + f * (g1 - g0));
        }
        vw += S->h * w[(long long)b * ng + j] * sv / (4.0 * ORA_PI);
        wg += S->h * sw / (2.0 * ORA_PI);
      }
    }
    out[k] = vw - wg;
  }
}

/* ------------------------------------------------------ initial potential --- */
/* Row f1: M_h^0 u0 of eq. (4) for the paper's own experiment:
 *   f[(a,i)] = <M_0 u0_h, phi^0_(a,i)> = int_{t_a}^{t_{a+1}} int_{gamma_i} int_Omega U*(x-y,t) u0_h(y) dy ds_x dt,
 * u0_h in S_h^1(Omega_h) (nodal values on a triangulation).  Time integral exact:
 *   int_{t_a}^{t_{a+1}} U*(x-y,t) dt = (alpha/(4 pi)) [E1(c/t_{a+1}) - E1(c/t_a)],  E1(c/0) := 0.
 * Space: qx Gauss points on gamma_i; per triangle the collapsed (Duffy) tensor Gauss rule
 *   y = v0 + u (v1-v0) + v (v2-v0), u = xi (1-eta), v = xi eta, dy = 2|tau| xi dxi deta,
 * with qt_near^2 points when the distance from gamma_i to the triangle's centroid is below
 * 2 max(h_i, longest edge), else qt_far^2 (reading R22).  OpenMP over elements i. */
static double seg_point_dist(const ora_seg* S, double px, double py) {
  double f = (px - S->ax) * S->tx + (py - S->ay) * S->ty;
  if (f < 0.0) f = 0.0;
  if (f > S->h) f = S->h;
  double qx = S->ax + f * S->tx - px, qy = S->ay + f * S->ty - py;
  return sqrt(qx * qx + qy * qy);
}

/* integral of F over the triangle (A,B,C) split at the apex P into (P,A,B), (P,B,C), (P,C,A)
 * with signed areas (P inside, on an edge or outside), each by the collapsed rule with the apex
 * at P: y = P + xi [(1-eta)(V1-P) + eta (V2-P)], dy = 2 area xi dxi deta; xi on a geometric
 * composite Gauss rule (ratio 0.15, 10 levels, 8 points each) so that the log singularity of
 * E1(c/t_1) at y = P is resolved; eta by 12-point Gauss. */
static void apex_rule_accumulate(double px, double py, const double* V, const double* uv,
                                 double alpha, double t1, double wx, double* acc) {
  const ora_rule* RE = &RULES[12];
  const ora_rule* RR = &RULES[16];   /* 16 per geometric level: Bernstein ratio 2.26, 5e-12 (R22) */
  for (int s = 0; s < 3; ++s) {
    const double v1x = V[2 * s], v1y = V[2 * s + 1], v2x = V[2 * ((s + 1) % 3)], v2y = V[2 * ((s + 1) % 3) + 1];
    const double u1 = uv[s], u2 = uv[(s + 1) % 3];
    const double e1x = v1x - px, e1y = v1y - py, e2x = v2x - px, e2y = v2y - py;
    const double area2 = e1x * e2y - e1y * e2x;          /* signed */
    if (fabs(area2) < 1e-300) continue;
    /* eta rule along the far side v1 -> v2: the xi-integrated kernel behaves like log rho(eta),
     * rho = |y(1, eta) - p|, near-singular at an end where the apex sits close to that vertex
     * (x near a corner of the triangle, reading R22): grade eta geometrically (ratio 0.15, 8 points
     * per level) toward that end down to the scale |p - v| / |v1 - v2|; else 12 Gauss points */
    const double l1 = sqrt(e1x * e1x + e1y * e1y), l2 = sqrt(e2x * e2x + e2y * e2y);
    const double lside = sqrt((v2x - v1x) * (v2x - v1x) + (v2y - v1y) * (v2y - v1y));
    const double dmin = l1 < l2 ? l1 : l2;
    double es[128], ew[128];
    int ne = 0;
    if (dmin < 0.15 * lside) {
      const int at0 = l1 < l2;                     /* grade toward eta = 0 (v1) or eta = 1 (v2) */
      int nlev = (int)ceil(log(dmin / lside) / log(0.15)) + 1;
      if (nlev > 14) nlev = 14;
      double top = 1.0;
      for (int lev = 0; lev < nlev; ++lev) {
        const double bot = lev == nlev - 1 ? 0.0 : 0.15 * top;
        for (int q = 0; q < 8; ++q) {
          const double d = bot + (top - bot) * RULES[8].x[q];
          es[ne] = at0 ? d : 1.0 - d; ew[ne] = (top - bot) * RULES[8].w[q]; ++ne;
        }
        top = bot;
      }
    } else {
      for (int q = 0; q < RE->n; ++q) { es[ne] = RE->x[q]; ew[ne] = RE->w[q]; ++ne; }
    }
    double hi = 1.0;
    for (int lev = 0; lev <= 10; ++lev) {
      const double lo = lev < 10 ? hi * 0.15 : 0.0;
      for (int r = 0; r < RR->n; ++r) {
        const double xi = lo + (hi - lo) * RR->x[r], wxi = (hi - lo) * RR->w[r];
        for (int e = 0; e < ne; ++e) {
          const double eta = es[e];
          /* u0_h at y: the linear interpolant of the triangle's three values */
          const double uh = uv[3] * 0.0 + (1.0 - xi) * uv[4] + xi * ((1.0 - eta) * u1 + eta * u2);
          /* y - p formed directly: p - y would cancel to 0 where y is within rounding of p */
          const double dx = xi * ((1.0 - eta) * e1x + eta * e2x), dy = xi * ((1.0 - eta) * e1y + eta * e2y);
          const double c = 0.25 * alpha * (dx * dx + dy * dy);
          *acc += wx * area2 * xi * wxi * ew[e] * uh * ora_e1(c / t1);
        }
      }
      hi = lo;
    }
  }
}

void ora_initial_rhs(const ora_mesh* m, int nnode, const double* nodes, int ntri, const int* tri,
                     const double* u0, int qx, int qt_far, int qt_near, double* out) {
  init_rules();
  (void)nnode;
  const int ng = m->ng, nt = m->nt;
  const double alpha = m->alpha;
#pragma omp parallel for schedule(dynamic, 1)
  for (int i = 0; i < ng; ++i) {
    const ora_seg* S = &m->seg[i];
    double* node_sum = (double*)calloc((size_t)(nt + 1), sizeof(double));   /* N(i, n), regular rule */
    double first = 0.0;                                                       /* step a = 0 */
    /* x rule of the step-0 terms (reading R22): the step-0 column is log-singular in x where the
     * element meets a corner of Gamma (the data density jumps there), so a half of the element
     * that ends at a corner takes 8 geometrically graded levels (ratio 0.15 toward the corner,
     * the last level reaching it) of 8 Gauss points; other halves 16 Gauss points; an element
     * with no corner end keeps the plain qx-point rule */
    const ora_seg* Sp = &m->seg[(i + ng - 1) % ng];
    const ora_seg* Sn = &m->seg[(i + 1) % ng];
    const int c_a = S->tx * Sp->tx + S->ty * Sp->ty < 1.0 - 1e-12;   /* corner at the start a */
    const int c_b = S->tx * Sn->tx + S->ty * Sn->ty < 1.0 - 1e-12;   /* corner at the end b */
    double xs[160], xw[160];
    int nx0 = 0;
    if (!c_a && !c_b) {
      for (int p = 0; p < qx; ++p) { xs[nx0] = RULES[qx].x[p]; xw[nx0] = RULES[qx].w[p]; ++nx0; }
    } else {
      for (int half = 0; half < 2; ++half) {
        const int graded = half == 0 ? c_a : c_b;
        /* d = distance from the half's element end (0 at the corner end) in [0, 1/2] */
        if (!graded) {
          for (int p = 0; p < 16; ++p) {
            const double d = 0.5 * RULES[16].x[p];
            xs[nx0] = half == 0 ? d : 1.0 - d; xw[nx0] = 0.5 * RULES[16].w[p]; ++nx0;
          }
        } else {
          double top = 0.5;
          for (int lev = 0; lev < 8; ++lev) {
            const double bot = lev == 7 ? 0.0 : 0.15 * top;
            for (int p = 0; p < 8; ++p) {
              const double d = bot + (top - bot) * RULES[8].x[p];
              xs[nx0] = half == 0 ? d : 1.0 - d; xw[nx0] = (top - bot) * RULES[8].w[p]; ++nx0;
            }
            top = bot;
          }
        }
      }
    }
    for (int k = 0; k < ntri; ++k) {
      const int i0 = tri[3 * k], i1 = tri[3 * k + 1], i2 = tri[3 * k + 2];
      const double ax = nodes[2 * i0], ay = nodes[2 * i0 + 1];
      const double e1x = nodes[2 * i1] - ax, e1y = nodes[2 * i1 + 1] - ay;
      const double e2x = nodes[2 * i2] - ax, e2y = nodes[2 * i2 + 1] - ay;
      const double area2 = fabs(e1x * e2y - e1y * e2x);
      const double gx = ax + (e1x + e2x) / 3.0, gy = ay + (e1y + e2y) / 3.0;
      double le = sqrt(e1x * e1x + e1y * e1y);
      double l2 = sqrt(e2x * e2x + e2y * e2y), l3 = sqrt((e2x - e1x) * (e2x - e1x) + (e2y - e1y) * (e2y - e1y));
      if (l2 > le) le = l2;
      if (l3 > le) le = l3;
      const double hm = S->h > le ? S->h : le;
      const int near = seg_point_dist(S, gx, gy) < 2.0 * hm;
      const int qt = near ? qt_near : qt_far;
      const ora_rule* RT = &RULES[qt];
      const ora_rule* RX = &RULES[qx];
      for (int p = 0; p < qx; ++p) {
        const double xx = S->ax + RX->x[p] * (S->bx - S->ax), xy = S->ay + RX->x[p] * (S->by - S->ay);
        for (int a1 = 0; a1 < qt; ++a1)
          for (int a2 = 0; a2 < qt; ++a2) {
            const double xi = RT->x[a1], eta = RT->x[a2];
            const double u = xi * (1.0 - eta), v = xi * eta;
            const double yx = ax + u * e1x + v * e2x, yy = ay + u * e1y + v * e2y;
            const double uh = (1.0 - u - v) * u0[i0] + u * u0[i1] + v * u0[i2];
            const double W = RX->w[p] * S->h * area2 * xi * RT->w[a1] * RT->w[a2] * uh;
            const double dx = xx - yx, dy = xy - yy;
            const double c = 0.25 * alpha * (dx * dx + dy * dy);
            for (int n = 1; n <= nt; ++n) node_sum[n] += W * ora_e1(c / m->t[n]);
          }
      }
      /* far triangles: the step-0 term is smooth in x (Gauss qx on gamma_i, corner or not); near
       * ones: the apex split at every point of the x rule above */
      const int npx = near ? nx0 : qx;
      for (int p = 0; p < npx; ++p) {
        const double xp = near ? xs[p] : RX->x[p], wxp = near ? xw[p] : RX->w[p];
        const double xx = S->ax + xp * (S->bx - S->ax), xy = S->ay + xp * (S->by - S->ay);
        double first_p = 0.0;
        if (!near) {
          /* step 0 alone (no difference of two nodes): E1(c/t_1) varies on ell_1 = sqrt(4 t_1 /
           * alpha); triangles longer than that by composite collapsed rules of ceil(2 l / ell_1)
           * cells per direction (reading R24) */
          const double ell1 = sqrt(4.0 * m->t[1] / alpha);
          int ns = (int)ceil(2.0 * le / ell1);
          if (ns < 1) ns = 1;
          if (ns > 24) ns = 24;
          for (int a1 = 0; a1 < qt * ns; ++a1)
            for (int a2 = 0; a2 < qt * ns; ++a2) {
              const double xi = (a1 / qt + RT->x[a1 % qt]) / ns, eta = (a2 / qt + RT->x[a2 % qt]) / ns;
              const double u = xi * (1.0 - eta), v = xi * eta;
              const double yx = ax + u * e1x + v * e2x, yy = ay + u * e1y + v * e2y;
              const double uh = (1.0 - u - v) * u0[i0] + u * u0[i1] + v * u0[i2];
              const double W = wxp * S->h * area2 * xi * RT->w[a1 % qt] * RT->w[a2 % qt] / ((double)ns * ns) * uh;
              const double dx = xx - yx, dy = xy - yy;
              first_p += W * ora_e1(0.25 * alpha * (dx * dx + dy * dy) / m->t[1]);
            }
        }
        if (near) {
          /* step 0 kernel E1(c/t_1) is log singular at y = x: apex-split rule at x */
          const double V[6] = {ax, ay, ax + e1x, ay + e1y, ax + e2x, ay + e2y};
          /* uv[0..2] vertex values, uv[4] = value at the apex x (linear extension) */
          const double det = e1x * e2y - e1y * e2x;
          const double uu = ((xx - ax) * e2y - (xy - ay) * e2x) / det, vv = ((xy - ay) * e1x - (xx - ax) * e1y) / det;
          const double uv[5] = {u0[i0], u0[i1], u0[i2], 0.0, (1.0 - uu - vv) * u0[i0] + uu * u0[i1] + vv * u0[i2]};
          apex_rule_accumulate(xx, xy, V, uv, alpha, m->t[1], wxp * S->h, &first_p);
        }
        first += first_p;
      }
    }
    out[i] = alpha / (4.0 * ORA_PI) * first;
    for (int a = 1; a < nt; ++a)
      out[(long long)a * ng + i] = alpha / (4.0 * ORA_PI) * (node_sum[a + 1] - node_sum[a]);
    free(node_sum);
  }
}


/* ------------------------------------------- initial potential in Q (row f2) --- */
/* (M~_0 u0)(x, t) = int_Omega U*(x - y, t) u0_h(y) dy (eq. 2), U*(z, t) =
 * alpha / (4 pi t) exp(-alpha |z|^2 / (4 t)), u0_h linear on each triangle.  Every
 * triangle V0 + u e1 + v e2 by the collapsed map u = xi (1 - eta), v = xi eta (Jacobian xi)
 * with q x q Gauss points on each of ns x ns equal cells of [0,1]^2, ns = ceil(2 l / ell),
 * l = longest edge, ell = sqrt(4 t / alpha) (the Gaussian's width; reading R24).  No
 * truncation.  out[k] = value at pts[k] = (x1, x2, t), t > 0. */
void ora_potential_initial(const ora_mesh* m, int nnode, const double* nodes, int ntri, const int* tri,
                           const double* u0, long long npts, const double* pts, int q, double* out) {
  (void)nnode;
  init_rules();
  const ora_rule* R = &RULES[q];
  const double alpha = m->alpha;
#pragma omp parallel for schedule(dynamic)
  for (long long k = 0; k < npts; ++k) {
    const double x1 = pts[3 * k], x2 = pts[3 * k + 1], t = pts[3 * k + 2];
    const double ell = sqrt(4.0 * t / alpha), pref = alpha / (4.0 * ORA_PI * t);
    double acc = 0.0;
    for (int e = 0; e < ntri; ++e) {
      const int i0 = tri[3 * e], i1 = tri[3 * e + 1], i2 = tri[3 * e + 2];
      const double ax = nodes[2 * i0], ay = nodes[2 * i0 + 1];
      const double e1x = nodes[2 * i1] - ax, e1y = nodes[2 * i1 + 1] - ay;
      const double e2x = nodes[2 * i2] - ax, e2y = nodes[2 * i2 + 1] - ay;
      const double area2 = fabs(e1x * e2y - e1y * e2x);
      double l = sqrt(e1x * e1x + e1y * e1y);
      double l2 = sqrt(e2x * e2x + e2y * e2y), l3 = sqrt((e2x - e1x) * (e2x - e1x) + (e2y - e1y) * (e2y - e1y));
      if (l2 > l) l = l2;
      if (l3 > l) l = l3;
      int ns = (int)ceil(2.0 * l / ell);
      if (ns < 1) ns = 1;
      double tri_sum = 0.0;
      for (int cx = 0; cx < ns; ++cx)
        for (int a1 = 0; a1 < q; ++a1) {
          const double xi = (cx + R->x[a1]) / ns;
          for (int cy = 0; cy < ns; ++cy)
            for (int a2 = 0; a2 < q; ++a2) {
              const double eta = (cy + R->x[a2]) / ns;
              const double u = xi * (1.0 - eta), v = xi * eta;
              const double yx = ax + u * e1x + v * e2x, yy = ay + u * e1y + v * e2y;
              const double uh = (1.0 - u - v) * u0[i0] + u * u0[i1] + v * u0[i2];
              const double dx = x1 - yx, dy = x2 - yy;
              tri_sum += R->w[a1] * R->w[a2] / ((double)ns * ns) * xi * uh *
                         exp(-alpha * (dx * dx + dy * dy) / (4.0 * t));
            }
        }
      acc += area2 * tri_sum;
    }
    out[k] = pref * acc;
  }
}
