"""Brute-force mpmath references that PIN the oracle (test infrastructure only).

Nothing here reuses the oracle's quadrature, E1, kernel split or Gauss rules:
E1 is mpmath's, the time kernels are the closed forms H, F, Q written again
from their definitions, and the space integrals are mpmath tanh-sinh
quadratures of the full (singular) integrands, iterated over the segment pair
(for identical segments through the exact 1-D reduction
int int f(|u-v|) S(u,v) = int_0^h f(w) G(w) dw, G(w) = int_0^{h-w} [Sx(v+w)Sy(v)+Sx(v)Sy(v+w)] dv).

Also: the closed-form right-hand sides of the two row-sum identities
  K 1 = M_0 1 - 1/2                      (eq. 2/3 with u = 1)
  D 1 = int_Gamma (n_x.n_y) U* ds_y      (D = -d_n W, with u = 1)
on the unit square, integrated over one test element by mpmath.
"""
import mpmath as mp

mp.mp.dps = 20


# ------------------------------------------------------------- time kernels
def H(alpha, r2, s):
    """double time antiderivative of (1/alpha) U* (0 for s <= 0)"""
    if s <= 0:
        return mp.mpf(0)
    c = mp.mpf(alpha) * r2 / 4
    x = c / s
    return ((s + c) * mp.e1(x) - s * mp.exp(-x)) / (4 * mp.pi)


def F(alpha, r2, s):
    """first time antiderivative of U*"""
    if s <= 0:
        return mp.mpf(0)
    return mp.mpf(alpha) * mp.e1(mp.mpf(alpha) * r2 / (4 * s)) / (4 * mp.pi)


def Q(alpha, r2, s):
    """double time antiderivative of (1/alpha) d_ny U*, divided by (x-y).n_y"""
    if s <= 0:
        return mp.mpf(0)
    c = mp.mpf(alpha) * r2 / 4
    x = c / s
    return mp.mpf(alpha) / (8 * mp.pi) * (mp.exp(-x) / x - mp.e1(x))


KER = {0: H, 1: F, 2: Q}


def lags(t, a, b):
    t = [mp.mpf(v) for v in t]
    s = [t[a + 1] - t[b], t[a] - t[b], t[a + 1] - t[b + 1], t[a] - t[b + 1]]
    return list(zip(s, [1, -1, -1, 1]))


def kernel_sum(ker, alpha, r2, L):
    f = KER[ker]
    return mp.fsum(e * f(alpha, r2, s) for s, e in L if s > 0)


# ------------------------------------------------------------ pair integral
def pair(ker, alpha, t, a, b, X, Y, nY, sx=(1, 1), sy=(1, 1), rel=0):
    """int_X int_Y Sx Sy kernel; X, Y = ((ax, ay), (bx, by)); rel 0 disjoint, 1 identical,
    2 X.end == Y.start, 3 X.start == Y.end."""
    L = lags(t, a, b)
    ax, ay = map(mp.mpf, X[0])
    bx, by = map(mp.mpf, X[1])
    cx, cy = map(mp.mpf, Y[0])
    dx, dy = map(mp.mpf, Y[1])
    hX = mp.sqrt((bx - ax) ** 2 + (by - ay) ** 2)
    hY = mp.sqrt((dx - cx) ** 2 + (dy - cy) ** 2)
    nx, ny = map(mp.mpf, nY)

    def Sx(f):
        return sx[0] + (sx[1] - sx[0]) * f

    def Sy(f):
        return sy[0] + (sy[1] - sy[0]) * f

    def integrand(fu, fv):
        x0, x1 = ax + fu * (bx - ax), ay + fu * (by - ay)
        y0, y1 = cx + fv * (dx - cx), cy + fv * (dy - cy)
        r2 = (x0 - y0) ** 2 + (x1 - y1) ** 2
        k = kernel_sum(ker, alpha, r2, L)
        if ker == 2:
            k *= (x0 - y0) * nx + (x1 - y1) * ny
        return Sx(fu) * Sy(fv) * k

    if rel == 1:
        if ker == 2:
            return mp.mpf(0)
        h = hX

        def G(w):
            return mp.quad(lambda v: Sx((v + w) / h) * Sy(v / h) + Sx(v / h) * Sy((v + w) / h),
                           [0, h - w], method="gauss-legendre")

        return mp.quad(lambda w: kernel_sum(ker, alpha, w * w, L) * G(w), [0, h])
    if rel in (2, 3):
        # singular corner at fu = 1 (rel 2) or fu = 0 (rel 3) and the matching fv end
        def inner(fu):
            return mp.quad(lambda fv: integrand(fu, fv), [0, 1])

        return hX * hY * mp.quad(inner, [0, 1])
    return hX * hY * mp.quad(lambda fu: mp.quad(lambda fv: integrand(fu, fv), [0, 1]), [0, 1])


# ----------------------------------------------------- row-sum identities
def _erf_int(k, x0, x1, c):
    """int_{x0}^{x1} erf(k (x - c)) dx (closed form)"""
    def A(x):
        z = k * (x - c)
        return (x - c) * mp.erf(z) + mp.exp(-z * z) / (k * mp.sqrt(mp.pi))
    return A(x1) - A(x0)


def K_rowsum_unit_square(alpha, t0, t1, s0, s1):
    """int_{t0}^{t1} int_{side y=0, x in [s0,s1]} (M_0 1 - 1/2) dx dt on the unit square.
    M_0 1 (x,t) = prod_d 1/2 [erf(x_d k) - erf((x_d - 1) k)], k = sqrt(alpha/(4t)); x_2 = 0."""
    alpha = mp.mpf(alpha)

    def f(t):
        k = mp.sqrt(alpha / (4 * t))
        fy = mp.erf(k) / 2                              # x_2 = 0
        fx = (_erf_int(k, s0, s1, 0) - _erf_int(k, s0, s1, 1)) / 2
        return fx * fy
    return mp.quad(f, [t0, t1]) - mp.mpf(1) / 2 * (s1 - s0) * (t1 - t0)


def D_rowsum_unit_square(alpha, t0, t1, pieces):
    """int_{t0}^{t1} int psi(x) [int_Gamma (n_x.n_y) U*(x-y,t) ds_y] ds_x dt on the unit square,
    for a psi given as linear pieces on the side y=0: pieces = [(x0, x1, v0, v1)], and pieces on
    the side x=0 (n=(-1,0)) given as ('L', y0, y1, v0, v1)."""
    alpha = mp.mpf(alpha)

    def side_term(u, t):
        # x at arc position u in [0,1] along a side of the square; same side (n.n = 1) and the
        # opposite side at distance 1 (n.n = -1); the two perpendicular sides give n.n = 0.
        k = mp.sqrt(alpha / (4 * t))
        line = mp.sqrt(mp.pi) / (2 * k) * (mp.erf(k * (1 - u)) + mp.erf(k * u))
        return alpha / (4 * mp.pi * t) * line * (1 - mp.exp(-k * k))

    total = mp.mpf(0)
    for pc in pieces:
        if pc[0] == 'L':
            _, y0, y1, v0, v1 = pc
            x0, x1 = y0, y1
        else:
            x0, x1, v0, v1 = pc
        x0, x1, v0, v1 = map(mp.mpf, (x0, x1, v0, v1))

        lo, hi = min(x0, x1), max(x0, x1)

        def g(t, x0=x0, x1=x1, v0=v0, v1=v1, lo=lo, hi=hi):
            return mp.quad(lambda u: (v0 + (v1 - v0) * (u - x0) / (x1 - x0)) * side_term(u, t),
                           [lo, hi])
        total += mp.quad(g, [t0, t1])
    return total
