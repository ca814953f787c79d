"""Pins of the CPU oracle against what the paper and the mathematics fix.

Every test here is independent of the oracle's own quadrature: closed forms,
mpmath brute force (oracle/brute.py), exact identities of the boundary
integral equations, Laplace steady limits, direct solves.
A plausible mistake in the oracle (a dropped term, a wrong sign, a wrong power
of alpha, a transposed operand, a wrong dual-hat value) fails at least one.
"""
import math

import mpmath as mp
import numpy as np
import pytest

import workloads as W
from oracle import brute as B
from oracle import oracle as O
from workloads.configs import Workload


@pytest.fixture(scope="module")
def c1():
    w = W.get("C1")
    return w, O.OracleMesh(w)


_DENSE = {}


def dense_c1(m, kind):
    """C1 matrices are computed once per session"""
    if kind not in _DENSE:
        _DENSE[kind] = m.dense(kind)
    return _DENSE[kind]


# ----------------------------------------------------------------- P1: U*
def test_ustar_closed_form():
    L = O.lib()
    # SPEC S:136-138 (closed-form instances of P:48-54)
    assert L.ora_ustar(10.0, 0.0, 1.0) == pytest.approx(10 / (4 * math.pi), rel=1e-15)
    assert L.ora_ustar(10.0, 1.0, 0.0) == 0.0
    assert L.ora_ustar(1.0, 4.0, 1.0) == pytest.approx(math.exp(-1) / (4 * math.pi), rel=1e-15)
    assert L.ora_ustar(1.0, 4.0, -1.0) == 0.0
    # d_{n_y} U* at alpha=1, x-y=(1,0), n_y=(1,0), s=1: e^{-1/4}/(8 pi) = 0.0309874986 (SPEC S:147 erratum)
    assert L.ora_ustar_dny(1.0, 1.0, 1.0, 1.0) == pytest.approx(0.0309874986, rel=1e-9)
    assert L.ora_ustar_dny(1.0, 1.0, 1.0, 1.0) == pytest.approx(math.exp(-0.25) / (8 * math.pi), rel=1e-15)
    # finite-difference consistency of d/dn_y: U*(x - (y + eps n)) derivative in eps
    alpha, x, y, n, s = 0.7, np.array([0.3, -0.2]), np.array([0.1, 0.25]), np.array([0.6, 0.8]), 0.37
    f = lambda e: L.ora_ustar(alpha, float(np.sum((x - y - e * n) ** 2)), s)
    fd = (f(1e-5) - f(-1e-5)) / 2e-5
    an = L.ora_ustar_dny(alpha, float(np.dot(x - y, n)), float(np.sum((x - y) ** 2)), s)
    assert fd == pytest.approx(an, rel=1e-8)


def test_ustar_normalisation():
    # int_{R^2} U*(z, t) dz = 1 (SPEC S:181 erratum), polar quadrature
    L = O.lib()
    for alpha, t in [(0.7, 0.3), (10.0, 2.0)]:
        v = mp.quad(lambda r: 2 * mp.pi * r * L.ora_ustar(alpha, float(r * r), t), [0, 1, 10, mp.inf])
        assert float(v) == pytest.approx(1.0, abs=1e-12)


# ----------------------------------------------------------------- P3: E1
def test_e1_against_mpmath():
    xs = np.concatenate([np.logspace(-14, 0, 60), np.linspace(1.0, 60.0, 120), [100.0, 300.0, 700.0]])
    for x in xs:
        ref = mp.e1(mp.mpf(x))
        assert abs(O.e1(x) - ref) <= 3e-15 * ref, x
    assert O.e1(1.0) == pytest.approx(0.21938393439552027, rel=1e-15)
    x = 1e-12
    assert abs(O.e1(x) + math.log(x) + 0.5772156649015329) < 1e-11


# ---------------------------------------------------- P2: time antiderivatives
@pytest.mark.parametrize("alpha,r2", [(0.7, 0.09), (1.0, 1e-4), (10.0, 0.5)])
def test_time_antiderivatives(alpha, r2):
    """H'' = (1/alpha) U*, F' = U*, Q'' = (1/alpha) d_ny U* / dot, with H, F, Q -> 0 at s -> 0"""
    L = O.lib()
    us = lambda s: mp.mpf(alpha) / (4 * mp.pi * s) * mp.exp(-mp.mpf(alpha) * r2 / (4 * s))
    for s in (0.05, 0.37, 2.0):
        Fs = mp.quad(us, [0, s])
        assert L.ora_F(alpha, r2, s) == pytest.approx(float(Fs), rel=1e-13)
        Hs = mp.quad(lambda v: (s - v) * us(v) / alpha, [0, s])         # double antiderivative
        assert L.ora_H(alpha, r2, s) == pytest.approx(float(Hs), rel=1e-13)
        dn = lambda v: mp.mpf(alpha) ** 2 / (8 * mp.pi * v * v) * mp.exp(-mp.mpf(alpha) * r2 / (4 * v))
        Qs = mp.quad(lambda v: (s - v) * dn(v) / alpha, [0, s])
        assert L.ora_Q(alpha, r2, s) == pytest.approx(float(Qs), rel=1e-13)


# ------------------------------------------- P4: entries vs mpmath brute force
BF_CASES = [
    # ker, a, b, p, q, rel, sx, sy      (C1 geometry: 4 segments per side, h = 1/4, h_t = 1/16)
    (0, 0, 0, 1, 1, 1, (1, 1), (1, 1)),      # V identical, d = 0 (log r)
    (0, 1, 0, 1, 1, 1, (1, 1), (1, 1)),      # V identical, d = 1 (r^2 log r)
    (0, 4, 1, 1, 1, 1, (1, 1), (1, 1)),      # V identical, d = 3
    (0, 0, 0, 3, 4, 2, (1, 1), (1, 1)),      # V corner (1,0), d = 0
    (0, 1, 0, 3, 4, 2, (1, 1), (1, 1)),      # V corner, d = 1
    (0, 0, 0, 1, 2, 2, (1, 1), (1, 1)),      # V collinear neighbours
    (0, 0, 0, 1, 3, 0, (1, 1), (1, 1)),      # V gap 1, d = 0
    (2, 0, 0, 3, 4, 2, (1, 1), (1, 0)),      # K corner, falling hat, d = 0 (dot/r^2)
    (2, 1, 0, 3, 4, 2, (1, 1), (0, 1)),      # K corner, rising hat, d = 1
    (2, 0, 0, 4, 3, 3, (1, 1), (1, 0)),      # K corner, other orientation
    (2, 0, 0, 2, 5, 0, (1, 1), (1, 0)),      # K near, d = 0
    (1, 0, 0, 2, 2, 1, (0.5, 1), (1, 0.5)),  # F identical, linear shapes
    (1, 1, 0, 3, 4, 2, (1, 0.5), (0.5, 0)),  # F corner, d = 1
]


@pytest.mark.parametrize("case", BF_CASES)
def test_pair_integrals_brute_force(c1, case):
    w, m = c1
    ker, a, b, p, q, rel, sx, sy = case
    X = (tuple(m.seg_a[p]), tuple(m.seg_b[p]))
    Y = (tuple(m.seg_a[q]), tuple(m.seg_b[q]))
    ref = float(B.pair(ker, w.alpha, w.t_breaks, a, b, X, Y, m.seg_n[q], sx, sy, rel))
    got = m.pair(ker, 0, a, b, p, q, sx, sy)
    assert got == pytest.approx(ref, rel=1e-12, abs=1e-18)


# large kappa = alpha h^2 / (4 min h_t) (here 44): U* varies on ell = sqrt(4 min h_t / alpha) =
# h / 6.7, the composite rules of DESIGN.md reading R24 resolve it (touching pairs near the
# singularity, the identical pair in a bulk cell, a 2-D integrand at the corner)
LK_CASES = [
    # ker, a, b, p, q, rel, sx, sy
    (0, 1, 0, 2, 1, 3, (1, 1), (1, 1)),      # V vertex pair at the corner (1,0), d = 1
    (0, 2, 0, 2, 2, 1, (1, 1), (1, 1)),      # V identical, bulk cell d = 2
    (2, 1, 0, 2, 3, 2, (1, 1), (1, 0)),      # K vertex pair, falling hat, d = 1
    (1, 1, 0, 4, 4, 1, (0.5, 1), (1, 0.5)),  # F identical, linear shapes
]


@pytest.mark.parametrize("case", LK_CASES)
def test_large_kappa_pair_integrals_brute_force(case):
    from workloads.edge import edge_workloads
    w = edge_workloads()["alpha_large"]
    m = O.OracleMesh(w)
    ker, a, b, p, q, rel, sx, sy = case
    X = (tuple(m.seg_a[p]), tuple(m.seg_b[p]))
    Y = (tuple(m.seg_a[q]), tuple(m.seg_b[q]))
    ref = float(B.pair(ker, w.alpha, w.t_breaks, a, b, X, Y, m.seg_n[q], sx, sy, rel))
    got = m.pair(ker, 0, a, b, p, q, sx, sy)
    assert got == pytest.approx(ref, rel=1e-11, abs=1e-18)


# large kappa, far pair (reading R24): pairs farther apart than 8 ell keep the plain Gauss rule
# (no composite cells; U* at the smallest lag is below e^{-64} of its peak there).  Segments 1 and
# 4 of alpha_large are sqrt(2)/3 = 9.4 ell apart; every lag d = 0 .. 7, the V, F and K kernels.
FAR_CASES = [(ker, a) for ker in (0, 1, 2) for a in range(8)]


@pytest.mark.parametrize("case", FAR_CASES)
def test_large_kappa_far_pair_cutoff_brute_force(case):
    from workloads.edge import edge_workloads
    w = edge_workloads()["alpha_large"]
    m = O.OracleMesh(w)
    ker, a = case
    p, q = 1, 4
    ell = np.sqrt(4 * (w.t_breaks[1] - w.t_breaks[0]) / w.alpha)
    gap = np.hypot(m.seg_a[q][0] - m.seg_b[p][0], m.seg_a[q][1] - m.seg_b[p][1])
    assert 8 * ell < gap < 10 * ell                  # the pair sits just beyond the cutoff
    sy = (1, 0) if ker == 2 else (1, 1)
    X = (tuple(m.seg_a[p]), tuple(m.seg_b[p]))
    Y = (tuple(m.seg_a[q]), tuple(m.seg_b[q]))
    ref = float(B.pair(ker, w.alpha, w.t_breaks, a, 0, X, Y, m.seg_n[q], (1, 1), sy, 0))
    got = m.pair(ker, 0, a, 0, p, q, (1, 1), sy)
    # scale of the matrix: the identical pair of the same kernel at d = 0 (the max-norm entries)
    scale = abs(m.pair(ker if ker != 2 else 0, 0, 0, 0, p, p, (1, 1), (1, 1)))
    assert abs(got - ref) <= 1e-11 * abs(ref) + 1e-14 * scale, (got, ref, scale)


# acute corner (about 25 degrees, reading R25): the vertex pair's Duffy integrand and the near
# cell of the second neighbour across the corner (distance 0.4 h), K kernel, d = 0
AC_CASES = [
    (2, 2, 2, 4, 3, 3, (1, 1), (1.0, 0.0)),     # K vertex pair at the acute corner, d = 0
    (2, 2, 2, 4, 2, 0, (1, 1), (0.0, 1.0)),     # K disjoint pair across the corner, d = 0
]


@pytest.mark.parametrize("case", AC_CASES)
def test_acute_corner_pair_integrals_brute_force(case):
    from workloads.edge import edge_workloads
    w = edge_workloads()["acute"]
    m = O.OracleMesh(w)
    ker, a, b, p, q, rel, sx, sy = case
    X = (tuple(m.seg_a[p]), tuple(m.seg_b[p]))
    Y = (tuple(m.seg_a[q]), tuple(m.seg_b[q]))
    ref = float(B.pair(ker, w.alpha, w.t_breaks, a, b, X, Y, m.seg_n[q], sx, sy, rel))
    got = m.pair(ker, 0, a, b, p, q, sx, sy)
    assert got == pytest.approx(ref, rel=1e-12, abs=1e-18)


def test_half_segment_pairs_brute_force():
    """half segments on the L-shape (re-entrant corner, graded steps, alpha = 1/2)"""
    w = W.get("LT")
    m = O.OracleMesh(w)
    half = []
    for i in range(m.ng):
        a, b = m.seg_a[i], m.seg_b[i]
        mid = 0.5 * (a + b)
        half += [(tuple(a), tuple(mid)), (tuple(mid), tuple(b))]
    nrm = np.repeat(m.seg_n, 2, axis=0)
    # re-entrant corner (0.5,0.5) is node 8 (4+2+2): half 15 ends there, half 16 starts there
    cases = [(0, 0, 0, 15, 16, 2, (1, 1), (1, 1)), (1, 0, 0, 20, 20, 1, (0.5, 1), (1, 0.5)),
             (1, 1, 0, 15, 16, 2, (0, 1), (1, 0)), (0, 2, 1, 20, 21, 2, (1, 1), (1, 1)),
             (1, 3, 3, 5, 8, 0, (1, 0), (0, 1))]
    for ker, a, b, p, q, rel, sx, sy in cases:
        ref = float(B.pair(ker, w.alpha, w.t_breaks, a, b, half[p], half[q], nrm[q], sx, sy, rel))
        got = m.pair(ker, 1, a, b, p, q, sx, sy)
        assert got == pytest.approx(ref, rel=1e-12, abs=1e-18), (ker, a, b, p, q)


# --------------------------------------------------------- P5: V_h structure
def test_V_structure(c1):
    w, m = c1
    V = dense_c1(m, "V")
    ng, nt = m.ng, m.nt
    for a in range(nt):
        for b in range(nt):
            blk = V[a * ng:(a + 1) * ng, b * ng:(b + 1) * ng]
            if b > a:
                assert np.all(blk == 0.0)                          # causality, bitwise
            else:
                assert np.all(blk > 0.0)                           # U* > 0
                assert np.abs(blk - blk.T).max() <= 1e-15 * np.abs(blk).max()
                ref = V[(a - b) * ng:(a - b + 1) * ng, :ng]          # Toeplitz in the lag
                assert np.abs(blk - ref).max() <= 1e-13 * np.abs(ref).max()
    ev = np.linalg.eigvalsh(0.5 * (V + V.T))
    assert ev[0] > 0.0                                              # P:92-93 positive definite
    assert np.abs(V - V.T).max() > 1e-6                             # but not symmetric


def _circle(nseg, alpha):
    th = 2 * np.pi * np.arange(nseg) / nseg
    return Workload(name="circle", vertices=list(zip(np.cos(th), np.sin(th))),
                    segments_per_side=[1] * nseg, t_breaks=np.array([0.0, 1e6]), alpha=alpha,
                    x_star=(2.0, 2.0), tol=1e-10)


@pytest.mark.parametrize("alpha", [1.0, 10.0])
def test_steady_limits_laplace(alpha):
    """one time step T -> infinity on the unit circle: V/T -> Laplace single layer (eigenvalues
    1/(2n)), K 1/T -> -1/2 (interior double layer), D_curl/T -> Laplace hypersingular (n/2).
    Independent of alpha: pins every 1/alpha prefactor."""
    nseg, T = 128, 1e6
    w = _circle(nseg, alpha)
    m = O.OracleMesh(w)
    V = m.dense("V") / T
    h = m.seg_h[0]
    th = 2 * np.pi * (np.arange(nseg) + 0.5) / nseg
    for n, ref in [(1, 0.5), (2, 0.25), (3, 1 / 6), (4, 0.125)]:
        v = np.cos(n * th)
        assert (v @ V @ v) / (h * v @ v) == pytest.approx(ref, rel=5e-3)
    K = m.dense("K") / T
    assert np.allclose(K.sum(axis=1) / (h * 1.0), -0.5, atol=2e-3)
    D = m.dense("D") / T
    thd = 2 * np.pi * np.arange(nseg) / nseg + np.pi / nseg        # dual nodes = midpoints
    Lt = m.seg_h[0]
    Myy = np.zeros((nseg, nseg))
    for l in range(nseg):
        Myy[l, l] = 4 * Lt / 6
        Myy[l, (l + 1) % nseg] = Myy[l, (l - 1) % nseg] = Lt / 6
    for n in (1, 2, 3, 4):
        v = np.cos(n * thd)
        assert (v @ D @ v) / (v @ Myy @ v) == pytest.approx(n / 2, rel=2e-3)


# ---------------------------------------------- P6: K row sums (1/2 I jump)
@pytest.mark.parametrize("a,i", [(0, 1), (3, 1), (0, 0), (5, 2), (15, 3)])
def test_K_rowsum_jump_relation(c1, a, i):
    """sum_{b<=a, n} K[(a,i),(b,n)] = int_{tau_a} int_{gamma_i} (M_0 1 - 1/2): K 1 = M_0 1 - 1/2
    from eq. (3) with u = 1; exact at the discrete level (trial hats sum to one)."""
    w, m = c1
    t = w.t_breaks
    s = sum(m.entry("K", a, i, b, n) for b in range(a + 1) for n in range(m.ng))
    ref = float(B.K_rowsum_unit_square(w.alpha, t[a], t[a + 1], m.seg_a[i][0], m.seg_b[i][0]))
    assert abs(s - ref) <= 1e-13 * 0.5 * m.seg_h[i] * (t[a + 1] - t[a])


def test_K_collinear_zero(c1):
    w, m = c1
    assert m.pair(2, 0, 0, 0, 1, 1) == 0.0          # identical
    assert m.pair(2, 0, 2, 0, 1, 2) == 0.0          # collinear neighbours
    assert m.pair(2, 0, 2, 0, 1, 3, (1, 1), (1, 0)) == 0.0   # collinear, disjoint


# ---------------------------------------------- P7: D normal-term row sums
@pytest.mark.parametrize("a,l", [(2, 1), (4, 0), (9, 1)])
def test_D_rowsum_identity(c1, a, l):
    """sum_{b<=a, k} D[(a,l),(b,k)] = int_{tau_a} int psi_l(x) int_Gamma (n_x.n_y) U*(x-y,t)
    (D = -d_n W, applied to u = 1; the curl term vanishes since sum_k psi_k' = 0)."""
    w, m = c1
    t = w.t_breaks
    pieces = {1: [(0.125, 0.25, 0, 0.5), (0.25, 0.375, 0.5, 1), (0.375, 0.5, 1, 0.5), (0.5, 0.625, 0.5, 0)],
              0: [("L", 0.125, 0.0, 0, 0.5), (0.0, 0.125, 0.5, 1), (0.125, 0.25, 1, 0.5),
                  (0.25, 0.375, 0.5, 0)]}[l]
    s = sum(m.entry("D", a, l, b, k) for b in range(a + 1) for k in range(m.ng))
    ref = float(B.D_rowsum_unit_square(w.alpha, t[a], t[a + 1], pieces))
    assert s == pytest.approx(ref, rel=1e-12)


def test_D_structure(c1):
    w, m = c1
    D = dense_c1(m, "D")
    ng = m.ng
    for a in range(m.nt):
        for b in range(a + 1):
            blk = D[a * ng:(a + 1) * ng, b * ng:(b + 1) * ng]
            assert np.abs(blk - blk.T).max() <= 1e-14 * np.abs(D).max()   # symmetric blocks
    assert np.linalg.eigvalsh(0.5 * (D + D.T))[0] > 0.0
    K = dense_c1(m, "K")
    assert np.abs(K[:ng, :ng] - K[:ng, :ng].T).max() > 1e-6          # K is not


# ------------------------------------------------------- P9: mass matrices
def test_mass_matrices(c1):
    w, m = c1
    h, ht = 0.25, 1.0 / 16
    Mp = m.mass_primal()
    assert Mp[0, 0] == pytest.approx(h * ht / 2, rel=1e-15) and Mp[0, 1] == pytest.approx(h * ht / 2)
    Md = m.mass_dual()
    assert Md[5, 5] == pytest.approx(0.75 * h * ht, rel=1e-15)
    assert Md[5, 4] == pytest.approx(h * ht / 8) and Md[5, 6] == pytest.approx(h * ht / 8)
    np.testing.assert_allclose(Md.sum(axis=1), h * ht, rtol=1e-14)      # row sums |sigma|
    np.testing.assert_allclose(Md.sum(axis=0), h * ht, rtol=1e-14)
    # non-uniform lengths: row sum = h_t (h_{l-1} + 2 h_l + h_{l+1}) / 4 (SURVEY a6 check h=(1,2,3))
    hm, h0, hp = 1.0, 2.0, 3.0
    vm, vp = hm / (hm + h0), hp / (h0 + hp)
    assert hm * vm / 4 + h0 * (2 + vm + vp) / 4 + hp * vp / 4 == pytest.approx(2.0, rel=1e-15)


# --------------------------------------------------------------- P10: GMRES
def test_gmres_identity_one_iteration():
    b = np.random.default_rng(0).normal(size=50)
    x, it, hist = O.gmres(lambda v: v, lambda r: r, b, 1e-10)
    assert it == 1 and np.allclose(x, b, rtol=1e-14)


def test_gmres_matches_direct_solve(c1):
    w, m = c1
    V, K = dense_c1(m, "V"), dense_c1(m, "K")
    b = m.rhs(K, W.dirichlet_data(w))
    wd = O.block_forward_solve(V, b, m.ng)
    assert np.abs(V @ wd - b).max() <= 1e-13 * np.abs(b).max()
    x, it, hist = O.gmres(lambda v: V @ v, lambda r: r, b, 1e-10)
    assert np.all(np.diff(hist) <= 1e-15)                          # monotone (full GMRES)
    assert np.abs(x - wd).max() <= 1e-8 * np.abs(wd).max()
    assert 20 <= it <= 35                                           # SURVEY 8(c) band: ~27
    D = dense_c1(m, "D")
    for mode, band in ((1, (14, 26)), (2, (10, 22))):
        C = O.make_preconditioner(mode, D, m.mass_dual(), m.lumped_dual())
        x, itp, hist = O.gmres(lambda v: V @ v, C, b, 1e-10)
        assert band[0] <= itp <= band[1]
        assert np.abs(x - wd).max() <= 1e-8 * np.abs(wd).max()


# ------------------------------------------- P11: convergence of w_h (end to end)
@pytest.mark.slow
def test_w_converges_under_refinement():
    errs = []
    for name in ("C1", "S32"):
        w = W.get(name)
        m = O.OracleMesh(w)
        V, K = m.dense("V"), m.dense("K")
        wd = O.block_forward_solve(V, m.rhs(K, W.dirichlet_data(w)), m.ng)
        e, r = m.l2_error(wd)
        errs.append(e / r)
    assert errs[0] == pytest.approx(0.330, abs=0.01)                # prototype: 0.330 -> 0.154
    assert errs[1] < errs[0] / 1.8


# ---------------------------------------------------------------- representation formula (f2)
def _brute_potential(w, j, b, x, t, kind, q=30):
    """mpmath: (1/alpha) int_{t_b}^{min(t_{b+1}, t)} int_{gamma_j} K(x - y, t - tau) phi(y) ds dtau,
    kind 'V' (U*, phi = 1) or 'W' (d_ny U*, phi = the hat of node j+1 rising along gamma_j)"""
    mp.mp.dps = 30
    nodes = W.data.nodes(w)
    a, c = nodes[j], nodes[(j + 1) % len(nodes)]
    h = float(np.hypot(*(c - a)))
    tan = (c - a) / h
    nrm = np.array([tan[1], -tan[0]])
    al = w.alpha
    t0, t1 = w.t_breaks[b], min(w.t_breaks[b + 1], t)

    def f(sarc, tau):
        y = a + float(sarc) * tan
        d = np.asarray(x) - y
        r2 = mp.mpf(float(d @ d))
        s = t - tau
        us = al / (4 * mp.pi * s) * mp.exp(-al * r2 / (4 * s))
        if kind == "V":
            return us / al
        return (us * al * float(d @ nrm) / (2 * s)) / al * (mp.mpf(sarc) / h)
    return float(mp.quad(f, [0, h], [t0, t1]))


@pytest.mark.parametrize("kind", ["V", "W"])
def test_potential_single_element_brute_force(kind):
    """one element, one time step: the closed-form time integrals and the Gauss rule of
    ora_potential against a 2-D mpmath quadrature of the kernel of eq. (2)"""
    w = W.get("T8")
    om = O.OracleMesh(w)
    n = w.n
    j, b = 3, 2
    dens = np.zeros(n)
    pts = np.array([[0.55, 0.4, float(w.t_breaks[b + 1]) + 0.03], [0.35, 0.6, float(w.t_breaks[b]) + 0.05]])
    if kind == "V":
        dens[b * w.n_gamma + j] = 1.0
        got = om.potential(dens, np.zeros(n), pts)
    else:   # g = hat of node j+1 in step b: rises along gamma_j, falls along gamma_{j+1}
        g = np.zeros(n)
        g[b * w.n_gamma + (j + 1)] = 1.0
        got = om.potential(np.zeros(n), g, pts)
    for k, (x1, x2, t) in enumerate(pts):
        ref = _brute_potential(w, j, b, (x1, x2), t, kind)
        if kind == "W":
            # -W g: rising part on gamma_j + falling part on gamma_{j+1} (= constant - rising)
            ref_next_full = _brute_potential_const(w, j + 1, b, (x1, x2), t)
            ref_next_rise = _brute_potential(w, j + 1, b, (x1, x2), t, "W")
            ref = -(ref + ref_next_full - ref_next_rise)
        assert abs(got[k] - ref) <= 1e-12 * max(1e-6, abs(ref)), (kind, k, got[k], ref)


def _brute_potential_const(w, j, b, x, t):
    """W-kernel with phi = 1 on gamma_j"""
    mp.mp.dps = 30
    nodes = W.data.nodes(w)
    a, c = nodes[j], nodes[(j + 1) % len(nodes)]
    h = float(np.hypot(*(c - a)))
    tan = (c - a) / h
    nrm = np.array([tan[1], -tan[0]])
    al = w.alpha
    t0, t1 = w.t_breaks[b], min(w.t_breaks[b + 1], t)

    def f(sarc, tau):
        y = a + float(sarc) * tan
        d = np.asarray(x) - y
        r2 = mp.mpf(float(d @ d))
        s = t - tau
        us = al / (4 * mp.pi * s) * mp.exp(-al * r2 / (4 * s))
        return us * float(d @ nrm) / (2 * s)
    return float(mp.quad(f, [0, h], [t0, t1]))


def test_potential_converges_to_manufactured_solution():
    """u_h = Vt w_h - W g_h at interior points tends to u = U*(x - x*, t) under refinement
    (T8 -> C1 -> S32; w_h from the oracle's own V_h, K_h and block forward substitution)"""
    pts = np.array([[0.5, 0.5, 0.5], [0.25, 0.5, 1.0], [0.5, 0.75, 0.75], [0.3, 0.3, 0.25]])
    errs = []
    for name in ("T8", "C1", "S32"):
        w = W.get(name)
        om = O.OracleMesh(w)
        g = W.dirichlet_data(w)
        wh = O.block_forward_solve(om.dense("V"), om.rhs(om.dense("K"), g), om.ng)
        ex = W.exact_solution(w, pts[:, :2], pts[:, 2])
        errs.append(np.abs(om.potential(wh, g, pts) - ex).max() / np.abs(ex).max())
    assert errs[0] > 2.0 * errs[1] > 4.0 * errs[2] * 0.5, errs
    assert errs[2] < 2e-3, errs


# ------------------------------------------------------ initial potential M_h^0 u0 (f1)
def test_initial_potential_closed_form_constant_u0():
    """u0 = 1: (M_0 1)(x,t) = int_(0,1)^2 U*(x-y,t) dy = prod_k (erf((1-x_k)/s) + erf(x_k/s)) / 2,
    s = sqrt(4t/alpha) (U* factorises); its integral over gamma_i x [t_a, t_{a+1}] by scipy
    against the oracle's M_h^0 1 (exact time integrals, Gauss / collapsed Gauss / apex-split rule)"""
    from scipy import integrate
    from scipy.special import erf
    import workloads.table1 as T
    w = T.table1(3)
    om = O.OracleMesh(w)
    nodes, tris = T.triangulation(w)
    f = om.initial_rhs(nodes, tris, np.ones(len(nodes)), 8, 6, 16)
    al = w.alpha

    def m0one(x, t):
        s = np.sqrt(4 * t / al)
        return np.prod([0.5 * (erf((1 - xk) / s) + erf(xk / s)) for xk in x])
    # elements 0, 4 start at a corner of Q (graded x and eta rules of the step-0 term, reading R22)
    for a, i, tol in [(0, 0, 1e-9), (0, 4, 1e-9), (1, 0, 1e-10), (0, 1, 1e-10), (0, 6, 1e-10), (1, 5, 1e-11),
                      (5, 9, 1e-11), (12, 12, 1e-11), (15, 15, 1e-11)]:
        A, B, h = om.seg_a[i], om.seg_b[i], om.seg_h[i]
        ref, _ = integrate.dblquad(lambda s, t: m0one(A + s * (B - A), t) * h, w.t_breaks[a],
                                   w.t_breaks[a + 1], 0, 1, epsabs=1e-16, epsrel=1e-13)
        assert abs(f[a * om.ng + i] - ref) <= tol * abs(ref), (a, i, f[a * om.ng + i], ref)


def test_initial_rhs_closed_form_linear_u0():
    """u0 = y1 (in S_h^1: the nodal interpolant is exact): (M_0 y1)(x,t) = int_(0,1)^2 U*(x-y,t) y1 dy
    = m1(x1) P(x2), the first Gaussian moment and the erf integral of the two 1-D factors of U*
    (variance 2t/alpha), integrated over gamma_i x [t_a, t_{a+1}] by scipy against the
    oracle's M_h^0 y1: pins the barycentric interpolation of u0 and the apex-split rule with a
    non-constant u0 (reading R22)"""
    from scipy import integrate
    import workloads.table1 as T
    w = T.table1(3)
    om = O.OracleMesh(w)
    nodes, tris = T.triangulation(w)
    f = om.initial_rhs(nodes, tris, nodes[:, 0].copy(), 8, 6, 16)
    al = w.alpha

    def m0y1(x, t):
        sigma = np.sqrt(2 * t / al)
        _, M1 = _gauss_moments(x[0], sigma)
        P2, _ = _gauss_moments(x[1], sigma)
        return M1 * P2
    # elements 0, 4 start at a corner of Q (graded rules of the step-0 term); elements on the sides
    # y1 = 0 (0..3) and y1 = 1 (4..7) see u0's extreme values
    for a, i, tol in [(0, 0, 1e-9), (0, 4, 1e-9), (0, 5, 1e-10), (1, 0, 1e-10), (0, 9, 1e-10), (1, 5, 1e-11),
                      (3, 2, 1e-11), (5, 9, 1e-11), (12, 12, 1e-11), (15, 6, 1e-11)]:
        A, Bp, h = om.seg_a[i], om.seg_b[i], om.seg_h[i]
        ref, _ = integrate.dblquad(lambda s, t: m0y1(A + s * (Bp - A), t) * h, w.t_breaks[a],
                                   w.t_breaks[a + 1], 0, 1, epsabs=1e-17, epsrel=1e-13)
        assert abs(f[a * om.ng + i] - ref) <= tol * max(abs(ref), 1e-3 * np.abs(f).max()), (a, i, f[a * om.ng + i], ref)


def test_table1_density_converges():
    """the paper's experiment: V_h w = (1/2 M_h + K_h) g - M_h^0 u0 solved by block
    forward substitution; the L2(Sigma) error of w_h against d_n u falls under refinement"""
    import workloads.table1 as T
    errs = []
    for L in (2, 3, 4):
        w = T.table1(L)
        om = O.OracleMesh(w)
        nodes, tris = T.triangulation(w)
        g = T.dirichlet_data(w)
        b = om.rhs(om.dense("K"), g) - om.initial_rhs(nodes, tris, T.initial_nodes(w), 4, 4, 12)
        wh = O.block_forward_solve(om.dense("V"), b, om.ng)
        err, ref = om.l2_error(wh, exact=lambda x, n, t: T.exact_neumann(x, n, t))
        errs.append(err / ref)
    assert errs[0] > 1.5 * errs[1] > 2.25 * errs[2], errs


# ------------------------------------------- initial potential in Q (row f2, u0 != 0)
def _gauss_moments(x, sigma):
    """int_0^1 N(y; x, sigma^2) dy and int_0^1 y N(y; x, sigma^2) dy (closed forms)"""
    from scipy.special import erf
    s2 = np.sqrt(2.0) * sigma
    P = 0.5 * (erf((1.0 - x) / s2) + erf(x / s2))
    m1 = x * P + sigma / np.sqrt(2.0 * np.pi) * (np.exp(-x * x / (2 * sigma * sigma)) - np.exp(-(1 - x) ** 2 / (2 * sigma * sigma)))
    return P, m1


@pytest.mark.parametrize("t", [0.5, 0.05, 0.002])
def test_initial_potential_in_Q_closed_forms(t):
    """(M~_0 u0)(x, t) = int_Omega U*(x - y, t) u0(y) dy on the unit square for u0 = 1 and u0 = y1
    (both in S_h^1, so the triangulation is exact): U* is the product of two 1-D Gaussians of
    variance 2t/alpha, the integrals are erf products and first Gaussian moments; small t makes
    the Gaussian narrower than the triangles (composite cells)"""
    import workloads.table1 as T
    w = T.table1(3)
    om = O.OracleMesh(w)
    nodes, tris = T.triangulation(w)
    alpha = w.alpha
    sigma = np.sqrt(2.0 * t / alpha)
    pts = np.array([[0.5, 0.5, t], [0.3, 0.8, t], [0.05, 0.6, t]])
    one = om.potential_initial(nodes, tris, np.ones(len(nodes)), pts)
    lin = om.potential_initial(nodes, tris, nodes[:, 0].copy(), pts)
    for k, (x1, x2, _) in enumerate(pts):
        P1, M1 = _gauss_moments(x1, sigma)
        P2, _ = _gauss_moments(x2, sigma)
        assert one[k] == pytest.approx(P1 * P2, rel=1e-12), (t, k)
        assert lin[k] == pytest.approx(M1 * P2, rel=1e-11, abs=1e-15), (t, k)


def test_rhs_rows_equal_the_dense_rhs():
    """oracle rhs_rows (row-wise (1/2 M_h + K_h) g for the full-size sampled tests) against the dense
    (1/2 M_h + K_h) g on C1: the causal row range and the mass row of P:89"""
    import workloads as W
    w = W.get("C1")
    om = O.OracleMesh(w)
    g = W.dirichlet_data(w)
    ref = om.rhs(om.dense("K"), g)
    rows = [0, 1, w.n_gamma - 1, w.n // 2, w.n - 1]
    assert np.abs(om.rhs_rows(rows, g) - ref[rows]).max() <= 1e-14 * np.abs(ref).max()


def test_matvec_rows_equal_the_dense_products():
    import workloads as W
    w = W.get("C1")
    om = O.OracleMesh(w)
    x = np.random.default_rng(5).standard_normal(w.n)
    rows = [0, 3, w.n // 2, w.n - 1]
    for kind in "VD":
        ref = om.dense(kind) @ x
        assert np.abs(om.matvec_rows(kind, rows, x) - ref[rows]).max() <= 1e-14 * np.abs(ref).max()


def test_uniform_grid_block_toeplitz_identity():
    """DESIGN.md reading R26 (the C3 golden density of oracle/gen_golden.py rests on it): on a
    uniform grid t_k = k h the four lags of entry (a, b) are (d+1) h, d h, d h, (d-1) h with
    d = a - b, so A(a, b) = A(a - b, 0); on the dyadic grids of C1-C4 the lags are the same doubles
    and the oracle's entries agree bitwise -- random entries of C2 against the first block column"""
    import workloads as W
    w = W.get("C2")
    m = O.OracleMesh(w)
    ng, nt = m.ng, m.nt
    rng = np.random.default_rng(26)
    a = rng.integers(0, nt, 400)
    b = (rng.random(400) * (a + 1)).astype(np.int64)
    i, j = rng.integers(0, ng, 400), rng.integers(0, ng, 400)
    for kind in "VKD":
        full = m.entries(kind, a * ng + i, b * ng + j)
        first = m.entries(kind, (a - b) * ng + i, j)
        assert np.array_equal(full, first), kind
