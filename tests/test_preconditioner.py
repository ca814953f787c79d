"""Theorem 1 of the paper: the opposite-order preconditioner C_V^{-1} = M_h^{-1} D_h
M_h^{-T} makes the condition number of C_V^{-1} V_h bounded independently of the mesh, while that
of V_h grows under refinement.  Checked on the oracle's dense matrices of T8 and C1 (SURVEY 8(f)
row f4; SPEC's stability surrogate S:428-436 asks the same of the small meshes).  CPU only."""
import numpy as np
import pytest

import workloads as W
from oracle import oracle as O


@pytest.fixture(scope="module")
def conds():
    out = {}
    for name in ("T8", "C1"):
        om = O.OracleMesh(W.get(name))
        V, D = om.dense("V"), om.dense("D")
        Md, dl = om.mass_dual(), om.lumped_dual()
        dinv = 1.0 / dl
        CV_lumped = dinv[:, None] * (D @ (dinv[:, None] * V))
        CV_exact = np.linalg.solve(Md, D @ np.linalg.solve(Md.T, V))
        out[name] = {"V": np.linalg.cond(V), "lumped": np.linalg.cond(CV_lumped),
                     "exact": np.linalg.cond(CV_exact)}
    return out


def test_preconditioned_condition_smaller(conds):
    for name, c in conds.items():
        assert c["lumped"] < 0.5 * c["V"], (name, c)
        assert c["exact"] < 0.5 * c["V"], (name, c)


def test_condition_bounded_under_refinement(conds):
    """T8 -> C1 halves h and h_t: kappa(V) grows (about like h^-1), the preconditioned one stays"""
    g_V = conds["C1"]["V"] / conds["T8"]["V"]
    assert g_V > 1.4, conds
    for mode in ("lumped", "exact"):
        assert conds["C1"][mode] / conds["T8"][mode] < 1.2, (mode, conds)


# ------------------------------------------------ the discrete stability condition (eq. 5)
def test_stability_ratio_closed_form_on_uniform_meshes():
    """SPEC's stability surrogate (eq. 5): on a closed boundary with equal elements
    the pairing, the dual-hat Gram matrix and G_X are circulant, h circ(1/8, 3/4, 1/8),
    h circ(1/6, 2/3, 1/6) and h I, so the inf-sup constant is min over theta of
    (3/4 + cos(theta)/4) / sqrt(2/3 + cos(theta)/3) = sqrt(3)/2 at theta = pi, for every level"""
    import workloads.table1 as T
    for L in (2, 3, 4):
        om = O.OracleMesh(T.table1(L))
        ratio, smin = om.stability_ratio()
        assert ratio == pytest.approx(np.sqrt(3.0) / 2.0, rel=1e-12), (L, ratio)
        assert smin > 0.0


def test_stability_ratio_nonuniform_and_gram_partition_of_unity():
    """unequal elements per side: the ratio stays bounded away from 0 (>= half the uniform value,
    SPEC's trend check); the dual hats sum to one, so each Gram row sums to int psi_l, the row
    sum of the dual mass"""
    from workloads.configs import Workload, uniform_times
    from workloads.edge import SQUARE
    w = Workload("nonuni", SQUARE, [2, 3, 4, 5], uniform_times(4), 1.0, (1.5, 1.5), 1e-10)
    om = O.OracleMesh(w)
    ratio, smin = om.stability_ratio()
    assert 0.5 * np.sqrt(3.0) / 2.0 <= ratio < 1.0 and smin > 0.0
    G = om.dual_gram()
    ng = om.ng
    np.testing.assert_allclose(G.sum(axis=1), om.mass_dual()[:ng, :ng].sum(axis=1) / om.ht[0], rtol=1e-14)
    np.testing.assert_allclose(G, G.T, rtol=0, atol=1e-16)
