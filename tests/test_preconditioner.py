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
