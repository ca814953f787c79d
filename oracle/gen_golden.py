"""Write oracle reference solutions under tests/golden/ (calls only oracle/ and the shared
input generators in workloads/).  Test infrastructure.

python -m oracle.gen_golden C2     (dense V_h, K_h at C2: ~3 min on 8 cores)
python -m oracle.gen_golden C3     (first block columns of V_h, K_h at C3: ~5 min on 8 cores)
python -m oracle.gen_golden C5     (the first 24 time steps of C5: ~12 min on 8 cores)

C2: the dense oracle matrices, b = (1/2 M_h + K_h) g (eq. 4), w by block forward
substitution (V_h is block lower triangular).

C3 (N = 65 536; the dense oracle matrices would be 2 x 34 GB and ~2 h): on a uniform time grid
every entry depends on the test and trial steps only through the lag d = a - b (DESIGN.md
reading R26: the four lags of P:86-88 are t_{a+1} - t_b, ... = (d + 1) h_t, ...; on C3's dyadic
grid t_k = k / 256 they are the same doubles for every (a, b) with the same d, so the oracle's
entries are bitwise equal -- tests/test_oracle_pins.py checks it on C2).  The oracle computes the
first block columns T_d = A(d, 0), d = 0 .. N_I - 1, of V_h and K_h entry by entry
(stbem_oracle.c), then in plain numpy
    (K_h g)_a = sum_{b <= a} T^K_{a-b} g_b,     b = 1/2 M_h g + K_h g,
    T^V_0 w_a = b_a - sum_{b < a} T^V_{a-b} w_b   (block forward substitution, a = 0 .. N_I - 1).

C5 (N = 98 304, graded steps: no Toeplitz structure): V_h and K_h are block lower triangular in time
(P:151-159), so the density of the first A0 steps depends only on the blocks (a, b), b <= a < A0:
the oracle computes those blocks entry by entry, b_a = 1/2 (M_h g)_a + sum_{b <= a} K_ab g_b for
a < A0, and w_a by block forward substitution -- the exact first A0 time steps of the C5 solution.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402
from oracle import oracle as O  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def first_block_column(m, kind):
    """T[d] = A(d, 0) (N_Gamma x N_Gamma), d = 0 .. N_I - 1: rows (d, i), columns (0, j)"""
    ng, nt = m.ng, m.nt
    rows = np.repeat(np.arange(nt * ng, dtype=np.int64), ng)
    cols = np.tile(np.arange(ng, dtype=np.int64), nt * ng)
    return m.entries(kind, rows, cols).reshape(nt, ng, ng)


def toeplitz_solve(TV, TK, m, g):
    """b = 1/2 M_h g + K_h g and w with V_h w = b for block-Toeplitz V_h, K_h (module docstring)"""
    ng, nt = m.ng, m.nt
    G = g.reshape(nt, ng)
    Kg = np.zeros((nt, ng))
    for a in range(nt):
        for b in range(a + 1):
            Kg[a] += TK[a - b] @ G[b]
    # primal mass: M[(a,i),(a,n)] = h_t(a) h_i / 2, n in {i, i+1}
    Mg = (m.ht[:, None] * m.seg_h[None, :] / 2) * (G + np.roll(G, -1, axis=1))
    B = 0.5 * Mg + Kg
    Wd = np.zeros((nt, ng))
    for a in range(nt):
        r = B[a].copy()
        for b in range(a):
            r -= TV[a - b] @ Wd[b]
        Wd[a] = np.linalg.solve(TV[0], r)
    return B.reshape(-1), Wd.reshape(-1)


def leading_steps(m, g, A0):
    """b and w of the first A0 time steps (block forward substitution over the oracle's blocks)"""
    ng = m.ng
    rows = np.repeat(np.arange(A0 * ng, dtype=np.int64), A0 * ng)
    cols = np.tile(np.arange(A0 * ng, dtype=np.int64), A0 * ng)
    keep = cols // ng <= rows // ng                     # causal blocks b <= a only
    rows, cols = rows[keep], cols[keep]
    Vd = np.zeros((A0 * ng, A0 * ng))
    Kd = np.zeros((A0 * ng, A0 * ng))
    Vd[rows, cols] = m.entries("V", rows, cols)
    Kd[rows, cols] = m.entries("K", rows, cols)
    G = g[: A0 * ng].reshape(A0, ng)
    Mg = (m.ht[:A0, None] * m.seg_h[None, :] / 2) * (G + np.roll(G, -1, axis=1))   # primal mass
    b = 0.5 * Mg.reshape(-1) + Kd @ g[: A0 * ng]
    w = O.block_forward_solve(Vd, b, ng)
    return b, w


def main(name):
    w = W.get(name)
    t0 = time.time()
    m = O.OracleMesh(w)
    g = W.dirichlet_data(w)
    if name == "C5":
        A0 = 24
        b, wd = leading_steps(m, g, A0)
        np.save(os.path.join(GOLDEN, "C5_oracle_b_first24.npy"), b)
        np.save(os.path.join(GOLDEN, "C5_oracle_w_first24.npy"), wd)
        meta = {"config": name, "steps": A0, "n": int(A0 * m.ng), "t_end": float(w.t_breaks[A0]),
                "seconds": time.time() - t0, "threads": int(O.lib().ora_num_threads()),
                "source": "oracle/gen_golden.py: the oracle's blocks (a, b), b <= a < 24, of V_h and K_h "
                          "(stbem_oracle.c), b = (1/2 M_h + K_h) g and w by block forward substitution "
                          "over the first 24 time steps (P:83, P:151-159)"}
        with open(os.path.join(GOLDEN, "C5_oracle_first24.json"), "w") as fh:
            json.dump(meta, fh, indent=1)
        print(meta)
        return
    if name == "C3":
        assert np.all(np.diff(w.t_breaks) == w.t_breaks[1]), "uniform steps required"
        TV = first_block_column(m, "V")
        TK = first_block_column(m, "K")
        b, wd = toeplitz_solve(TV, TK, m, g)
        how = ("oracle first block columns T_d = A(d, 0) of V_h and K_h (stbem_oracle.c; block-Toeplitz "
               "on the uniform dyadic grid, DESIGN.md R26), b = (1/2 M_h + K_h) g, w = block forward "
               "substitution of V_h w = b (P:83, P:151-159)")
    else:
        V = m.dense("V")
        K = m.dense("K")
        b = m.rhs(K, g)
        wd = O.block_forward_solve(V, b, m.ng)
        how = ("oracle V_h, K_h (stbem_oracle.c), b = (1/2 M_h + K_h) g, w = block forward substitution "
               "of V_h w = b (P:83, P:151-159)")
    e, r = m.l2_error(wd)
    os.makedirs(GOLDEN, exist_ok=True)
    np.save(os.path.join(GOLDEN, f"{name}_oracle_b.npy"), b)
    np.save(os.path.join(GOLDEN, f"{name}_oracle_w.npy"), wd)
    meta = {"config": name, "n": int(m.n), "l2_rel_error_w": float(e / r), "seconds": time.time() - t0,
            "threads": int(O.lib().ora_num_threads()), "source": "oracle/gen_golden.py: " + how}
    with open(os.path.join(GOLDEN, f"{name}_oracle.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(meta)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C2")
