"""relative max-norm errors of the bench-configuration GPU solve against the oracle goldens (C2, C3,
the first 24 steps of C5): b (right-hand side) and w (density)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1811_05224_b200 import stbem as S  # noqa: E402

G = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
for name, suffix in (("C2", ""), ("C3", ""), ("C5", "_first24")):
    w = W.get(name)
    wd, bd = np.load(os.path.join(G, f"{name}_oracle_w{suffix}.npy")), np.load(os.path.join(G, f"{name}_oracle_b{suffix}.npy"))
    m = S.Mesh.from_workload(w)
    V, D = m.assemble_V(), m.assemble_D()
    Mp, Md = m.assemble_M(S.MASS_PRIMAL), m.assemble_M(S.MASS_DUAL)
    g = torch.tensor(W.dirichlet_data(w), dtype=torch.float64, device="cuda")
    b = torch.empty_like(g)
    S.rhs_fused(m, Mp, g, b)
    wv = torch.zeros_like(g)
    rep = S.solve_gmres(V, b, wv, D=D, M=Md, precond=2, rel_tol=w.tol, history=False)
    k = len(wd)
    eb = np.abs(b.cpu().numpy()[:k] - bd).max() / np.abs(bd).max()
    ew = np.abs(wv.cpu().numpy()[:k] - wd).max() / np.abs(wd).max()
    print(f"{name}{suffix}: iterations {rep['iterations']}, b rel max err {eb:.2e}, w rel max err {ew:.2e}", flush=True)
    for A in (V, D, Mp, Md):
        A.close()
    m.close()
