"""row f2 on the paper's Table-1 problem (u0 != 0): u_h = M~_0 u0 + Vt w_h - W g at interior points
after the preconditioned solve, against u = e^{-t/alpha} sin(x . d); one JSON line per level"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import workloads.table1 as T
from paper_1811_05224_b200 import stbem as S

pts = np.array([[0.5, 0.5, 0.25], [0.5, 0.5, 0.5], [0.5, 0.5, 0.9]])
for L in [int(v) for v in (sys.argv[1:] or "2 3 4 5 6 7".split())]:
    w = T.table1(L)
    m = S.Mesh.from_workload(w)
    V, D, Mp, Md = m.assemble_V(), m.assemble_D(), m.assemble_M(S.MASS_PRIMAL), m.assemble_M(S.MASS_DUAL)
    nodes, tris = T.triangulation(w)
    u0 = torch.tensor(T.initial_nodes(w), dtype=torch.float64, device="cuda")
    g = torch.tensor(T.dirichlet_data(w), dtype=torch.float64, device="cuda")
    b = torch.empty_like(g)
    S.rhs_fused(m, Mp, g, b)
    S.rhs_initial(m, nodes, tris, u0, b)
    wv = torch.zeros_like(g)
    S.solve_gmres(V, b, wv, D=D, M=Md, precond=2, rel_tol=1e-10, history=False)
    P = torch.tensor(pts, device="cuda")
    u = S.eval_potential(m, wv, g, P)
    S.eval_potential_initial(m, nodes, tris, u0, P, u)
    ex = np.array([float(T.exact(p[None, :2], p[2])[0]) for p in pts])
    err = np.abs(u.cpu().numpy() - ex) / np.abs(ex)
    print(json.dumps({"L": L, "N": w.n, "points": pts.tolist(), "u_h": u.cpu().numpy().tolist(),
                      "exact": ex.tolist(), "rel_err": err.tolist()}), flush=True)
