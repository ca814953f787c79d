"""exact vs lumped dual-mass preconditioning on uniform and
graded meshes.  GMRES iterations and solve times for precond 0 / 1 / 2 (tol 1e-10) on
C1, S32, C2, C3, C5 (C5: graded steps, L-shape), and the condition numbers of V_h and C_V^{-1} V_h
(dense readback of the GPU matrices, numpy) on T8, C1, S32, C2.  Writes one JSON document."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import workloads as W
from paper_1811_05224_b200 import stbem as S

out = {"iterations": {}, "condition": {}}
for name in sys.argv[1:] or ["C1", "S32", "C2", "C3", "C5"]:
    w = W.get(name)
    m = S.Mesh.from_workload(w)
    V, D = m.assemble_V(), m.assemble_D()
    Mp = m.assemble_M(S.MASS_PRIMAL)
    Ml, Me = m.assemble_M(S.MASS_DUAL_LUMPED), m.assemble_M(S.MASS_DUAL)
    g = torch.tensor(W.dirichlet_data(w), dtype=torch.float64, device="cuda")
    b = torch.empty_like(g)
    S.rhs_fused(m, Mp, g, b)
    res = {}
    for prec, Mc in ((0, None), (1, Ml), (2, Me)):
        wv = torch.zeros_like(g)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = S.solve_gmres(V, b, wv, D=D if prec else None, M=Mc, rel_tol=1e-10, max_iter=400,
                            precond=prec, history=False)
        torch.cuda.synchronize()
        res[["none", "lumped", "exact"][prec]] = {"iterations": rep["iterations"], "converged": bool(rep["converged"]),
                                                  "true_rel_residual": rep["true_rel_residual"],
                                                  "seconds": time.perf_counter() - t0}
    out["iterations"][name] = {"N": w.n, "kappa": m.info.kappa, **res}
    print(name, json.dumps(out["iterations"][name]), flush=True)
    if w.n <= 4096:
        Vd, Dd = V.dense(), D.dense()
        ng = w.n_gamma
        # dual mass matrices from the solves (dense, small): columns of M^{-1}
        eye = torch.eye(w.n, dtype=torch.float64, device="cuda")
        Minv_l = np.stack([Ml.solve(eye[:, k].contiguous(), torch.empty(w.n, dtype=torch.float64, device="cuda")).cpu().numpy() for k in range(w.n)], 1)
        Minv_e = np.stack([Me.solve(eye[:, k].contiguous(), torch.empty(w.n, dtype=torch.float64, device="cuda")).cpu().numpy() for k in range(w.n)], 1)
        MinvT_e = np.stack([Me.solve(eye[:, k].contiguous(), torch.empty(w.n, dtype=torch.float64, device="cuda"), transpose=True).cpu().numpy() for k in range(w.n)], 1)
        out["condition"][name] = {"V": float(np.linalg.cond(Vd)),
                                  "lumped": float(np.linalg.cond(Minv_l @ Dd @ Minv_l @ Vd)),
                                  "exact": float(np.linalg.cond(Minv_e @ Dd @ MinvT_e @ Vd))}
        print(name, "cond", out["condition"][name], flush=True)
    for A in (V, D, Mp, Ml, Me):
        A.close()
    m.close()
json.dump(out, open(os.environ.get("OUT", "gpurun_out/precond_study.json"), "w"), indent=1)
