"""the paper's own experiment (Table 1) on the GPU path.
alpha = 10, u = exp(-t/alpha) sin(x . d), u0 != 0: b = (1/2 M_h + K_h) g - M_h^0 u0 (fused K g,
bem_rhs_initial), GMRES to 1e-8 without and with the lumped preconditioner (the paper's choice,
P:185) and with the exact dual mass; the L2(Sigma) error of w_h against d_n u.  Levels 2..7 on the
dense path, levels 8 and 9 (N = 262 144, 1 048 576: the paper's largest) on the block-Toeplitz variant.
Prints one JSON line per level."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import workloads.table1 as T
from workloads.data import nodes as boundary_nodes
from paper_1811_05224_b200 import stbem as S

PAPER = {2: (14, 17), 3: (19, 18), 4: (24, 20), 5: (35, 20), 6: (50, 20), 7: (67, 20), 8: (91, 19), 9: (122, 19)}


def l2_error(w, wh, nq=6):
    xg, wg = np.polynomial.legendre.leggauss(nq)
    xg, wg = 0.5 * (xg + 1), 0.5 * wg
    x = boundary_nodes(w)
    ng, nt = w.n_gamma, w.n_steps
    a = x, np.roll(x, -1, axis=0)
    h = np.linalg.norm(a[1] - a[0], axis=1)
    tan = (a[1] - a[0]) / h[:, None]
    nrm = np.stack([tan[:, 1], -tan[:, 0]], 1)
    t = np.asarray(w.t_breaks)
    W = wh.reshape(nt, ng)
    pts = a[0][:, None, :] + xg[None, :, None] * (a[1] - a[0])[:, None, :]          # (ng, nq, 2)
    err2 = ref2 = 0.0
    for b in range(nt):
        tt = t[b] + (t[b + 1] - t[b]) * xg                                           # (nq,)
        ex = T.exact_neumann(pts[:, :, None, :], nrm[:, None, None, :], tt[None, None, :])   # (ng, nq, nq)
        ww = (wg[:, None] * wg[None, :])[None] * h[:, None, None] * (t[b + 1] - t[b])
        err2 += np.sum(ww * (W[b][:, None, None] - ex) ** 2)
        ref2 += np.sum(ww * ex ** 2)
    return float(np.sqrt(err2 / ref2))


for L in [int(v) for v in (sys.argv[1:] or "2 3 4 5 6 7 8 9".split())]:
    w = T.table1(L)
    toep = L >= 8
    m = S.Mesh.from_workload(w)
    g = torch.tensor(T.dirichlet_data(w), dtype=torch.float64, device="cuda")
    u0 = torch.tensor(T.initial_nodes(w), dtype=torch.float64, device="cuda")
    nodes, tris = T.triangulation(w)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    V = m.assemble_toeplitz("V") if toep else m.assemble_V()
    D = m.assemble_toeplitz("D") if toep else m.assemble_D()
    Mp = m.assemble_M(S.MASS_PRIMAL)
    b = torch.empty_like(g)
    if toep:
        Kt = m.assemble_toeplitz("K")
        S.rhs(Kt, Mp, g, b)
        Kt.close()
    else:
        S.rhs_fused(m, Mp, g, b)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    S.rhs_initial(m, nodes, tris, u0, b)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    res = {"L": L, "N": w.n, "variant": "toeplitz" if toep else "dense", "assembly_s": t1 - t0, "initial_rhs_s": t2 - t1,
           "paper_it": PAPER[L][0], "paper_it_prec": PAPER[L][1]}
    for prec, M in ((0, None), (1, m.assemble_M(S.MASS_DUAL_LUMPED)), (2, m.assemble_M(S.MASS_DUAL))):
        wv = torch.zeros_like(g)
        torch.cuda.synchronize()
        ts = time.perf_counter()
        rep = S.solve_gmres(V, b, wv, D=D if prec else None, M=M, rel_tol=1e-8, max_iter=300, precond=prec, history=False)
        torch.cuda.synchronize()
        key = ["none", "lumped", "exact"][prec]
        res[f"it_{key}"] = rep["iterations"]
        res[f"solve_s_{key}"] = time.perf_counter() - ts
        if prec == 1:
            res["l2_error_w"] = l2_error(w, wv.cpu().numpy())
    print(json.dumps(res), flush=True)
    for A in (V, D, Mp):
        A.close()
    m.close()
