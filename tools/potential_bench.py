"""row f2 throughput: representation formula u = Vt w - W g at interior points of C3 after the
solve (evaluations = points x space-time elements x Gauss points); CUDA events, median of 5"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_1811_05224_b200 import stbem as S
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
npts = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
w = W.get(name)
m = S.Mesh.from_workload(w)
V, D = m.assemble_V(), m.assemble_D()
g = torch.tensor(W.dirichlet_data(w), dtype=torch.float64, device="cuda")
b = torch.empty_like(g)
S.rhs_fused(m, m.assemble_M(S.MASS_PRIMAL), g, b)
wv = torch.zeros_like(g)
S.solve_gmres(V, b, wv, D=D, M=m.assemble_M(S.MASS_DUAL), rel_tol=1e-10, max_iter=200, precond=2)
rng = np.random.default_rng(1811)
pts = np.stack([rng.uniform(0.1, 0.9, npts), rng.uniform(0.1, 0.9, npts), rng.uniform(0.05, 1.0, npts)], 1)
P = torch.tensor(pts, device="cuda")
out = torch.empty(npts, dtype=torch.float64, device="cuda")
S.eval_potential(m, wv, g, P, out)
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); S.eval_potential(m, wv, g, P, out); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts))
u = out.cpu().numpy()
ex = W.exact_solution(w, pts[:, :2], pts[:, 2])
elems = float(np.sum(np.searchsorted(w.t_breaks, pts[:, 2]) * w.n_gamma))   # (b, j) with t_b < t
print(json.dumps({"config": name, "points": npts, "ms": ms, "points_per_s": npts / ms * 1e3,
                  "element_integrals_per_s": elems / ms * 1e3,
                  "max_rel_error_vs_exact": float(np.abs(u - ex).max() / np.abs(ex).max())}))
