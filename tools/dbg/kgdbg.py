import sys, numpy as np, torch
sys.path.insert(0, ".")
import workloads as W
from paper_1811_05224_b200 import stbem as S
for name in sys.argv[1:]:
    w = W.get(name); m = S.Mesh.from_workload(w)
    g = torch.tensor(W.dirichlet_data(w), dtype=torch.float64, device="cuda")
    Mp = m.assemble_M(S.MASS_PRIMAL)
    bt, be = torch.empty_like(g), torch.empty_like(g)
    S.rhs_fused(m, Mp, g, bt); S.rhs_fused(m, Mp, g, be, entrywise=True)
    d = (bt - be).abs().cpu().numpy().reshape(w.n_steps, w.n_gamma); mx = be.abs().max().item()
    ra = d.max(1) / mx; ri = d.max(0) / mx
    print(name, "max", d.max() / mx, "worst steps", np.argsort(ra)[-5:], ra[np.argsort(ra)[-5:]], "worst segs", np.argsort(ri)[-5:])
    print(" per-step err (every 16th):", np.round(np.log10(ra[::16] + 1e-30), 1))
