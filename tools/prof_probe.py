"""assemble one matrix kind of a config once (for ncu --set full captures); kind 'Kg' = fused K g"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from paper_1811_05224_b200 import stbem as S
name, kind = sys.argv[1], sys.argv[2]
w = W.get(name)
m = S.Mesh.from_workload(w)
if kind == "Kg":
    g = torch.tensor(W.dirichlet_data(w), dtype=torch.float64, device="cuda")
    b = torch.empty_like(g)
    print(name, kind, S.rhs_fused(m, m.assemble_M(S.MASS_PRIMAL), g, b, stats=True))
else:
    A = getattr(m, f"assemble_{kind}")()
    torch.cuda.synchronize()
    print(name, kind, A.stats())
