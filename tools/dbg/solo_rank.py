"""one rank (r of G, solo communicator) of C5: V_h, D_h, K_h g assembly, for a launch list"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import workloads as W
from paper_1811_05224_b200 import stbem as S
G, r = int(sys.argv[1]), int(sys.argv[2])
w = W.get(sys.argv[3] if len(sys.argv) > 3 else "C5")
c = S.Comm.solo(G, r, 0)
m = S.Mesh.from_workload(w, n_slices=2 * G, comm=c)
Mp = m.assemble_M(S.MASS_PRIMAL)
g = torch.tensor(W.dirichlet_data(w), dtype=torch.float64, device="cuda")
b = torch.empty_like(g)
for it in range(2):
    V = m.assemble_V(); D = m.assemble_D(); S.rhs_fused(m, Mp, g, b)
    torch.cuda.synchronize()
    V.close(); D.close()
print("ok")
