"""host-side timing of one bench step (where does the host spend time between GPU phases)"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from paper_1811_05224_b200 import stbem as S
w = W.get(sys.argv[1] if len(sys.argv) > 1 else "C3")
g = torch.tensor(W.dirichlet_data(w), dtype=torch.float64, device="cuda")
b = torch.empty_like(g); wv = torch.empty_like(g)
for it in range(4):
    T = {}
    t0 = time.perf_counter()
    def mark(k):
        T[k] = time.perf_counter() - t0
    mesh = S.Mesh.from_workload(w); mark("mesh")
    V = mesh.assemble_V(); mark("V")
    K = mesh.assemble_K(); mark("K")
    D = mesh.assemble_D(); mark("D")
    Mp = mesh.assemble_M(S.MASS_PRIMAL); Mc = mesh.assemble_M(S.MASS_DUAL_LUMPED); mark("M")
    S.rhs(K, Mp, g, b); mark("rhs")
    rep = S.solve_gmres(V, b, wv, D=D, M=Mc, rel_tol=1e-10, max_iter=200, precond=1, history=False); mark("solve")
    torch.cuda.synchronize(); mark("sync")
    st = [A.stats() for A in (V, K, D)]; mark("stats")
    for A in (V, K, D, Mp, Mc): A.close()
    mark("close")
    mesh.close(); mark("mesh_close")
    torch.cuda.synchronize(); mark("end")
    print(" ".join(f"{k} {1e3*v:.1f}" for k, v in T.items()), flush=True)
