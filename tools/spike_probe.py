"""repeat the bench step and report per-phase device time and kernel-family times (spike hunt)"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from paper_1811_05224_b200 import stbem as S
w = W.get(sys.argv[1] if len(sys.argv) > 1 else "C3")
g = torch.tensor(W.dirichlet_data(w), dtype=torch.float64, device="cuda")
b = torch.empty_like(g); wv = torch.empty_like(g)
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 10):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    th = [time.perf_counter()]
    ev[0].record()
    mesh = S.Mesh.from_workload(w); th.append(time.perf_counter())
    V = mesh.assemble_V(); ev[1].record(); th.append(time.perf_counter())
    K = mesh.assemble_K(); ev[2].record(); th.append(time.perf_counter())
    D = mesh.assemble_D(); ev[3].record(); th.append(time.perf_counter())
    Mp = mesh.assemble_M(S.MASS_PRIMAL); Mc = mesh.assemble_M(S.MASS_DUAL_LUMPED)
    S.rhs(K, Mp, g, b); ev[4].record()
    rep = S.solve_gmres(V, b, wv, D=D, M=Mc, rel_tol=1e-10, max_iter=200, precond=1, history=False)
    ev[5].record(); torch.cuda.synchronize(); th.append(time.perf_counter())
    dev = [ev[0].elapsed_time(ev[k]) for k in range(1, 6)]
    st = {k: A.stats() for k, A in zip("VKD", (V, K, D))}
    fam = " ".join(f"{k}:{s['ms_records']:.1f}/{s['ms_bulk']:.1f}/{s['ms_near']:.1f}/{s['ms_sing']:.2f}" for k, s in st.items())
    hst = " ".join(f"{1e3*(th[i+1]-th[i]):.1f}" for i in range(len(th) - 1))
    print(f"it {it}: dev cum {' '.join(f'{x:.1f}' for x in dev)} | kernels rec/bulk/near/sing {fam} | host {hst}", flush=True)
    for A in (V, K, D, Mp, Mc): A.close()
    mesh.close()
