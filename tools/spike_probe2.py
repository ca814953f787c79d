"""spike hunt: the bench step with/without the nvidia-smi sampler and with gc toggling"""
import sys, os, time, gc, subprocess, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from paper_1811_05224_b200 import stbem as S
w = W.get("C3")
g = torch.tensor(W.dirichlet_data(w), dtype=torch.float64, device="cuda")
b = torch.empty_like(g); wv = torch.empty_like(g)
mode = sys.argv[1]
proc = None
if "smi" in mode:
    proc = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,clocks_event_reasons.active",
                             "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    rows = []
    def rd():
        for line in proc.stdout:
            rows.append((time.perf_counter(), line.strip()))
    threading.Thread(target=rd, daemon=True).start()
if "nogc" in mode:
    gc.collect(); gc.disable()
t_start = time.perf_counter()
for it in range(10):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    t0 = time.perf_counter()
    ev[0].record()
    mesh = S.Mesh.from_workload(w)
    V = mesh.assemble_V(); ev[1].record()
    K = mesh.assemble_K(); ev[2].record()
    D = mesh.assemble_D(); ev[3].record()
    Mp = mesh.assemble_M(S.MASS_PRIMAL); Mc = mesh.assemble_M(S.MASS_DUAL_LUMPED)
    S.rhs(K, Mp, g, b); ev[4].record()
    rep = S.solve_gmres(V, b, wv, D=D, M=Mc, rel_tol=1e-10, max_iter=200, precond=1, history=False)
    ev[5].record(); ev[5].synchronize()
    st = {k: A.stats() for k, A in zip("VKD", (V, K, D))}
    for A in (V, K, D, Mp, Mc): A.close()
    mesh.close()
    dev = [ev[k].elapsed_time(ev[k + 1]) for k in range(5)]
    print(f"{mode} it {it} t={time.perf_counter()-t_start:.2f}s: phases {' '.join(f'{x:.1f}' for x in dev)} host {1e3*(time.perf_counter()-t0):.1f}", flush=True)
if proc:
    proc.terminate()
    print("smi samples:", [(round(t - t_start, 2), r) for t, r in rows][:60])
