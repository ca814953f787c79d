"""quick timing probe: assemble V/K/D of a config on cuda:0 (twice; stats of the second), one GEMV"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_1811_05224_b200 import stbem as S
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
kinds = sys.argv[2] if len(sys.argv) > 2 else "VKD"
w = W.get(name)
m = S.Mesh.from_workload(w)
print(name, "ng", m.ng, "nt", m.nt, "q_bulk", m.info.q_bulk, "kappa", round(m.info.kappa, 4), "entries", m.info.entries_total, flush=True)
mats = {}
for k in kinds:
    for rep in range(2):
        mats[k] = None
        torch.cuda.synchronize(); t = time.time()
        mats[k] = getattr(m, f"assemble_{k}")()
        torch.cuda.synchronize(); dt = time.time() - t
    st = mats[k].stats()
    nb, nn = st["nodes_bulk"], st["nodes_near"]
    fb = [v / max(1, sum(nb)) for v in nb]
    fn = [v / max(1, sum(nn)) for v in nn]
    print(f"assemble {k}: {dt:.3f} s  {st['entries']/dt/1e9:.3f} G computed entries/s | ms rec {st['ms_records']:.2f} "
          f"bulk {st['ms_bulk']:.2f} near {st['ms_near']:.2f} sing {st['ms_sing']:.2f} | bulk regimes A/B/Z/C "
          f"{fb[0]:.4f}/{fb[1]:.4f}/{fb[2]:.4f}/{fb[3]:.5f} near {fn[0]:.3f}/{fn[1]:.3f}/{fn[2]:.3f}/{fn[3]:.4f}", flush=True)
x = torch.tensor(W.random_vector(w.n), device="cuda"); y = torch.empty_like(x)
A = mats[kinds[0]]
for _ in range(3): A.matvec(x, y)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): A.matvec(x, y)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
nbytes = A.info()["bytes"] + 16 * w.n   # stored doubles (symmetric packed V_h / D_h) + x and y
print(f"gemv {ms:.3f} ms  {nbytes/ms/1e6:.1f} GB/s (bytes read: stored entries + 16 N)", flush=True)
