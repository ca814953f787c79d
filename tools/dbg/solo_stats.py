import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import workloads as W
from paper_1811_05224_b200 import stbem as S
w = W.get(sys.argv[1] if len(sys.argv) > 1 else "C5")
for G in (1, 2, 4, 8):
    c = S.Comm.solo(G, 0, 0) if G > 1 else None
    m = S.Mesh.from_workload(w, n_slices=2 * G if G > 1 else 1, comm=c)
    for k in "VD":
        for it in range(2):
            A = getattr(m, f"assemble_{k}")()
            torch.cuda.synchronize()
            st = A.stats()
            A.close()
        nb = sum(st["nodes_bulk"])
        print(G, k, "entries", m.info.entries_owned, "nodes_bulk", nb, "nodes/entry %.3f" % (nb / m.info.entries_owned),
              "ms_bulk %.3f" % st["ms_bulk"], "TF %.2f" % (st["flops_bulk"] / st["ms_bulk"] / 1e9),
              "ns/node %.4f" % (st["ms_bulk"] * 1e6 / nb), "B share %.3f" % (st["nodes_bulk"][1] / nb), flush=True)
    Mp = m.assemble_M(S.MASS_PRIMAL)
    g = torch.tensor(W.dirichlet_data(w), dtype=torch.float64, device="cuda")
    b = torch.empty_like(g)
    for it in range(2):
        st = S.rhs_fused(m, Mp, g, b, stats=True)
        torch.cuda.synchronize()
    nb = sum(st["nodes_bulk"])
    print(G, "K", "nodes/entry %.3f" % (nb / m.info.entries_owned), "ms_bulk %.3f" % st["ms_bulk"],
          "TF %.2f" % (st["flops_bulk"] / st["ms_bulk"] / 1e9), "ns/node %.4f" % (st["ms_bulk"] * 1e6 / nb), flush=True)
    Mp.close()
    m.close()
    if c: c.close()
