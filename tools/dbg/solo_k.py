"""per-family kernel times of one solo rank (rank r of G, P = 2G) of a config: V_h, D_h, K_h g
python tools/dbg/solo_k.py C5 8 0"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1811_05224_b200 import stbem as S  # noqa: E402

name, G, r = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
entrywise = len(sys.argv) > 4 and sys.argv[4] == 'entrywise'
w = W.get(name)
for rep in range(2):
    c = S.Comm.solo(G, r, 0) if G > 1 else None
    m = S.Mesh.from_workload(w, n_slices=2 * G if G > 1 else 1, comm=c)
    Mp = m.assemble_M(S.MASS_PRIMAL)
    g = torch.tensor(W.dirichlet_data(w), dtype=torch.float64, device="cuda")
    b = torch.empty_like(g)
    st = S.rhs_fused(m, Mp, g, b, stats=True, entrywise=entrywise)
    torch.cuda.synchronize()
    V = m.assemble_V(); D = m.assemble_D(); torch.cuda.synchronize()
    if rep:
        for k, s in (("K", st), ("V", V.stats()), ("D", D.stats())):
            print(name, G, r, "entrywise" if entrywise else "table", k, {f: round(s[f], 3) for f in ("ms_records", "ms_bulk", "ms_near", "ms_sing")},
                  "launches", s.get("launches"), flush=True)
    V.close(); D.close(); Mp.close(); m.close()
    if c:
        c.close()
