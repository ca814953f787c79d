"""Context for the paper's Table 2: D_h assembly wall time on the Table-1 meshes
(alpha = 10, L = 7 / 8: 65 536 / 262 144 space-time elements) on one B200, dense (symmetric packed)
storage, against the paper's Haswell-node timings (184.1 s on 1 node / 3.0 s on 64 nodes for L = 7;
373.6 s on 8 nodes for L = 8).  Prints one JSON line per level."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads.table1 as T
from paper_1811_05224_b200 import stbem as S

PAPER = {7: {"nodes_1": 184.1, "nodes_64": 3.0}, 8: {"nodes_8": 373.6, "nodes_128": 24.0}}
for L in [int(v) for v in (sys.argv[1:] or ["7", "8"])]:
    w = T.table1(L)
    m = S.Mesh.from_workload(w)
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        D = m.assemble_D()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        info = D.info()
        st = D.stats()
        if rep == 0:
            D.close()
    ent = w.n_gamma ** 2 * w.n_steps * (w.n_steps + 1) // 2
    print(json.dumps({"L": L, "N": w.n, "kappa": m.info.kappa, "D_assembly_s": ms / 1e3, "bytes": info["bytes"],
                      "entries_represented": ent, "entries_per_s": ent / (ms / 1e3),
                      "kernel_ms": {k: st[k] for k in ("ms_records", "ms_bulk", "ms_near", "ms_sing")},
                      "paper_s": PAPER.get(L)}), flush=True)
    D.close()
    m.close()
    S.lib().bem_release_storage()
