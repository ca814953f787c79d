"""assembly kernel timing probe: V_h, D_h and the fused K_h g of the named configs, each assembled
alone three times; median device times per kernel family (CUDA events, bem_matrix_stats) and the
bulk kernels' algorithmic FP64 rate"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1811_05224_b200 import stbem as S  # noqa: E402

PEAK = 148 * 64 * 2 * 1.965e9 / 1e12
out = {}
for name in (sys.argv[1:] or ["C3", "C5"]):
    w = W.get(name)
    m = S.Mesh.from_workload(w)
    Mp = m.assemble_M(S.MASS_PRIMAL)
    g = torch.tensor(W.dirichlet_data(w), dtype=torch.float64, device="cuda")
    b = torch.empty_like(g)
    res = {}
    for k in "VDK":
        rows = []
        for rep in range(3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if k == "K":
                st = S.rhs_fused(m, Mp, g, b, stats=True)
                e1.record()
            else:
                A = getattr(m, f"assemble_{k}")()
                e1.record()
                st = A.stats()
                A.close()
            e1.synchronize()
            rows.append((e0.elapsed_time(e1), st))
        ms = float(np.median([r[0] for r in rows]))
        st = rows[-1][1]
        bulk = float(np.median([r[1]["ms_bulk"] for r in rows]))
        nb = st["nodes_bulk"]
        res[k] = {"ms": round(ms, 3), "bulk": round(bulk, 3), "near": round(st["ms_near"], 3),
                  "rec": round(st["ms_records"], 3), "sing": round(st["ms_sing"], 3),
                  "tflops_bulk": round(st["flops_bulk"] / bulk / 1e9, 2),
                  "frac": round(st["flops_bulk"] / bulk / 1e9 / PEAK, 3),
                  "B_share": round(nb[1] / max(1, sum(nb)), 4)}
        print(name, k, json.dumps(res[k]), flush=True)
    out[name] = res
    m.close()
print(json.dumps(out))
