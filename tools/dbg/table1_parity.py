"""GPU vs oracle matrices on the paper's Table-1 levels (kappa = 20 2^-L)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import workloads.table1 as T
from oracle import oracle as O
from paper_1811_05224_b200 import stbem as S
for L in [int(v) for v in sys.argv[1:]]:
    w = T.table1(L)
    om = O.OracleMesh(w)
    m = S.Mesh.from_workload(w)
    out = []
    for k in "VKD":
        got = getattr(m, f"assemble_{k}")().dense(); ref = om.dense(k)
        out.append(f"{k} {np.abs(got - ref).max() / np.abs(ref).max():.2e}")
    print("L", L, "kappa", round(m.info.kappa, 3), "q_bulk", m.info.q_bulk, *out, flush=True)
