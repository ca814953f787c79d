"""parity of V/K/D against the oracle for several singular orders q_sing (edge workloads)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from workloads.edge import edge_workloads
from oracle import oracle as O
from paper_1811_05224_b200 import stbem as S
for name in sys.argv[1:]:
    w = edge_workloads()[name]
    om = O.OracleMesh(w)
    m = S.Mesh.from_workload(w)
    for qs in (12, 14, 16):
        out = []
        for k in "VKD":
            got = getattr(m, f"assemble_{k}")(q_sing=qs).dense(); ref = om.dense(k)
            out.append(f"{k} {np.abs(got - ref).max() / np.abs(ref).max():.2e}")
        print(name, "q_sing", qs, *out, flush=True)
