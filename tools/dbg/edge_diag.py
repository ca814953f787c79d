"""diagnose edge-case parity: per kind the relative max-norm error and where it sits"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from workloads.edge import edge_workloads
from oracle import oracle as O
from paper_1811_05224_b200 import stbem as S
for name in sys.argv[1:]:
    w = edge_workloads()[name]
    om = O.OracleMesh(w)
    m = S.Mesh.from_workload(w)
    ng = w.n_gamma
    print(name, "ng", ng, "nt", w.n_steps, "q_bulk", m.info.q_bulk, "kappa", m.info.kappa)
    for kind in "VKD":
        for legacy in (False, True):
            A = getattr(m, f"assemble_{kind}")(legacy_sing=legacy)
            got = A.dense(); ref = om.dense(kind)
            d = np.abs(got - ref); k = np.unravel_index(np.argmax(d), d.shape)
            a, i_ = divmod(k[0], ng); b, j_ = divmod(k[1], ng)
            print(f"  {kind} legacy={legacy} rel {d.max()/np.abs(ref).max():.3e} at a={a} b={b} i={i_} j={j_} got {got[k]:.6e} ref {ref[k]:.6e} fused_sing {A.stats()['fused_sing']}")
