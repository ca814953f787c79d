"""full-matrix parity of one library build against the oracle (A/B debugging of kernel variants):
python tools/dbg/lib_parity.py <dir with libstbem.so | default> MESH [MESH ...]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from oracle import oracle as O  # noqa: E402
from workloads.edge import edge_workloads  # noqa: E402
from paper_1811_05224_b200 import stbem as S  # noqa: E402

if sys.argv[1] != "default":
    S.LIB_PATH = os.path.join(sys.argv[1], "libstbem.so")
for name in sys.argv[2:]:
    w = W.get(name) if name in ("T8", "LT", "C1", "S32", "C2") else edge_workloads()[name]
    m = S.Mesh.from_workload(w)
    om = O.OracleMesh(w)
    for k in "VKD":
        A = getattr(m, f"assemble_{k}")()
        got, ref = A.dense(), om.dense(k)
        err = np.abs(got - ref).max() / np.abs(ref).max()
        i = np.unravel_index(np.argmax(np.abs(got - ref)), ref.shape)
        print(sys.argv[1], name, k, f"{err:.2e}", "at", i, "ng", w.n_gamma if hasattr(w, "n_gamma") else "", flush=True)
        A.close()
