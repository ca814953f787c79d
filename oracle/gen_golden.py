"""Write oracle reference solutions under tests/golden/ (calls only oracle/ and the shared
input generators in workloads/).  Test infrastructure.

python -m oracle.gen_golden C2     (V_h, K_h at C2: ~4 min on 8 cores)
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402
from oracle import oracle as O  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def main(name):
    w = W.get(name)
    t0 = time.time()
    m = O.OracleMesh(w)
    V = m.dense("V")
    K = m.dense("K")
    g = W.dirichlet_data(w)
    b = m.rhs(K, g)
    wd = O.block_forward_solve(V, b, m.ng)
    e, r = m.l2_error(wd)
    os.makedirs(GOLDEN, exist_ok=True)
    np.save(os.path.join(GOLDEN, f"{name}_oracle_b.npy"), b)
    np.save(os.path.join(GOLDEN, f"{name}_oracle_w.npy"), wd)
    meta = {"config": name, "n": int(m.n), "l2_rel_error_w": float(e / r), "seconds": time.time() - t0,
            "source": "oracle/gen_golden.py: oracle V_h, K_h (stbem_oracle.c), b = (1/2 M_h + K_h) g, "
                      "w = block forward substitution of V_h w = b (P:83, P:151-159)"}
    with open(os.path.join(GOLDEN, f"{name}_oracle.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(meta)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C2")
