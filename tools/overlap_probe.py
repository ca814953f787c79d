"""Probe: does an HBM-bound product (k_gemv_sym on V_h) overlap with an FP64-bound assembly (D_h)
on one B200?  Times (CUDA events) n products alone, one D_h assembly alone, and both launched
together on two streams.  Not part of the product; input for the DESIGN.md pipelining note."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1811_05224_b200 import stbem as S  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def main(name="C5", nprod=6, prio=0):
    w = W.get(name)
    m = S.Mesh.from_workload(w)
    V = m.assemble_V()
    x = torch.tensor(W.random_vector(w.n), dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream(priority=prio)   # prio -1: products first
    res = {}
    for rep in range(3):
        # products alone
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record(s2)
        for _ in range(nprod):
            V.matvec(x, y, stream=s2)
        b.record(s2)
        torch.cuda.synchronize()
        t_prod = a.elapsed_time(b)
        # assembly alone
        a, b = ev(), ev()
        a.record(s1)
        D = m.assemble_D(stream=s1)
        b.record(s1)
        torch.cuda.synchronize()
        t_asm = a.elapsed_time(b)
        D.close()
        # together
        torch.cuda.synchronize()
        a, b1, b2 = ev(), ev(), ev()
        a.record(s1)
        s2.wait_event(a)
        D = m.assemble_D(stream=s1)
        b1.record(s1)
        for _ in range(nprod):
            V.matvec(x, y, stream=s2)
        b2.record(s2)
        torch.cuda.synchronize()
        t_asm_c, t_prod_c = a.elapsed_time(b1), a.elapsed_time(b2)
        D.close()
        res = {"prio": prio, "prod_alone_ms": t_prod, "asm_alone_ms": t_asm, "sum_ms": t_prod + t_asm,
               "together_ms": max(t_asm_c, t_prod_c), "asm_done_ms": t_asm_c, "prod_done_ms": t_prod_c}
        print(json.dumps({k: round(v, 2) for k, v in res.items()}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C5", 6, int(sys.argv[2]) if len(sys.argv) > 2 else 0)
