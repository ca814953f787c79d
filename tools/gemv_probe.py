"""GEMV bandwidth probe: V_h and D_h of the named configs (symmetric packed), CUDA-event timing of
one product (median of 20 after warm-up) and the bytes it reads (stored doubles + 16 N)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1811_05224_b200 import stbem as S  # noqa: E402

for name in (sys.argv[1:] or ["C3"]):
    w = W.get(name)
    m = S.Mesh.from_workload(w)
    x = torch.tensor(W.random_vector(w.n), device="cuda")
    y = torch.empty_like(x)
    for kind in "VD":
        A = getattr(m, f"assemble_{kind}")()
        ts = []
        for _ in range(25):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            A.matvec(x, y)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts[5:]))
        nbytes = A.info()["bytes"] + 16 * w.n
        print(f"{name} {kind} gemv median {ms:.3f} ms  {nbytes / 1e9:.2f} GB  {nbytes / ms / 1e6:.1f} GB/s", flush=True)
        A.close()
    m.close()
buf = torch.empty(2 * 1024**3, dtype=torch.float64, device="cuda").uniform_()
for _ in range(3):
    buf.sum()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    buf.sum()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"torch.sum over 16 GiB: {ms:.3f} ms  {buf.numel() * 8 / ms / 1e6:.1f} GB/s")
