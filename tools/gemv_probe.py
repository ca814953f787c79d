"""GEMV bandwidth probe on one assembled matrix (C3 V by default): CUDA-event timing, median of 20"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_1811_05224_b200 import stbem as S
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
w = W.get(name)
m = S.Mesh.from_workload(w)
A = m.assemble_V()
x = torch.tensor(W.random_vector(w.n), device="cuda"); y = torch.empty_like(x)
ts = []
for _ in range(25):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); A.matvec(x, y); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts[5:]))
nbytes = A.info()["bytes"] + 16 * w.n
print(f"{name} gemv median {ms:.3f} ms  {nbytes/ms/1e6:.1f} GB/s (bytes read: stored doubles of the packed V_h + 16 N)")
# pure-read reference: torch sum over a 16 GiB FP64 buffer
buf = torch.empty(2 * 1024**3, dtype=torch.float64, device="cuda").uniform_()
for _ in range(3): buf.sum()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): buf.sum()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"torch.sum over 16 GiB: {ms:.3f} ms  {buf.numel()*8/ms/1e6:.1f} GB/s")
