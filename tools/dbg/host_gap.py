"""host-side cost of the pieces between two bench steps (C5): mesh creation, stats, closes"""
import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
import workloads as W
from paper_1811_05224_b200 import stbem as S
w = W.get(sys.argv[1] if len(sys.argv) > 1 else "C5")
g = torch.tensor(W.dirichlet_data(w), dtype=torch.float64, device="cuda")
b = torch.empty_like(g)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mesh = S.Mesh.from_workload(w)
    t1 = time.perf_counter()
    V = mesh.assemble_V(); t2 = time.perf_counter()
    D = mesh.assemble_D(); t3 = time.perf_counter()
    Mp = mesh.assemble_M(S.MASS_PRIMAL); Mc = mesh.assemble_M(S.MASS_DUAL); t4 = time.perf_counter()
    st = S.rhs_fused(mesh, Mp, g, b, stats=True); t5 = time.perf_counter()
    torch.cuda.synchronize(); t6 = time.perf_counter()
    sv, sd = V.stats(), D.stats(); iv, idd = V.info(), D.info(); t7 = time.perf_counter()
    info = {f: getattr(mesh.info, f) for f, _ in mesh.info._fields_}; t8 = time.perf_counter()
    for A in (V, D, Mp, Mc):
        A.close()
    t9 = time.perf_counter()
    mesh.close(); t10 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"mesh {1e3*(t1-t0):.2f} V-enq {1e3*(t2-t1):.2f} D-enq {1e3*(t3-t2):.2f} M {1e3*(t4-t3):.2f} Kg(sync) {1e3*(t5-t4):.2f} "
          f"stats {1e3*(t7-t6):.2f} info {1e3*(t8-t7):.2f} close {1e3*(t9-t8):.2f} mesh.close {1e3*(t10-t9):.2f}")
