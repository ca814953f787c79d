"""assemble one matrix kind of a config once (for ncu --set full captures)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from paper_1811_05224_b200 import stbem as S
name, kind = sys.argv[1], sys.argv[2]
m = S.Mesh.from_workload(W.get(name))
A = getattr(m, f"assemble_{kind}")()
torch.cuda.synchronize()
print(name, kind, A.stats())
