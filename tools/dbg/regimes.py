"""regime statistics of V/K/D assembly on a Table-1 level (alpha = 10) or a named workload"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import workloads as W
import workloads.table1 as T
from paper_1811_05224_b200 import stbem as S
arg = sys.argv[1]
w = T.table1(int(arg[1:])) if arg.startswith("L") else W.get(arg)
m = S.Mesh.from_workload(w)
for k in sys.argv[2] if len(sys.argv) > 2 else "VKD":
    for rep in range(2):
        A = getattr(m, f"assemble_{k}")()
        torch.cuda.synchronize()
        st = A.stats()
        A.close()
    nb, nn = st["nodes_bulk"], st["nodes_near"]
    print(k, "bulk ABZC", [round(v / max(1, sum(nb)), 5) for v in nb], "near ABZC", [round(v / max(1, sum(nn)), 5) for v in nn],
          "ms rec %.2f bulk %.2f near %.2f sing %.2f" % (st["ms_records"], st["ms_bulk"], st["ms_near"], st["ms_sing"]), flush=True)
