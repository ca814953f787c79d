"""per execution-count bucket: warp-level and thread-level instructions (SIMT efficiency) and stall samples"""
import csv, subprocess, sys
from collections import defaultdict
path = sys.argv[1]
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
ie, it, iss, isrc = h.index("Instructions Executed"), h.index("Thread Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
b = defaultdict(lambda: [0, 0, 0, 0, None])
tot_s = 0
for k, r in enumerate(rows[2:]):
    if len(r) != len(h): continue
    e, t, s = int(r[ie] or 0), int(r[it] or 0), int(r[iss] or 0)
    x = b[e]; x[0] += 1; x[1] += e; x[2] += t; x[3] += s; tot_s += s
    if x[4] is None: x[4] = k
for cnt, (n, e, t, s, first) in sorted(b.items(), key=lambda kv: -kv[1][3])[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"count {cnt:>10} n {n:4d} @{first:5d} simt {t / max(1, e) :5.1f} samples {s / tot_s:.3f}")
