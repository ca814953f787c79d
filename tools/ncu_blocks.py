"""bucket the SASS of an ncu report by execution count (one bucket ~ one basic block family)"""
import csv, subprocess, sys
from collections import defaultdict

path = sys.argv[1]
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if "Address" in r)
h = rows[hi]
rows = rows[hi - 1:]
ia, isrc = h.index("Address"), h.index("Source")
iss, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
recs = [(int(r[ia], 16), r[isrc].strip(), int(r[iss] or 0), int(r[iex] or 0)) for r in rows[2:] if len(r) == len(h)]
tot_s = sum(r[2] for r in recs) or 1
tot_e = sum(r[3] for r in recs) or 1
print("total executed", tot_e, "samples", tot_s)
b = defaultdict(lambda: [0, 0, 0, None])
for k, r in enumerate(recs):
    x = b[r[3]]
    x[0] += 1; x[1] += r[3]; x[2] += r[2]
    if x[3] is None:
        x[3] = k
for cnt, (n, e, sm, first) in sorted(b.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    ops = defaultdict(int)
    for r in recs:
        if r[3] == cnt:
            ops[r[1].split()[0].lstrip("@!P0123456789 ").split(".")[0] if not r[1].startswith("@") else r[1].split()[1].split(".")[0]] += 1
    top = ", ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:6])
    print(f"count {cnt:>11}: {n:4d} instrs @{first:5d}, exec {e / tot_e:.3f}, samples {sm / tot_s:.3f} | {top}")
