"""stall samples and SIMT efficiency per CUDA source line of an ncu report (needs -lineinfo)"""
import csv, subprocess, sys
path = sys.argv[1]
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
res, fname = [], "?"
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 10 and r[0].isdigit() and r[2] == "-":
        try:
            s, e, t = int(r[4] or 0), int(r[7] or 0), int(r[8] or 0)
        except ValueError:
            continue
        res.append((s, fname, r[0], r[1][:100], e, t))
tot = sum(x[0] for x in res) or 1
for s, f, ln, src, e, t in sorted(res, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{s / tot:.3f} {f}:{ln:5s} simt {t / max(e, 1):4.1f} | {src}")
