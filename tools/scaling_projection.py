"""Projection (NOT a measurement) of the multi-GPU step from per-rank work measured on one GPU.

Every rank r of G (cyclic K_P plan, P = 2G temporal slices; P = 1 at G = 1) is run ALONE on the GPU
through a solo communicator (bem_comm_create_solo: the owned blocks only, partial products): its
V_h, D_h and K_h g assembly and its V_h, D_h products are timed with CUDA events.  The projected
step of G GPUs is
    max_r (assembly_r + n_V gemv_V,r + n_D gemv_D,r)  +  n_coll x t_allreduce  +  replicated vector work
with the products per solve of the measured single-GPU solve (n_matvec_V, n_matvec_D of its report), one
all-reduce of N doubles per product (t_allreduce ASSUMED, see --allreduce-us: NVLink all-reduce of
0.5-0.8 MB, latency-bound) and the replicated Krylov work taken from the single-GPU solve.  A solo
rank computes every pair record itself; with a real communicator the records of V_h and D_h are
split into G chunks and all-gathered (assemble.cu), which the projection models as
    records_r -> records_r / G + (G - 1) / G x record_bytes / --allgather-gbs
(record bytes from the field counts; V_h, D_h and K_h g alike, as `launch_assembly` splits every
kind's records over a real communicator).  The all-gathers run on each matrix's own assembly stream
while the other assemblies compute (bench.py's
step puts V_h, D_h and K_h g on three streams), so the default model takes a rank's assembly as
    max(sum of its kernel times,  the longest stream: records / G + all-gather + that matrix's kernels)
and `step_serial_s` keeps the pessimistic sum with the all-gathers serialised.  It shows the load
balance of the ownership plan with the real kernels; it is not a scaling measurement.

python tools/scaling_projection.py C5 [--allreduce-us 30]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1811_05224_b200 import stbem as S  # noqa: E402


# doubles per pair record, bulk + near fields (moments.cuh rec_fields + rec_fields_near)
# nf + nfn: rec_fields = RF_COMMON + n_fam FAMSZ, rec_fields_near = rec_fields + R2_FAM + n_fam R2_FAMSZ
REC_FIELDS = {"V": 144 + 262, "D": 283 + 515, "K": 144 + 262}


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e-3, out


def rank_work(w, G, r, pfac=2):
    c = S.Comm.solo(G, r, 0) if G > 1 else None
    m = S.Mesh.from_workload(w, n_slices=pfac * G if G > 1 else 1, comm=c)
    Mp = m.assemble_M(S.MASS_PRIMAL)
    g = torch.tensor(W.dirichlet_data(w), dtype=torch.float64, device="cuda")
    b = torch.empty_like(g)
    tV, V = timed(lambda: m.assemble_V())
    tD, D = timed(lambda: m.assemble_D())
    tK, stK = timed(lambda: S.rhs_fused(m, Mp, g, b, stats=True))
    x = torch.tensor(W.random_vector(w.n), dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    gv, gd = [], []
    for _ in range(6):
        gv.append(timed(lambda: V.matvec(x, y))[0])
        gd.append(timed(lambda: D.matvec(x, y))[0])
    stV, stD = V.stats(), D.stats()
    rec = 1e-3 * (stV["ms_records"] + stD["ms_records"] + stK["ms_records"])
    fam = {k: {f: round(st[f], 3) for f in ("ms_records", "ms_bulk", "ms_near", "ms_sing")}
           for k, st in (("V", stV), ("D", stD), ("K", stK))}
    out = {"assembly_s": tV + tD + tK, "asm": [tV, tD, tK], "records_s": rec, "kernels_ms": fam, "gemv_V_s": float(np.median(gv[1:])),
           "gemv_D_s": float(np.median(gd[1:])), "entries": m.info.entries_owned, "blocks": m.info.n_owned_blocks}
    V.close(); D.close(); Mp.close(); m.close()
    if c:
        c.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="C5")
    ap.add_argument("--allreduce-us", type=float, default=30.0)
    ap.add_argument("--allgather-gbs", type=float, default=400.0)   # ASSUMED NVLink all-gather bus bandwidth
    ap.add_argument("--pfac", type=int, default=2)   # P = pfac x G temporal slices
    args = ap.parse_args()
    w = W.get(args.config)
    # the single-GPU solve: iterations and the replicated (non-product) part of its time
    m = S.Mesh.from_workload(w)
    V, D = m.assemble_V(), m.assemble_D()
    Mp, Md = m.assemble_M(S.MASS_PRIMAL), m.assemble_M(S.MASS_DUAL)
    g = torch.tensor(W.dirichlet_data(w), dtype=torch.float64, device="cuda")
    b = torch.empty_like(g)
    S.rhs_fused(m, Mp, g, b)
    wv = torch.zeros_like(g)
    S.solve_gmres(V, b, wv, D=D, M=Md, precond=2, rel_tol=w.tol, history=False)   # warm
    rep = S.solve_gmres(V, b, wv, D=D, M=Md, precond=2, rel_tol=w.tol, history=False)
    it = rep["iterations"]
    n_v, n_d = rep["n_matvec_V"], rep["n_matvec_D"]
    replicated = rep["seconds_total"] - rep["seconds_matvec"]
    for A in (V, D, Mp, Md):
        A.close()
    m.close()
    res = {"config": args.config, "iterations": it, "replicated_solve_s": replicated,
           "allreduce_us_assumed": args.allreduce_us, "projection": {}}
    base = base_serial = None
    for G in (1, 2, 4, 8):
        rank_work(w, G, 0, args.pfac)   # warm-up: the storage of this size is mapped once (first touch)
        ranks = [rank_work(w, G, r, args.pfac) for r in range(G)]
        # distributed records: 1/G of the V_h, D_h records per rank plus their all-gather
        rec_bytes = 8.0 * w.n_gamma ** 2 * sum(REC_FIELDS.values())
        gather = (G - 1) / G * rec_bytes / (args.allgather_gbs * 1e9) if G > 1 else 0.0
        gshare = {k: REC_FIELDS[k] / sum(REC_FIELDS.values()) for k in "VDK"}
        per, per_serial = [], []
        for rk in ranks:
            rk["records_distributed_s"] = rk["records_s"] / G + gather
            compute = rk["assembly_s"] - rk["records_s"] + rk["records_s"] / G
            chains = [rk["asm"][i] - 1e-3 * rk["kernels_ms"][k]["ms_records"] * (1.0 - 1.0 / G) + gather * gshare[k]
                      for i, k in ((0, "V"), (1, "D"), (2, "K"))]
            rk["assembly_overlapped_s"] = max(compute, max(chains))
            prod = n_v * rk["gemv_V_s"] + n_d * rk["gemv_D_s"]
            per.append(rk["assembly_overlapped_s"] + prod)
            per_serial.append(rk["assembly_s"] - rk["records_s"] + rk["records_distributed_s"] + prod)
        n_coll = (n_v + n_d + 1) if G > 1 else 0   # one per product + the fused right-hand side
        step = max(per) + replicated + n_coll * args.allreduce_us * 1e-6
        step_serial = max(per_serial) + replicated + n_coll * args.allreduce_us * 1e-6
        base = base or step
        base_serial = base_serial or step_serial
        res["projection"][G] = {"step_s": step, "speedup": base / step, "max_rank_s": max(per),
                                "mean_rank_s": float(np.mean(per)), "imbalance": max(per) / float(np.mean(per)),
                                "step_serial_s": step_serial, "speedup_serial": base_serial / step_serial,
                                "ranks": ranks}
        print(f"{args.config} G={G}: projected step {1e3 * step:.1f} ms, speedup {base / step:.2f} "
              f"(all-gathers serialised: {base_serial / step_serial:.2f}), rank max/mean {max(per) / np.mean(per):.3f}",
              flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
