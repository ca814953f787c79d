#!/usr/bin/env python
"""bench.py — one step = the whole hot path of arXiv:1811.05224 on one workload, by default the
largest BASELINE.json configuration that fits one GPU: configs[4], C5 (L-shape, 384 segments x
256 steps graded toward t = 0, N = 98 304, alpha = 0.5):
  mesh (a1) -> assemble V_h, D_h (a2, a3, a5) -> mass matrices (a6) -> b = 1/2 M g + K g with K_h
  computed and applied on the fly (a4, a7) -> GMRES to 1e-10 preconditioned by
  M_h^{-1} D_h M_h^{-T} with the exact dual mass (a8-a10; --precond 1: the lumped mass of P:185).

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference] [--config C5]
--gpus N > 1 without torchrun: the script re-launches itself under torch.distributed.run with N
ranks (one per GPU); P = 2N temporal slices owned by the cyclic K_P plan.  Prints ONE JSON line on
rank 0 (contract in the task statement / DESIGN.md section 6).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "element-pair integrals/s (assembly), matvec HBM GB/s, GMRES solve s at 1/2/4/8 GPU"
UNIT = "element-pair integrals/s"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
# FP64 DFMA peak: 148 SMs x 64 FP64 FMA/clk x 2 flop x 1.965 GHz (B200_PROFILING.md unit counts,
# MEASURED_PEAKS sm_max_mhz); tools/fp64_peak.cu measured 34.1 TFLOP/s on this pool (profiles/).
FP64_PEAK_DERIVED = 148 * 64 * 2 * 1.965e9 / 1e12
FP64_TC_PEAK = 37.1   # measured DMMA m8n8k4 throughput, profiles/r01_dmma_peak.txt
# the paper's own distributed-memory CPU timings, context only (other hardware, other workload:
# alpha = 10, the paper's Table-1 meshes): D_h assembly wall time, Table 2
PAPER_CONTEXT = {
    "source": "arXiv:1811.05224 Table 2 (PAPER.md P:212-240): D_h assembly wall time",
    "hardware": "Salomon cluster: 2x Intel Xeon E5-2680v3 (12-core Haswell) per node, 2 MPI x 12 OpenMP per node",
    "D_h_assembly_s": {"65536 elements, 1 node": 184.1, "65536 elements, 64 nodes": 3.0,
                       "262144 elements, 8 nodes": 373.6, "262144 elements, 128 nodes": 24.0,
                       "1048576 elements, 64 nodes": 747.0, "1048576 elements, 256 nodes": 193.5},
    "note": "context only, not a target (BASELINE.md section 1); this repo's L = 7 / 8 D_h on one B200: "
            "DESIGN.md section 6.1b"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)   # ~0.75 s timed: several nvidia-smi samples
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", default="C5")
    # 2: exact dual mass (cyclic-tridiagonal solves on the device, the north star's "sparse
    # mass-matrix solves"); 1: the lumped diagonal of P:185 (study in DESIGN.md section 6.2)
    ap.add_argument("--precond", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # uniform time steps only; avoids the dense work, reported as its own metric
    ap.add_argument("--variant", default="dense", choices=["dense", "toeplitz"])
    ap.add_argument("--overlap", type=int, default=1)   # V_h, D_h assembled on side streams
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-isolated", action="store_true")   # skip the serialised per-matrix pass
    return ap.parse_args()


def relaunch_distributed(args):
    """--gpus N > 1 outside torchrun: run this script under torch.distributed.run with N ranks (one
    process per GPU, rendezvous on 127.0.0.1) and return its exit code"""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def config_of(w, args, world):
    """the workload description shared by both arms (same keys, same values)"""
    names = "C1 C2 C3 C4 C5".split()
    idx = names.index(w.name) if w.name in names else "-"
    P = 1 if world == 1 else 2 * world
    return {"workload": f"BJ configs[{idx}] ({w.name}): {w.note}", "variant": args.variant,
            "n_gamma": w.n_gamma, "n_steps": w.n_steps, "N": w.n, "alpha": w.alpha,
            "slices_P": P, "gmres_tol": w.tol, "precond": ["none", "lumped", "exact"][args.precond],
            "parallelism": f"cyclic K_P plan, P = {P} temporal slices over {world} GPU" + ("s" if world > 1 else ""),
            "l2": "inputs larger than L2: V_h and D_h (symmetric packed) %.1f GB each >> 126 MB, streamed "
                  "once per product" % (8e-9 * w.n_gamma * (w.n_gamma + 32) / 2 * w.n_steps * (w.n_steps + 1) / 2)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region"""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([time.perf_counter()] + [x.strip() for x in line.split(",")])

    def window(self, t0, t1):
        """keep only the samples taken inside [t0, t1] (the timed region)"""
        self.t0, self.t1 = t0, t1

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        t0, t1 = getattr(self, "t0", -1e30), getattr(self, "t1", 1e30)
        rows = [r[1:] for r in self.rows if len(r) >= 8 and t0 <= r[0] <= t1]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------- oracle baseline
def cpu_baseline(w, seconds, steps=1, threads=None):
    """the oracle as it stands (oracle/stbem_oracle.c, OpenMP, all host cores or `threads`) on a
    bounded sample of the same workload: V, K, D entries of test row a = N_I/2 (random trial
    entries b <= a), sized to ~`seconds` of CPU work; value = entries computed per second."""
    from oracle import oracle as O
    all_threads = O.lib().ora_num_threads()
    if threads:
        O.lib().omp_set_num_threads(int(threads))   # libgomp, loaded with the oracle
    try:
        return _cpu_baseline(O, w, seconds)
    finally:
        if threads:
            O.lib().omp_set_num_threads(int(all_threads))


def _cpu_baseline(O, w, seconds):
    m = O.OracleMesh(w)
    ng, nt = w.n_gamma, w.n_steps
    a = nt // 2
    rng = np.random.default_rng(1811)
    # calibrate on a small sample, then size the timed sample
    def run(kind, cnt):
        rows = a * ng + rng.integers(0, ng, cnt)
        cols = rng.integers(0, (a + 1) * ng, cnt)
        t0 = time.perf_counter()
        m.entries(kind, rows, cols)
        return time.perf_counter() - t0
    per = {k: max(run(k, 2000), 1e-6) / 2000 for k in "VKD"}
    cost = sum(per.values())                      # seconds for one (V, K, D) entry triple
    triples = max(1000, int(seconds / cost))
    done, dt = 0, 0.0
    while dt < 0.67 * seconds and done < 50 * triples:   # the calibration can underestimate
        t0 = time.perf_counter()
        for k in "VKD":
            run(k, triples)
        dt += time.perf_counter() - t0
        done += triples
    return {"value": 3 * done / dt, "unit": UNIT, "cores": O.lib().ora_num_threads(), "kind": "oracle",
            "sample": f"{done} random entries each of V_h, K_h, D_h in test row a={a} of {w.name} "
                      f"(all b <= a), {dt:.1f} s", "seconds": dt, "cpu_model": cpu_model(),
            "host_cpus": os.cpu_count()}


# ---------------------------------------------------------------------- native step
def native(args):
    import torch
    import torch.distributed as dist

    import workloads as W
    from paper_1811_05224_b200 import stbem as S

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = S.Comm(rank, world, local) if world > 1 else None
    w = W.get(args.config)
    P = 1 if world == 1 else 2 * world
    dev = torch.device("cuda", local)
    g_host = torch.tensor(W.dirichlet_data(w), dtype=torch.float64).pin_memory()
    w_host = torch.empty(w.n, dtype=torch.float64).pin_memory()
    g = g_host.to(dev)
    b = torch.empty_like(g)
    wv = torch.empty_like(g)
    tol = w.tol
    Mkind = S.MASS_DUAL_LUMPED if args.precond == 1 else S.MASS_DUAL
    side = (torch.cuda.Stream(), torch.cuda.Stream())

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    def step(e2e):
        """one pass of the hot path; e2e: the host copies of the public API are inside"""
        ph = {}
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        ev[0].record()
        mesh = S.Mesh.from_workload(w, n_slices=P, comm=comm)
        gg = g
        if e2e:
            gg = torch.empty_like(g)
            gg.copy_(g_host, non_blocking=True)
        toep = args.variant == "toeplitz"
        cur = torch.cuda.current_stream()
        if args.overlap:
            # V_h and D_h on two side streams, concurrently with K_h g on the main stream: the
            # three assemblies are independent; the solve waits for all of them
            side[0].wait_stream(cur)
            side[1].wait_stream(cur)
            V = mesh.assemble_toeplitz("V", stream=side[0]) if toep else mesh.assemble_V(stream=side[0])
            D = mesh.assemble_toeplitz("D", stream=side[1]) if toep else mesh.assemble_D(stream=side[1])
            ev[1].record()
            ev[2].record()
        else:
            V = mesh.assemble_toeplitz("V") if toep else mesh.assemble_V()
            ev[1].record()
            D = mesh.assemble_toeplitz("D") if toep else mesh.assemble_D()
            ev[2].record()
        Mp = mesh.assemble_M(S.MASS_PRIMAL)
        Mc = mesh.assemble_M(Mkind) if args.precond else None
        if toep:
            Kt = mesh.assemble_toeplitz("K")
            S.rhs(Kt, Mp, gg, b)
            st_K = Kt.stats()
            Kt.close()
        else:
            # K_h is computed entry by entry and multiplied by g on the fly (never stored)
            st_K = S.rhs_fused(mesh, Mp, gg, b, stats=True)
        ev[3].record()
        if args.overlap:
            cur.wait_stream(side[0])
            cur.wait_stream(side[1])
        ev[4].record()
        rep = S.solve_gmres(V, b, wv, D=D if args.precond else None, M=Mc, rel_tol=tol, max_iter=200,
                            precond=args.precond, history=False)
        if e2e:
            w_host.copy_(wv, non_blocking=True)
        ev[5].record()
        ev[5].synchronize()
        ph["assemble_V"] = ev[0].elapsed_time(ev[1]) / 1e3
        ph["assemble_D"] = ev[1].elapsed_time(ev[2]) / 1e3
        ph["assemble_K"] = ev[2].elapsed_time(ev[3]) / 1e3     # fused K g (+ mass matrices)
        ph["rhs"] = ev[3].elapsed_time(ev[4]) / 1e3            # overlap: the wait for V_h, D_h
        ph["assembly"] = ev[0].elapsed_time(ev[4]) / 1e3
        ph["solve"] = ev[4].elapsed_time(ev[5]) / 1e3
        ph["total"] = ev[0].elapsed_time(ev[5]) / 1e3
        stats = {k: A.stats() for k, A in zip("VD", (V, D))}
        for k, A in zip("VD", (V, D)):
            stats[k]["bytes"] = A.info()["bytes"]
        stats["K"] = dict(st_K, bytes=0)
        for k in "VKD":
            ph[f"kern_{k}"] = (stats[k]["ms_records"] + stats[k]["ms_bulk"] + stats[k]["ms_near"] + stats[k]["ms_sing"]) / 1e3
        info = {f: getattr(mesh.info, f) for f, _ in mesh.info._fields_}
        for A in (V, D, Mp) + ((Mc,) if Mc else ()):
            A.close()
        mesh.close()
        return ph, rep, stats, info

    # the clock sampler (nvidia-smi) starts before the warm-up: its start-up stalls the driver for
    # ~0.1 s, which must not land in the timed region; only samples inside the region are kept
    clocks = ClockSampler(local)
    if rank == 0:
        clocks.start()
    for _ in range(args.warmup):
        step(False)
    barrier()
    S.launch_count(reset=True)
    # host jitter: a Python garbage collection during the timed steps stalls the enqueueing thread
    # (observed 70-130 ms once per run); collect now and pause the collector until the end
    import gc
    gc.collect()
    gc.disable()
    barrier()
    t_wall = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    phases, reps, stats = [], [], None
    step_wall = []
    for _ in range(args.steps):
        t_s = time.perf_counter()
        ph, rep, stats, info = step(False)
        step_wall.append(1e3 * (time.perf_counter() - t_s))
        phases.append(ph)
        reps.append(rep)
    e1.record()
    barrier()
    t_dev = e0.elapsed_time(e1) / 1e3
    launches = S.launch_count()
    wall = time.perf_counter() - t_wall
    # e2e: same step through the public API with host buffers (H2D of g, D2H of w inside)
    barrier()
    e2 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e2[0].record()
    e2e_wall = []
    for _ in range(args.steps):
        t_s = time.perf_counter()
        step(True)
        e2e_wall.append(1e3 * (time.perf_counter() - t_s))
    e2[1].record()
    barrier()
    t_e2e = e2[0].elapsed_time(e2[1]) / 1e3
    gc.enable()
    # after the timed regions: one serialised pass, each assembly alone on the GPU (the timed steps
    # overlap V_h and D_h with K_h g), for per-matrix seconds and the isolated kernel rates
    iso = None if args.no_isolated else isolated_pass(S, w, P, comm, g, b, args)
    if rank == 0:
        clocks.window(t_wall, time.perf_counter())
    ck = clocks.stop() if rank == 0 else None
    if world > 1:
        tt = torch.tensor([t_dev, t_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_dev, t_e2e = tt.tolist()
    entries_total = info["entries_total"]
    # units: the distinct element-pair integrals computed and stored per step (V_h and D_h keep the
    # N_Gamma (N_Gamma + 1) / 2 distinct entries of their symmetric spatial blocks, K_h all); the matrix
    # entries they represent (3 x entries_total) are reported beside
    units_per_step = sum(stats[k]["entries"] for k in "VKD")   # this rank's owned blocks
    if world > 1:   # whole-job units: every rank computes the integrals of its own blocks
        uu = torch.tensor([float(units_per_step)], dtype=torch.float64, device=dev)
        dist.all_reduce(uu, op=dist.ReduceOp.SUM)
        units_per_step = uu.item()
    represented_per_step = 3 * entries_total
    ms = 1e3 * t_dev / args.steps
    value = units_per_step * args.steps / t_dev
    e2e = units_per_step * args.steps / t_e2e
    ph = {k: float(np.median([p[k] for p in phases])) for k in phases[0]}
    rep = reps[-1]
    # GEMV bandwidth: algorithmic bytes per product = 8 * stored entries (owned) + 16 N
    n = w.n
    # bytes actually read per product of the solve (V_h and D_h alternate) + x and y
    bytes_per_gemv = (rep["n_matvec_V"] * stats["V"]["bytes"] + rep["n_matvec_D"] * stats["D"]["bytes"]) / \
        max(1, rep["n_matvec_V"] + rep["n_matvec_D"]) + 16 * n
    n_mv = rep["n_matvec_V"] + rep["n_matvec_D"]
    gemv_s = rep["seconds_matvec"] / max(1, n_mv)
    peaks = json.load(open(PEAKS_PATH)) if os.path.exists(PEAKS_PATH) else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    gemv_gbs = bytes_per_gemv / gemv_s / 1e9 if gemv_s > 0 else None
    # assembly roofline: the longest bulk kernel (k_bulk_m<KIND>), FP64 flops from the exact
    # per-regime node counts x the static FP64 counts of the shipped forms,
    # and its store stream (8 B per stored entry)
    # (the isolated pass when it ran: each assembly alone on the GPU; else the timed steps' own
    # kernel events, taken while V_h, D_h and K_h g overlap)
    src = iso["stats"] if iso else stats
    fam = []
    for k in "VKD":
        st = src[k]
        fam.append((st["ms_bulk"], k, "bulk", st))
    ms_dom, kdom, _, st = max(fam)
    flops = st["flops_bulk"]
    achieved = flops / (ms_dom * 1e-3) / 1e12
    all_bulk_flops = sum(src[k]["flops_bulk"] for k in "VKD")
    all_bulk_ms = sum(src[k]["ms_bulk"] for k in "VKD")
    nt_ = w.n_steps
    cells = nt_ * (nt_ + 1) / 2
    bulk_entries = stats[kdom]["entries"] * (cells - (2 * nt_ - 1)) / cells   # stored entries of cells d >= 2
    store_gbs = 8.0 * bulk_entries / (ms_dom * 1e-3) / 1e9
    # ncu dram__bytes_read.sum + dram__bytes_write.sum per launch of the same kernel on the same
    # config (profiles/traffic.json, from the committed ncu summaries), None where not captured
    traffic = {}
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        for tj in json.load(open(tpath))["entries"]:
            if tj.get("config") == args.config:
                traffic[tj["kernel"]] = tj["traffic_bytes_per_launch"]
    try:
        # context for the isolated pass (skipped with it: a launch-list run measures the step only)
        fp64_live = S.diag_fp64_rate(2.0) if (args.variant != "toeplitz" and iso) else None
    except Exception:
        fp64_live = None
    roof_asm = {"bound": "alu", "kernel": f"k_bulk_m<{kdom}>", "achieved": achieved, "peak": FP64_PEAK_DERIVED,
                "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_DERIVED,
                "traffic": traffic.get(f"k_bulk_m<{kdom}>"),
                "store_gbs": store_gbs, "store_frac_of_hbm": store_gbs / hbm_peak,
                "peak_note": "FP64 DFMA: 148 SM x 64 FMA/clk x 2 x 1.965 GHz (derived from the guide's unit counts "
                             "and MEASURED_PEAKS sm_max_mhz); tools/fp64_peak.cu measured 34.1 TFLOP/s",
                "flops_per_launch": flops, "node_evals_per_launch": st["evals_bulk"],
                "timing": "isolated (serialised pass after the timed region)" if iso else "inside the overlapped step",
                "all_bulk_kernels": {"flops": all_bulk_flops, "ms": all_bulk_ms,
                                     "tflops": all_bulk_flops / (all_bulk_ms * 1e-3) / 1e12,
                                     "frac": all_bulk_flops / (all_bulk_ms * 1e-3) / 1e12 / FP64_PEAK_DERIVED},
                "nodes_by_regime_ABZC": st["nodes_bulk"],
                "peak_live_sustained": fp64_live,
                "frac_of_live_sustained": (achieved / fp64_live) if fp64_live else None,
                "live_note": "bem_diag_fp64_rate: a DFMA loop back to back for 2 s right after the isolated pass "
                             "(the same power / thermal state; the board power cap lowers the FP64 clock), "
                             "context for frac, which stays against the max-clock peak",
                "flops_note": "algorithmic: exact per-regime node counts x static FP64 flops of the shipped "
                              "moment forms (DFMA = 2), DESIGN.md section 6"}
    roof_gemv = {"bound": "hbm", "kernel": "k_gemv_sym", "achieved": gemv_gbs, "peak": hbm_peak, "unit": "GB/s",
                 "frac": (gemv_gbs / hbm_peak) if gemv_gbs else None, "traffic": traffic.get("k_gemv_sym"),
                 "bytes_per_launch": bytes_per_gemv,
                 "peak_note": "MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)",
                 "bytes_note": "algorithmic: 8 B per stored double of the product's matrix (block lower "
                               "triangle; V_h / D_h symmetric packed spatial blocks) + 16 N"}
    if args.variant == "toeplitz":
        # the product is the FP64 tensor-core GEMM k_toeplitz_tma (TMA-staged DMMA): algorithmic flops per product
        # 2 ng^2 sum_a (a + 1) (the block lower triangle of lags) against the measured DMMA peak
        ng_, nt_t = w.n_gamma, w.n_steps
        fl = 2.0 * ng_ * ng_ * nt_t * (nt_t + 1) / 2
        tf = fl / gemv_s / 1e12 if gemv_s > 0 else None
        roof_gemv = {"bound": "tensor", "kernel": "k_toeplitz_tma<256,32,3>", "achieved": tf, "peak": FP64_TC_PEAK,
                     "unit": "TFLOP/s", "frac": (tf / FP64_TC_PEAK) if tf else None,
                     "traffic": traffic.get("k_toeplitz_tma"),
                     "flops_per_launch": fl,
                     "peak_note": "FP64 tensor cores (DMMA m8n8k4) measured 37.1 TFLOP/s on this pool's B200 "
                                  "(profiles/r01_dmma_peak.txt; DFMA 34.1)",
                     "flops_note": "algorithmic: 2 ng^2 per (row block a, lag d <= a) pair, per product; "
                                   "time = the solve's products incl. the fixed-order partial reduction"}
    # context for the HBM roofline: MEASURED_PEAKS hbm_gbs is a copy (read + write) figure; a pure
    # streaming read (torch.sum over 8 GiB, after the timed region) can exceed it
    try:
        if args.variant == "toeplitz":
            raise RuntimeError("no HBM roofline for the tensor-bound variant")
        buf = torch.empty(1024 ** 3, dtype=torch.float64, device=dev).fill_(1.0)
        for _ in range(2):
            buf.sum()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record()
        for _ in range(5):
            buf.sum()
        r1.record()
        r1.synchronize()
        read_gbs = 5 * buf.numel() * 8 / (r0.elapsed_time(r1) * 1e-3) / 1e9
        del buf
    except Exception:
        read_gbs = None
    roof_gemv["read_peak_live_gbs"] = read_gbs
    roof_gemv["frac_of_read_peak"] = (gemv_gbs / read_gbs) if (gemv_gbs and read_gbs) else None
    # the dominant kernel of the step by device time: the GEMV (all products of the solve) or the
    # longest assembly kernel
    gemv_total_ms = 1e3 * rep["seconds_matvec"]
    roofline = roof_gemv if gemv_total_ms >= ms_dom else roof_asm
    roofline = dict(roofline, share_of_step=(gemv_total_ms if roofline is roof_gemv else ms_dom) / ms)
    asm_s = ph["assembly"]          # mesh -> V_h, D_h, K_h g all done (overlapped or not)
    out = {
        "metric": METRIC + (" [block-Toeplitz variant, SURVEY 8(f) f3]" if args.variant == "toeplitz" else ""),
        "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(w, args, world),
        "components": {
            "assembly_pairs_per_s": units_per_step / asm_s,
            "integrals_per_step": {k: stats[k]["entries"] for k in "VKD"},
            "matrix_entries_represented_per_s": represented_per_step / (1e-3 * ms),
            "storage": "V_h, D_h: symmetric packed spatial blocks (upper triangle: 32x32 tiles, triangular "
                       "diagonal tiles); K_h computed and applied to g on the fly (bem_rhs_fused), never stored",
            "assembly_s": {"all_in_step": ph["assembly"],
                           "isolated": iso["seconds"] if iso else None,
                           "isolated_pairs_per_s": iso["pairs_per_s"] if iso else None,
                           "note": "all_in_step: mesh -> V_h, D_h (side streams) and K_h g done, median of the timed "
                                   "steps; isolated: each matrix assembled alone after the timed region (CUDA events "
                                   "on its stream, mesh and mass matrices excluded)"},
            "matvec_gbs": gemv_gbs, "matvec_frac_of_hbm": (gemv_gbs / hbm_peak) if gemv_gbs else None,
            "gmres_solve_s": ph["solve"], "gmres_iterations": rep["iterations"],
            "gmres_true_rel_residual": rep["true_rel_residual"], "time_to_solution_s": ph["total"],
            # per-kernel-class device ms of each matrix: from the isolated pass when it ran (each class's
            # events on an otherwise idle GPU); inside the overlapped step the events of one stream also
            # span the other streams' kernels, so those are reported apart and only as an upper bound
            "kernel_ms": {k: {"records": src[k]["ms_records"], "bulk": src[k]["ms_bulk"], "near": src[k]["ms_near"],
                              "sing": src[k]["ms_sing"]} for k in "VKD"},
            "kernel_ms_timing": "isolated (serialised pass after the timed region)" if iso else "inside the overlapped step",
            "kernel_ms_in_step_overlapped": {k: {"records": stats[k]["ms_records"], "bulk": stats[k]["ms_bulk"],
                                                 "near": stats[k]["ms_near"], "sing": stats[k]["ms_sing"]}
                                             for k in "VKD"},
            # time to solution against its roofline: the bulk kernels' algorithmic flops at the FP64
            # peak plus the solve's products' bytes at the HBM peak (near cells, records and the
            # Krylov vector kernels counted as zero)
            "time_to_solution_roofline": None if args.variant == "toeplitz" else {
                "ideal_s": all_bulk_flops / (FP64_PEAK_DERIVED * 1e12) + n_mv * bytes_per_gemv / (hbm_peak * 1e9),
                "frac": (all_bulk_flops / (FP64_PEAK_DERIVED * 1e12) + n_mv * bytes_per_gemv / (hbm_peak * 1e9)) / ph["total"],
                "note": "ideal = bulk-assembly flops / FP64 peak + products x bytes / MEASURED_PEAKS hbm_gbs"},
        },
        "roofline": roofline,
        "paper_context": PAPER_CONTEXT,
        "roofline_gemv": roof_gemv,
        "roofline_assembly": roof_asm,
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n},
        "gpu_launches": int(launches),
        "host_step_ms": {"device_timed": [round(x, 2) for x in step_wall], "e2e": [round(x, 2) for x in e2e_wall]},
        "phases_ms": [{k: round(1e3 * v, 2) for k, v in p.items()} for p in phases],
        "clocks": ck,
        "wall_s": wall,
    }
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(w, args.cpu_seconds)
            one = cpu_baseline(w, max(3.0, args.cpu_seconds / 3), threads=1)
            out["cpu_baseline"]["single_thread"] = {"value": one["value"], "cores": 1, "sample": one["sample"]}
        print(json.dumps(out), flush=True)
    if comm:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


def isolated_pass(S, w, P, comm, g, b, args):
    """each matrix assembled alone (serialised, synchronised), timed with CUDA events on the
    launching stream: per-matrix seconds, pairs/s and the kernel statistics of that assembly"""
    import torch
    mesh = S.Mesh.from_workload(w, n_slices=P, comm=comm)
    Mp = mesh.assemble_M(S.MASS_PRIMAL)
    torch.cuda.synchronize()
    out = {"seconds": {}, "pairs_per_s": {}, "stats": {}}
    toep = args.variant == "toeplitz"
    for k in "VDK":
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if k == "K" and not toep:
            st = S.rhs_fused(mesh, Mp, g, b, stats=True)      # K_h g, K_h never stored (as in the step)
            e1.record()
        else:
            A = mesh.assemble_toeplitz(k) if toep else getattr(mesh, f"assemble_{k}")()
            e1.record()
            st = A.stats()
            A.close()
        e1.synchronize()
        sec = e0.elapsed_time(e1) / 1e3
        out["seconds"][k] = sec
        out["pairs_per_s"][k] = st["entries"] / sec
        out["stats"][k] = st
    Mp.close()
    mesh.close()
    torch.cuda.synchronize()
    return out


# ---------------------------------------------------------------------- reference arm
def reference(args):
    """the oracle (this tier's reference arm) on the host cores, same config/metric/unit; each step
    is a bounded sample of the workload (rank 0 only; other ranks exit 0)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import workloads as W
    w = W.get(args.config)
    per_step = max(3.0, 60.0 / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        cpu_baseline(w, per_step / 3)
    vals, secs = [], []
    for _ in range(args.steps):
        r = cpu_baseline(w, per_step)
        vals.append(r["value"])
        secs.append(r["seconds"])
    v = float(np.median(vals))
    out = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.median(secs)),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "impl": "reference",
           "config": config_of(w, args, int(os.environ.get("WORLD_SIZE", "1"))),
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": r["cores"], "kind": "oracle", "sample": r["sample"],
                            "cpu_model": r["cpu_model"], "host_cpus": r["host_cpus"]},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(a))
    if a.impl == "reference":
        reference(a)
    else:
        native(a)
