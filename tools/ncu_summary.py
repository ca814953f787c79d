"""print the key metrics of an ncu report (raw page): time, pipes, occupancy, stalls, DRAM"""
import csv, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
        "l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum", "lts__t_bytes.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {}
        for i, n in enumerate(h):
            if n in KEYS or (n.startswith("smsp__average_warp_latency_issue_stalled") and n.endswith(".ratio")) or \
               (n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("_not_issued")):
                d[n] = (v[i], u[i])
        res.append((v[h.index("Kernel Name")] if "Kernel Name" in h else "?", d))
    return res


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for name, d in summary(p):
            print("==", p, name[:90])
            stalls = []
            for k, (val, unit) in d.items():
                if "pcsamp" in k:
                    try:
                        stalls.append((float(val.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                    except ValueError:
                        pass
                else:
                    print(f"  {k} = {val} {unit}")
            stalls.sort(reverse=True)
            tot = sum(x for x, _ in stalls) or 1
            print("  stalls (pc samples):", ", ".join(f"{n} {100*x/tot:.0f}%" for x, n in stalls[:7]))
