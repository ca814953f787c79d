#!/usr/bin/env bash
# One measurement pass of the round on a B200 (run under gpurun from the repo root):
#   bench lines (C3 default with cpu_baseline, C5, block-Toeplitz C3 / C4, the reference arm),
#   the ncu launch list of the default bench command (time shares, cold-cache and serialised),
#   and ncu --set full captures of the dominant kernels (GEMV, fused K g bulk, D bulk).
# Outputs under gpurun_out/prof/ (copied to profiles/ by hand after reading).
set -u
R=${1:-r01}
O=gpurun_out/prof
mkdir -p $O
python bench.py > $O/${R}_bench_C3.json 2> $O/bench_C3.err
python bench.py --config C5 --no-cpu-baseline > $O/${R}_bench_C5.json 2> $O/bench_C5.err
python bench.py --variant toeplitz --config C3 --no-cpu-baseline > $O/${R}_bench_toeplitz_C3.json 2> $O/tz3.err
python bench.py --variant toeplitz --config C4 --steps 5 --no-cpu-baseline > $O/${R}_bench_toeplitz_C4.json 2> $O/tz4.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/${R}_bench_reference_C3.json 2> $O/ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_launches_bench_C3.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
python tools/launch_summary.py $O/${R}_launches_bench_C3.csv > $O/${R}_launches_bench_C3_summary.txt
ncu --set full --clock-control none --import-source on -k regex:k_gemv_sym -s 3 -c 1 -o $O/gemv_sym \
    python tools/probe.py C3 V > $O/ncu_gemv.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bulk_m -c 1 -o $O/bulk_Kg \
    python tools/prof_probe.py C3 Kg > $O/ncu_kg.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bulk_m -c 1 -o $O/bulk_D \
    python tools/prof_probe.py C3 D > $O/ncu_d.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_toeplitz_mm -s 20 -c 1 -o $O/toeplitz_mm \
    python bench.py --variant toeplitz --config C4 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_tz.log 2>&1
echo done
