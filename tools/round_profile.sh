#!/usr/bin/env bash
# One measurement pass of the round on a B200 (run under gpurun from the repo root):
#   bench lines (C5 default with cpu_baseline, C3, block-Toeplitz C3 / C4, the reference arm),
#   the ncu launch list of the default bench command (time shares, cold-cache and serialised),
#   and ncu --set full captures of the dominant kernels (GEMV, the three bulk kernels, D_h near
#   records), each after the same command ran without ncu.
# Outputs under gpurun_out/<R>/ (summaries copied to profiles/ after reading).
set -u
R=${1:-r02}
O=gpurun_out/$R
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
python bench.py > $O/${R}_bench_C5.json 2> $O/bench_C5.err
python bench.py --config C3 --no-cpu-baseline > $O/${R}_bench_C3.json 2> $O/bench_C3.err
python bench.py --variant toeplitz --config C3 --no-cpu-baseline --no-isolated > $O/${R}_bench_toeplitz_C3.json 2> $O/tz3.err
python bench.py --variant toeplitz --config C4 --steps 5 --no-cpu-baseline --no-isolated > $O/${R}_bench_toeplitz_C4.json 2> $O/tz4.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/${R}_bench_reference_C5.json 2> $O/ref.err
python tools/asm_probe.py C3 C5 > $O/${R}_asm_probe.txt 2>&1
python tools/gemv_probe.py C3 C5 > $O/${R}_gemv_probe.txt 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-isolated > $O/plain_bench.json 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_launches_bench_C5.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-isolated > $O/ncu_launch.log 2>&1
python tools/launch_summary.py $O/${R}_launches_bench_C5.csv > $O/${R}_launches_bench_C5_summary.txt
python tools/gemv_probe.py C5 > $O/plain_gemv.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_gemv_sym -s 5 -c 1 -o $O/gemv_C5 \
    python tools/gemv_probe.py C5 > $O/ncu_gemv.log 2>&1
for K in D Kg V; do
  python tools/prof_probe.py C5 $K > $O/plain_$K.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:k_bulk_m -c 1 -o $O/bulk_${K}_C5 \
      python tools/prof_probe.py C5 $K > $O/ncu_$K.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_records -s 1 -c 2 -o $O/rec_D_near_C5 \
    python tools/prof_probe.py C5 D > $O/ncu_rec.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_toeplitz_tma -s 4 -c 1 -o $O/toeplitz_C4 \
    python bench.py --variant toeplitz --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-isolated > $O/ncu_tz.log 2>&1
# text summaries on the box (gpurun copies back at most 64 MiB): keep the GEMV and K g reports
for f in $O/*.ncu-rep; do
  b=$(basename $f .ncu-rep)
  python tools/ncu_summary.py $f > $O/${R}_ncu_${b}.txt 2>&1
  python tools/ncu_lines.py $f 30 >> $O/${R}_ncu_${b}.txt 2>&1
  python tools/ncu_blocks.py $f 14 >> $O/${R}_ncu_${b}.txt 2>&1
done
rm -f $O/bulk_D_C5.ncu-rep $O/bulk_V_C5.ncu-rep $O/rec_D_near_C5.ncu-rep
echo done
