# ncu evidence for one round step (run under gpurun from the repo root):
#   launch list of the default bench command (C5), ncu --set full of the three bulk kernels on C5
set -u
O=gpurun_out/${1:-prof}
mkdir -p $O
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-isolated > $O/plain_bench.json 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_C5.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-isolated > $O/ncu_launch.log 2>&1
for K in D Kg V; do
  python tools/prof_probe.py C5 $K > $O/plain_$K.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:k_bulk_m -c 1 -o $O/bulk_${K}_C5 \
      python tools/prof_probe.py C5 $K > $O/ncu_$K.log 2>&1
done
echo done
