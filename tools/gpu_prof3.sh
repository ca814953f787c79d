# ncu --set full of the bulk kernels (V, fused K g) on C5 (run under gpurun from the repo root)
set -u
O=gpurun_out/${1:-prof}
mkdir -p $O
for K in Kg V; do
  python tools/prof_probe.py C5 $K > $O/plain_$K.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:k_bulk_m -c 1 -o $O/bulk_${K}_C5 \
      python tools/prof_probe.py C5 $K > $O/ncu_$K.log 2>&1
done
echo done
