# A/B of the bulk kernels under an environment variable ($1=VAR=value)
for e in "" "$1" "" "$1"; do
  env $e python tools/asm_probe.py C5 2>&1 | grep "C5 [VDK]" | sed "s/^/[$e] /"
done
