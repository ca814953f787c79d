# A/B of the bulk kernels: in-tree libstbem.so vs an alternative build ($1: directory with libstbem.so)
for lib in default $1 default $1; do
  STB_ALT=$lib python - <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
from paper_1811_05224_b200 import stbem as S
alt = os.environ["STB_ALT"]
if alt != "default":
    S.LIB_PATH = os.path.join(alt, "libstbem.so")
    import ctypes
    _L = ctypes.CDLL(S.LIB_PATH)
    for _n in list(S._SIGS):          # an older library: drop the entry points it does not have
        if not hasattr(_L, _n):
            del S._SIGS[_n]
sys.argv = ["asm_probe", "C5"]
print("LIB", alt, flush=True)
exec(open("tools/asm_probe.py").read())
PY
done
