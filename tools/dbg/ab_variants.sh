# A/B of the bulk kernels: the in-tree library against every tools/dbg/alt_<i>/libstbem.so, twice,
# interleaved ($1: config, default C5)
C=${1:-C5}
for rep in 1 2; do
  for lib in default tools/dbg/alt_*; do
    STB_ALT=$lib STB_CFG=$C python - <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
from paper_1811_05224_b200 import stbem as S
alt = os.environ["STB_ALT"]
tag = "default" if alt == "default" else open(os.path.join(alt, "flags.txt")).read().strip()
if alt != "default":
    S.LIB_PATH = os.path.join(alt, "libstbem.so")
sys.argv = ["asm_probe", os.environ["STB_CFG"]]
import io, contextlib
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    exec(open("tools/asm_probe.py").read())
for line in buf.getvalue().splitlines():
    if line.startswith(os.environ["STB_CFG"] + " "):
        print(f"[{tag}] {line}", flush=True)
PY
  done
done
