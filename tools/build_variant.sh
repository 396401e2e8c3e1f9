# Build libtmg_gpu.so with extra compile-time defines into OUT (for same-box
# A/B timing through TMG_LIB_PATH):  bash tools/build_variant.sh OUT -DNAME=V ...
out=$1; shift
python - "$out" "$@" <<'PY'
import subprocess, sys
sys.path.insert(0, ".")
from paper_2301_07457_b200 import build as b
out, defs = sys.argv[1], sys.argv[2:]
cmd = [b.NVCC, *b.ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
       *defs, "-o", out, *[str(b.CSRC / s) for s in b.SOURCES]]
subprocess.run(cmd, check=True)
PY
