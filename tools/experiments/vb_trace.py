#!/usr/bin/env python3
"""Stage times of k_vbottom (a TMG_VB_TRACE build through TMG_LIB_PATH)."""
import ctypes as C, pathlib, sys
import numpy as np
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2301_07457_b200 as P  # noqa: E402
cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
nx, ny, nc, recipe, seed, desc = bench.CONFIGS[cfg]
g, bc, E, b = bench.make_inputs(nx, ny, recipe, seed)
ops = P.MultigridOperators(g, nc, 0.3, bc)
ops.set_moduli(E, bench.OMEGA)
f = np.random.default_rng(0).standard_normal(b.size)
for _ in range(3):
    P.mg_cycle(ops, np.zeros_like(f), f)
t = (C.c_ulonglong * 64)()
assert P._lib.load().tmg_debug_vb_trace(t) == 0
v = np.array(t[:], dtype=np.int64); v = v[v > 0]
print(cfg, "stage ns:", " ".join(str(x) for x in np.diff(v)), "total", v[-1] - v[0])
