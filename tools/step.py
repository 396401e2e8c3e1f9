#!/usr/bin/env python3
"""Run N device-resident solves of a bench config (for ncu / sanitizer runs).

  python tools/step.py --config c4 --solves 1
"""
import argparse
import ctypes as C
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_2301_07457_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4", choices=sorted(bench.CONFIGS))
ap.add_argument("--solves", type=int, default=1)
ap.add_argument("--kernels", type=int, default=0, help="also time K.u / sweep this many reps")
ap.add_argument("--slabs", type=int, default=1, help="x-slabs driven from this process (LocalComm)")
ap.add_argument("--rep", type=int, default=-1, help="replicated level of the slab decomposition")
a = ap.parse_args()
nx, ny, nc, recipe, seed, desc = bench.CONFIGS[a.config]
g, bc, E, b = bench.make_inputs(nx, ny, recipe, seed)
ops = P.MultigridOperators(g, nc, 0.3, bc, slabs=a.slabs, replicated_level=a.rep)
ops.set_moduli(E, bench.OMEGA)
lib = P._lib.load()
ops._check(lib.tmg_gpu_upload_rhs(ops.h, P._lib.dptr(b)))
it, fr, cv, sec, hl = C.c_int(), C.c_double(), C.c_int(), C.c_double(), C.c_int()
hist = np.empty(5001)
for _ in range(a.solves):
    ops._check(lib.tmg_gpu_setup(ops.h, bench.OMEGA))
    ops._check(lib.tmg_gpu_solve_resident(ops.h, 0, 1e-8, 5000, 1, 2, 2, C.byref(it), C.byref(fr), C.byref(cv),
                                          C.byref(sec), P._lib.dptr(hist), hist.size, C.byref(hl)))
    print(f"{desc} [{a.slabs} slab(s)]: iterations={it.value} relres={fr.value:.3e} pcg={sec.value * 1e3:.2f} ms "
          f"({sec.value * 1e3 / max(it.value, 1):.3f} ms/iteration)", flush=True)
if a.kernels:
    for w, name in ((0, "K.u"), (1, "sweep"), (2, "update+2 sweeps")):
        ms, by = ops.time_kernel(w, a.kernels)
        print(f"{name}: {ms * 1e3:.1f} us  {by / ms / 1e6:.0f} GB/s", flush=True)
