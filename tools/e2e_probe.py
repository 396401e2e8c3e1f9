#!/usr/bin/env python3
"""Where the pipelined e2e step's time goes (c4): per-step PCG seconds of
resident solves, of pipelined solves and of blocking solves, and the copy
rates of the staging copies alone.   python tools/e2e_probe.py [--steps 8]"""
import argparse
import ctypes as C
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2301_07457_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=8)
ap.add_argument("--config", default="c4")
a = ap.parse_args()
nx, ny, nc, recipe, seed, desc = bench.CONFIGS[a.config]
g, bc, E, b = bench.make_inputs(nx, ny, recipe, seed)
ops = P.MultigridOperators(g, nc, 0.3, bc)
lib = ops.lib
D = P._lib.dptr
pE, pb, px, px2 = P.PinnedArray(E.size), P.PinnedArray(b.size), P.PinnedArray(b.size), P.PinnedArray(b.size)
pE.a[:] = E
pb.a[:] = b
ops.set_moduli(pE.a, 0.6)
ops._check(lib.tmg_gpu_upload_rhs(ops.h, D(pb.a)))
it, fr, cv, sec, hl = C.c_int(), C.c_double(), C.c_int(), C.c_double(), C.c_int()
hist = np.empty(5001)
ms = C.c_double()


def timed(fn, n):
    ops._check(lib.tmg_gpu_event_record(ops.h, 2))
    t0 = time.perf_counter()
    out = [fn(k) for k in range(n)]
    ops._check(lib.tmg_gpu_event_record(ops.h, 3))
    ops._check(lib.tmg_gpu_event_elapsed(ops.h, 2, 3, C.byref(ms)))
    return ms.value / n, (time.perf_counter() - t0) * 1e3 / n, out


def resident(k):
    ops._check(lib.tmg_gpu_setup(ops.h, 0.6))
    ops._check(lib.tmg_gpu_solve_resident(ops.h, 0, 1e-8, 5000, 1, 2, 2, C.byref(it), C.byref(fr), C.byref(cv),
                                          C.byref(sec), D(hist), hist.size, C.byref(hl)))
    return sec.value * 1e3


def blocking(k):
    ops._check(lib.tmg_gpu_set_moduli(ops.h, D(pE.a), E.size, 0.6))
    ops._check(lib.tmg_gpu_solve(ops.h, D(pb.a), None, 1e-8, 5000, 1, 2, 2, D(px.a), C.byref(it), C.byref(fr),
                                 C.byref(cv), C.byref(sec), D(hist), hist.size, C.byref(hl)))
    return sec.value * 1e3


n = a.steps
outs = (px, px2)


def pipelined(k):
    if k == 0:
        ops._check(lib.tmg_gpu_stage_inputs(ops.h, 0, D(pE.a), E.size, D(pb.a)))
    if k + 1 < n:
        ops._check(lib.tmg_gpu_stage_inputs(ops.h, (k + 1) & 1, D(pE.a), E.size, D(pb.a)))
    ops._check(lib.tmg_gpu_solve_staged(ops.h, k & 1, 0.6, 1e-8, 5000, 1, 2, 2, D(outs[k & 1].a), C.byref(it),
                                        C.byref(fr), C.byref(cv), C.byref(sec), D(hist), hist.size, C.byref(hl)))
    if k == n - 1:
        ops._check(lib.tmg_gpu_sync_outputs(ops.h))
    return sec.value * 1e3


for name, fn in (("resident", resident), ("pipelined", pipelined), ("blocking", blocking), ("resident", resident),
                 ("pipelined", pipelined)):
    dev, wall, pcg = timed(fn, n)
    print(f"{name:9s} device {dev:7.2f} ms/step  wall {wall:7.2f}  pcg per step {np.round(pcg, 1).tolist()}", flush=True)
