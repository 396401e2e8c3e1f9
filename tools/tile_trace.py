#!/usr/bin/env python3
"""Per-phase times of the tile kernels in one V-cycle (a TMG_TILE_TRACE build
loaded through TMG_LIB_PATH):  python tools/tile_trace.py --config c1"""
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
ap.add_argument("--config", default="c1")
a = ap.parse_args()
nx, ny, nc, recipe, seed, desc = bench.CONFIGS[a.config]
g, bc, E, b = bench.make_inputs(nx, ny, recipe, seed)
ops = P.MultigridOperators(g, nc, 0.3, bc)
ops.set_moduli(E, bench.OMEGA)
f = np.random.default_rng(0).standard_normal(b.size)
lib = P._lib.load()
t = (C.c_ulonglong * 512)()
for _ in range(3):
    assert lib.tmg_debug_tile_trace(t, 1) == 0
    P.mg_cycle(ops, np.zeros_like(f), f)
assert lib.tmg_debug_tile_trace(t, 0) == 0
v = np.array(t[:], dtype=np.int64).reshape(64, 8)
print(desc)
prev_end = None
for k in range(64):
    r = v[k]
    if r[0] == 0:
        break
    up = r[4] == 0
    ph = [r[1] - r[0], r[2] - r[1], r[3] - r[2]] + ([r[5] - r[3]] if up else [r[4] - r[3], r[5] - r[4]])
    gap = "" if prev_end is None else f" gap {r[0] - prev_end:5d}"
    print(f"launch {k:2d} {'UP  ' if up else 'DOWN'} total {r[5] - r[0]:5d} ns: " + " ".join(f"{x:5d}" for x in ph) + gap)
    prev_end = r[5]
