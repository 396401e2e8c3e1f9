#!/usr/bin/env python3
"""Print a hash of the solution, residual history and one V-cycle of a bench
config (to check that two builds are bitwise identical, via TMG_LIB_PATH):

  TMG_LIB_PATH=$PWD/libA.so python tools/hash_solve.py --config c1
"""
import argparse
import hashlib
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_2301_07457_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1", choices=sorted(bench.CONFIGS))
ap.add_argument("--slabs", type=int, default=1)
a = ap.parse_args()
nx, ny, nc, recipe, seed, desc = bench.CONFIGS[a.config]
g, bc, E, b = bench.make_inputs(nx, ny, recipe, seed)
ops = P.MultigridOperators(g, nc, 0.3, bc, slabs=a.slabs)
ops.set_moduli(E, bench.OMEGA)
rep = P.pcgmg_solve(ops, b, P.SolverConfig(tol=1e-8, max_iter=5000))
f = np.random.default_rng(3).standard_normal(b.size)
v = P.mg_cycle(ops, np.zeros_like(f), f)
h = hashlib.sha256()
for arr in (rep.solution, np.asarray(rep.residual_history), v):
    h.update(np.ascontiguousarray(arr).tobytes())
print(f"{a.config} slabs={a.slabs} iterations={rep.iterations} sha256={h.hexdigest()[:16]}")
