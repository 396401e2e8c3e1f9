#!/usr/bin/env python3
"""Generate tests/golden/c4_recipe_4096.npz from the UNMODIFIED reference.

The reference cannot assemble BASELINE c4 itself (8192^2): its CSR row
offsets are int (proj/include/topmg/sparse.hpp:53, proj/src/sparse.cpp:44-45)
and c4 has ~2.42e9 nonzeros > INT_MAX. The largest c4-recipe mesh it can run
on a 62 GB host is 4096^2 (0.60e9 nonzeros, ~41 GB peak during assembly).
This script runs oracle/_ref (the reference compiled from its own sources by
oracle/Makefile) on that mesh with the c4 recipe -- iid U(0,1) densities from
seed 1 with the oracles.hpp:21-23 generator, E = {1, 0.5, 0.2, 1e-9}, p = 3,
nu = 0.3, bottom edge clamped, unit total load over the top edge, 10 levels
(coarsest 8x8), damped Jacobi omega = 0.6 2+2, V-cycle, tol 1e-8 -- through
assemble_from_moduli + build_multigrid_operators + pcgmg_solve, as
acceptance.cpp:156-190 drives it, and stores what a full-size GPU test needs:
the iteration count, the residual history, the compliance u^T K u, |u|_2, the
sum of u, u on a fixed sample of dofs (every 1021st dof plus every top-edge
v-dof) and u projected on four seeded random +-1 vectors (numpy PCG64, seeds
11..14, regenerated at test time); then it continues the reference's solve
from u to tol 1e-12 and stores that answer's compliance, sample and norm and
|u - u_tight|, the reference's own distance to its converged solution. Run once in this container (takes ~10 min
and ~41 GB of RAM); the fixture is committed, the test never needs
/root/reference.
"""
from __future__ import annotations

import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import pyoracle as po  # noqa: E402

N, NC, SEED = 4096, 9, 1
PM, PEN, NU = [1.0, 0.5, 0.2, 1e-9], 3.0, 0.3
STRIDE = 1021
PROJ_SEEDS = (11, 12, 13, 14)


def sample_index(nx, ny):
    n = 2 * (nx + 1) * (ny + 1)
    top_v = 2 * (np.arange(nx + 1) * (ny + 1) + ny) + 1
    return np.union1d(np.arange(0, n, STRIDE), top_v).astype(np.int64)


def projections(u):
    out = []
    for s in PROJ_SEEDS:
        r = np.random.default_rng(s).integers(0, 2, u.size, dtype=np.int8).astype(np.float64) * 2.0 - 1.0
        out.append(float(r @ u))
    return np.array(out)


def main():
    if not po.available("ref"):
        raise SystemExit("oracle/_ref not built (make -C oracle ref)")
    t0 = time.time()
    alpha = po.density_iid("ref", N, N, SEED)
    E = po.effective_moduli("ref", N, N, alpha, PM, PEN)
    del alpha
    fixed, loads = po.wall_uniform_bc(N, N)
    s = po.System("ref", N, N, E, NU, fixed, loads)
    print(f"assembled in {time.time() - t0:.1f} s", flush=True)
    s.build_mg(NC, 0.6)
    print(f"hierarchy built at {time.time() - t0:.1f} s", flush=True)
    b = s.rhs()
    r = s.solve(b, tol=1e-8, max_iter=5000, gamma=1, pre=2, post=2)
    u = r["solution"]
    comp = s._f("system_compliance")(s.h, po._d(u))
    t = s.times()
    # the reference's own distance to its converged answer (SURVEY.md 8(c)
    # protocol, step 4): continue from u to tol 1e-12
    rt = s.solve(b, tol=1e-12, max_iter=5000, gamma=1, pre=2, post=2, x0=u)
    ut = rt["solution"]
    comp_t = s._f("system_compliance")(s.h, po._d(ut))
    idx = sample_index(N, N)
    np.savez_compressed(
        pathlib.Path(__file__).resolve().parent / "c4_recipe_4096.npz",
        nx=N, ny=N, num_coarsenings=NC, seed=SEED, iterations=r["iterations"], converged=r["converged"],
        residual_history=r["residual_history"], compliance=comp, u_norm=np.linalg.norm(u), u_sum=u.sum(),
        sample_index=idx, u_sample=u[idx], projections=projections(u), proj_seeds=np.array(PROJ_SEEDS),
        ref_seconds=np.array([t["assemble"], t["setup"], t["pcg"]]),
        tight_iterations=rt["iterations"], compliance_tight=comp_t, u_sample_tight=ut[idx],
        u_norm_tight=np.linalg.norm(ut), u_dist_tight=np.linalg.norm(u - ut))
    print(f"iterations {r['iterations']} converged {r['converged']} compliance {comp!r} "
          f"assemble {t['assemble']:.1f} s setup {t['setup']:.1f} s pcg {t['pcg']:.1f} s "
          f"total {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main()
