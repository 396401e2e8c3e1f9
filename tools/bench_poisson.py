"""The paper's Poisson pCGMG bench (run_poisson_bench pcgmg rows,
bench.cpp:30-111) on the B200 beside the unmodified
reference on the host.

  python tools/bench_poisson.py [--grids 16,32,64,128,256,1024,4096]

Per grid: constant source 1, every boundary node fixed, coarsest 2x2,
omega 0.6, 2+2 sweeps, V-cycle, tol 1e-6. A row's time is hierarchy +
operators + solve, as the reference measures it (bench.cpp:69-81): on the
GPU tmg_poisson_setup + tmg_poisson_solve (wall clock, median of 5 after a
warm-up); the reference runs grids up to 256^2 (1 host thread). Prints one
JSON line per grid."""
import argparse
import json
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grids", default="16,32,64,128,256,1024,4096")
    ap.add_argument("--ref-max", type=int, default=256)
    args = ap.parse_args()
    import paper_2301_07457_b200 as P
    from oracle import pyoracle as po  # reference leg only

    kind = "ref" if po.available("ref") else "orc"
    for g in (int(v) for v in args.grids.split(",")):
        nc = P.poisson_full_depth(g)
        grid = P.GridLevel(g, g)
        b = P.assemble_poisson_rhs(grid, 1.0)
        cfg = P.SolverConfig(tol=1e-6, max_iter=2000, omega=0.6, num_coarsenings=nc)
        ops = P.PoissonMultigrid(grid, nc)
        times, rep = [], None
        for k in range(6):
            t0 = time.perf_counter()
            ops._check(ops.lib.tmg_poisson_setup(ops.h, 0.6))
            rep = ops.solve(b, cfg)
            if k:
                times.append(time.perf_counter() - t0)
        t = float(np.median(times))
        out = {"metric": "Poisson pCGMG time to solution (hierarchy + operators + solve)", "grid": f"{g}x{g}",
               "levels": nc + 1, "value": t, "unit": "s", "higher_is_better": False,
               "iterations": rep.iterations, "final_residual": rep.final_residual,
               "solve_device_s": rep.seconds}
        if g <= args.ref_max:
            t0 = time.perf_counter()
            s = po.poisson_system(kind, g, g, 1.0).build_mg(nc, 0.6)
            r = s.solve(s.rhs(), tol=1e-6, max_iter=2000)
            tr = time.perf_counter() - t0
            out["cpu_baseline"] = {"value": tr, "unit": "s", "cores": 1,
                                   "kind": "reference" if kind == "ref" else "port",
                                   "iterations": r["iterations"],
                                   "sample": "same grid, assemble_poisson + build_multigrid_operators + pcgmg_solve"}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
