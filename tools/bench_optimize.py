"""Measure the device-resident optimizer (tmg_gpu_optimize, SURVEY.md 8(f)
item 2) on the BASELINE optimization configs, beside the unmodified
reference's optimize() on the host.

  python tools/bench_optimize.py [--configs c0,c3] [--ref-prefix 2]

c0: 64^2, 4 levels, r_f 1.5, 50 outer iterations (outer tol tiny so all run).
c3: 1024^2, 8 levels, r_f 3, warm start, 100 outer iterations.
Both: E = {1, 0.5, 0.2, 1e-9}, nu 0.3, p 3, V = {0.15, 0.15, 0.15, 0.55},
damped Jacobi 0.6 with 2+2 sweeps, solver tol 1e-8, unit total load spread
over the top edge. The reference runs c0 in full and the
first --ref-prefix outer iterations of c3 (about 25 s each on one core).
Prints one JSON line per config: outer iterations/s on the GPU (whole loop,
wall clock incl. the final density download) and for the reference."""
import argparse
import json
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

PHASES = [1.0, 0.5, 0.2, 1e-9]
FRACTIONS = [0.15, 0.15, 0.15, 0.55]
CONFIGS = {"c0": dict(n=64, nc=3, radius=1.5, outer=50, warm=False),
           "c3": dict(n=1024, nc=7, radius=3.0, outer=100, warm=True)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c0,c3")
    ap.add_argument("--ref-prefix", type=int, default=2)
    args = ap.parse_args()
    import paper_2301_07457_b200 as P
    from oracle import pyoracle as po  # reference leg only

    kind = "ref" if po.available("ref") else "orc"
    for name in args.configs.split(","):
        c = CONFIGS[name]
        n = c["n"]
        g = P.GridLevel(n, n)
        bc = P.wall_boundary_conditions(g, "uniform")
        ops = P.MultigridOperators(g, c["nc"], 0.3, bc)
        mat = P.MaterialModel(phase_moduli=PHASES, poisson_ratio=0.3, penalty=3.0)
        cfg = P.OptimConfig(volume_fractions=FRACTIONS, filter_radius=c["radius"], tol=1e-12,
                            max_outer=c["outer"], warm_start=c["warm"],
                            solver=P.SolverConfig(tol=1e-8, max_iter=5000, num_coarsenings=c["nc"]))
        P.optimize(ops, mat, P.OptimConfig(**{**cfg.__dict__, "max_outer": 2}))  # warm-up
        t0 = time.perf_counter()
        rep = P.optimize(ops, mat, cfg)
        wall = time.perf_counter() - t0
        ref_outer = c["outer"] if name == "c0" else args.ref_prefix
        t0 = time.perf_counter()
        r = po.optimize(kind, n, n, list(bc.fixed_dofs), list(bc.point_loads), PHASES, 3.0, 0.3, FRACTIONS,
                        filter_radius=c["radius"], tol=1e-12, max_outer=ref_outer, warm_start=c["warm"],
                        num_coarsenings=c["nc"], solver_max_iter=5000)
        ref_wall = time.perf_counter() - t0
        k = min(ref_outer, rep.outer_iterations)
        out = {"metric": "optimizer outer iterations/s (optimize(), Method::pcgmg)", "config": name,
               "mesh": f"{n}x{n}", "levels": c["nc"] + 1, "filter_radius": c["radius"], "warm_start": c["warm"],
               "value": rep.outer_iterations / wall, "unit": "outer iterations/s",
               "outer_iterations": rep.outer_iterations, "seconds": wall,
               "total_solver_iterations": rep.total_solver_iterations,
               "final_compliance": rep.compliance_history[-1],
               "matches_reference_prefix": {
                   "outer_iterations": k,
                   "max_rel_compliance_diff": max(abs(a - b) / abs(b) for a, b in
                                                  zip(rep.compliance_history[:k], r["compliance_history"][:k])),
                   "solver_iterations_gpu": rep.solver_iteration_history[:k],
                   "solver_iterations_ref": [int(v) for v in r["solver_iteration_history"][:k]]},
               "cpu_baseline": {"value": ref_outer / ref_wall, "unit": "outer iterations/s", "cores": 1,
                                "kind": "reference" if kind == "ref" else "port",
                                "sample": f"first {ref_outer} outer iterations, {ref_wall:.1f} s"},
               "data": "synthetic (BASELINE config recipe: uniform start, wall supports, top load)"}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
