#!/usr/bin/env python3
"""A few outer iterations of the device-resident optimizer on a small mesh
(run under compute-sanitizer by tools/sanitize.sh)."""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import paper_2301_07457_b200 as P  # noqa: E402

n, nc = 32, 2
g = P.GridLevel(n, n)
bc = P.wall_boundary_conditions(g, "uniform")
mat = P.MaterialModel(phase_moduli=[1.0, 0.5, 0.2, 1e-9], poisson_ratio=0.3, penalty=3.0)
cfg = P.OptimConfig(volume_fractions=[0.15, 0.15, 0.15, 0.55], filter_radius=1.5, max_outer=3, warm_start=True,
                    solver=P.SolverConfig(tol=1e-8, max_iter=2000, num_coarsenings=nc))
rep = P.optimize(P.MultigridOperators(g, nc, 0.3, bc), mat, cfg)
print("optimizer:", rep.outer_iterations, "outer iterations, compliance", rep.compliance_history)
