"""Diagnostics of the GPU solve on the 4096^2 c4-recipe fixture (GPU box)."""
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2301_07457_b200 as P  # noqa: E402
from helpers import MAT  # noqa: E402

fx = np.load(ROOT / "tests" / "golden" / "c4_recipe_4096.npz")
n, nc = int(fx["nx"]), int(fx["num_coarsenings"])
g = P.GridLevel(n, n)
bc = P.wall_boundary_conditions(g, "uniform")
E = P.effective_moduli(P.density_iid(n, n, 1), MAT)
ops = P.MultigridOperators(g, nc, 0.3, bc)
ops.set_moduli(E, 0.6)
b = P.assemble_rhs(g, bc)
idx = fx["sample_index"]
rel = lambda a, c: float(np.linalg.norm(a - c) / np.linalg.norm(c))  # noqa: E731
for tol in (1e-8, 1e-10, 1e-12):
    rep = P.pcgmg_solve(ops, b, P.SolverConfig(tol=tol, max_iter=5000, num_coarsenings=nc))
    u = rep.solution
    C = P.compliance(ops)
    print(f"tol {tol:g}: it {rep.iterations} relres {rep.final_residual:.3e} | sample vs ref {rel(u[idx], fx['u_sample']):.3e}"
          f" vs ref-tight {rel(u[idx], fx['u_sample_tight']):.3e} | |u| vs ref {abs(np.linalg.norm(u) / fx['u_norm'] - 1):.3e}"
          f" | C {C!r} vs ref {C / fx['compliance'] - 1:.3e} vs ref-tight {C / fx['compliance_tight'] - 1:.3e}"
          f" | b.u {float(b @ u)!r}")
    if tol == 1e-8:
        h = np.asarray(rep.residual_history)
        print("history rel diff:", np.array2string(np.abs(h[:22] / fx["residual_history"][:22] - 1), precision=2))
