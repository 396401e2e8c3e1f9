"""The whole optimizer on the B200 (tmg_gpu_optimize; optimize() with
Method::pcgmg, mto.cpp:229-354) against the pinned
CPU checker, which is bit-exact to the reference's optimize().

Protocol: optimization is chaotic in the late iterations.
Small problems are gated closed loop over their first <= 10 outer iterations
(compliance history to 1e-9 relative, PCG counts within +-2, the density
change history and the final design to 1e-8); BASELINE c0 itself closed loop
over 25 outer iterations (design to the north-star 1e-6), and in open loop
at outer iterations 25 and 50 (the reference's design through the device
solve, compliance, sensitivities and filter)."""
import pathlib

import numpy as np
import pytest

import paper_2301_07457_b200 as P
from oracle import pyoracle as po

pytestmark = pytest.mark.gpu
GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"
PHASES = [1.0, 0.5, 0.2, 1e-9]


def wall(n):
    g = P.GridLevel(n, n)
    bc = P.wall_boundary_conditions(g, "uniform")
    fixed = list(bc.fixed_dofs)
    loads = list(bc.point_loads)
    return g, bc, fixed, loads


def run_both(n, nc, fractions=(0.15, 0.15, 0.15, 0.55), **kw):
    g, bc, fixed, loads = wall(n)
    mat = P.MaterialModel(phase_moduli=PHASES, poisson_ratio=0.3, penalty=3.0)
    solver = P.SolverConfig(tol=1e-8, max_iter=2000, num_coarsenings=nc)
    cfg = P.OptimConfig(volume_fractions=list(fractions), solver=solver, **kw)
    ops = P.MultigridOperators(g, nc, 0.3, bc)
    got = P.optimize(ops, mat, cfg)
    want = po.optimize("orc", n, n, fixed, loads, PHASES, 3.0, 0.3, list(fractions), num_coarsenings=nc,
                       filter_radius=cfg.filter_radius, filter_tol=cfg.filter_tol, tol=cfg.tol,
                       inner_sweeps=cfg.inner_sweeps, move_limit=cfg.move_limit, oc_damping=cfg.oc_damping,
                       warm_start=cfg.warm_start, max_outer=cfg.max_outer, density_floor=cfg.density_floor)
    return got, want


def check(got, want):
    assert got.outer_iterations == want["outer_iterations"]
    assert got.converged == want["converged"]
    np.testing.assert_allclose(got.compliance_history, want["compliance_history"], rtol=1e-9)
    assert all(abs(a - b) <= 2 for a, b in zip(got.solver_iteration_history, want["solver_iteration_history"]))
    np.testing.assert_allclose(got.change_history, want["change_history"], rtol=1e-6, atol=1e-9)
    assert np.max(np.abs(got.density - want["density"])) <= 1e-8
    # the design stays a partition of unity with the volume targets met
    assert np.max(np.abs(got.density.sum(1) - 1.0)) <= 1e-12
    assert len(got.seconds_history) == got.outer_iterations and got.seconds > 0


@pytest.mark.parametrize("n,nc", [(32, 2), (64, 3)])
def test_config0_style_run(n, nc):
    got, want = run_both(n, nc, filter_radius=1.5, tol=1e-12, max_outer=10)
    check(got, want)


def test_warm_start_inner_sweeps_wide_filter():
    got, want = run_both(48, 2, filter_radius=3.0, tol=1e-12, max_outer=8, warm_start=True, inner_sweeps=2)
    check(got, want)


def test_converges_and_stops_like_the_reference():
    got, want = run_both(24, 1, filter_radius=1.5, tol=0.25, max_outer=30, move_limit=0.1)
    check(got, want)
    assert got.converged and got.outer_iterations < 30


def test_config_errors_mirror_reference():
    g, bc, _, _ = wall(16)
    ops = P.MultigridOperators(g, 1, 0.3, bc)
    mat = P.MaterialModel(phase_moduli=PHASES, poisson_ratio=0.3, penalty=3.0)
    for kw in (dict(volume_fractions=[0.5, 0.6]), dict(move_limit=0.0), dict(oc_damping=1.5), dict(max_outer=0),
               dict(density_floor=0.5), dict(inner_sweeps=0), dict(filter_tol=0.0)):
        base = dict(volume_fractions=[0.15, 0.15, 0.15, 0.55])
        base.update(kw)
        with pytest.raises(P.ConfigError):
            P.optimize(ops, mat if len(base["volume_fractions"]) == 4 else
                       P.MaterialModel(phase_moduli=[1.0, 1e-9], poisson_ratio=0.3, penalty=3.0),
                       P.OptimConfig(solver=P.SolverConfig(num_coarsenings=1), **base))


C0 = dict(n=64, nc=3, filter_radius=1.5)  # BASELINE configs[0]: 64^2, 4 levels, r_f 1.5


def test_config0_closed_loop_first_25():
    """BASELINE c0 run closed loop for 25 outer iterations, the horizon over
    which SURVEY.md 8(c) measured a 1e-15 perturbation of the load to stay
    within 6e-9 in the design: the north-star design bar (1e-6 per element)
    holds there, with compliance to 1e-8 and PCG counts within +-2."""
    got, want = run_both(C0["n"], C0["nc"], filter_radius=C0["filter_radius"], tol=1e-12, max_outer=25)
    assert got.outer_iterations == want["outer_iterations"] == 25
    np.testing.assert_allclose(got.compliance_history, want["compliance_history"], rtol=1e-8)
    assert all(abs(a - b) <= 2 for a, b in zip(got.solver_iteration_history, want["solver_iteration_history"]))
    d = float(np.max(np.abs(got.density - want["density"])))
    print(f"c0 closed loop, 25 outer iterations: max |design diff| = {d:.2e}")
    assert d <= 1e-6


@pytest.mark.parametrize("k", [25, 50])
def test_config0_open_loop(k):
    """Past ~25 outer iterations the c0 run is chaotic, so
    the late iterations are compared in open loop: the reference's own
    design after k outer iterations (the checker is bit-exact to the
    reference's optimize) goes through the device solve, compliance,
    sensitivities and filter, against the checker's solve of the same design.
    Late designs carry void (E = 1e-9) next to solid phases, the regime where
    SURVEY.md 8(c) says a reordered CG can move u by up to ~1e-7; the bars are
    the residual under the checker's operator, u and compliance to the
    checker's own tol-1e-8 solution error (measured against a tol-1e-13 solve)
    plus margin, and PCG counts within +-2 where the solve is well
    conditioned. At k = 50 the CG takes ~750 iterations and the checker's own
    tol-1e-8 solution is ~4e-6 from the exact one (measured on the B200:
    device 748, checker 753 iterations, u 5e-7 apart, sensitivities 1e-8,
    filtered 3e-8). There any change of rounding moves the count by several
    iterations (a different coarsest inverse gave 745 with the same bars
    met), so, as SURVEY.md 8(c) recommends for ill-conditioned solves, the
    count is reported and only sanity-checked (5 %)."""
    n, nc, rf = C0["n"], C0["nc"], C0["filter_radius"]
    g, bc, fixed, loads = wall(n)
    mat = P.MaterialModel(phase_moduli=PHASES, poisson_ratio=0.3, penalty=3.0)
    want = po.optimize("orc", n, n, fixed, loads, PHASES, 3.0, 0.3, [0.15, 0.15, 0.15, 0.55],
                       num_coarsenings=nc, filter_radius=rf, tol=1e-12, max_outer=k)
    alpha = want["density"]
    E = P.effective_moduli(alpha, mat)
    ops = P.MultigridOperators(g, nc, 0.3, bc)
    ops.set_moduli(E, 0.6)
    b = P.assemble_rhs(g, bc)
    rep = P.pcgmg_solve(ops, b, P.SolverConfig(tol=1e-8, max_iter=5000))
    sysc = po.System("orc", n, n, E, 0.3, bc.fixed_dofs, bc.point_loads).build_mg(nc)
    ref = sysc.solve(b, tol=1e-8, max_iter=5000)
    exact = sysc.solve(b, tol=1e-13, max_iter=20000)["solution"]
    u, ur = rep.solution, ref["solution"]
    ref_err = np.linalg.norm(ur - exact) / np.linalg.norm(exact)
    du = np.linalg.norm(u - ur) / np.linalg.norm(ur)
    res = np.linalg.norm(b - sysc.matvec(nc, u)) / np.linalg.norm(b)  # under the checker's fine K
    c_gpu, c_ref = P.compliance(ops), sysc.compliance(ur)
    s_gpu = P.sensitivities(ops, alpha, mat)
    s_ref = po.sensitivities("orc", n, n, alpha, PHASES, 3.0, 0.3, ur)
    ds = max(np.max(np.abs(s_gpu[p] - s_ref[p])) / np.max(np.abs(s_ref[p])) for p in range(3))
    f_gpu = [P.filter_sensitivities(ops, s_gpu[p], alpha, p, rf) for p in range(3)]
    f_ref = [po.filter_sensitivities("orc", n, n, alpha, p, rf, s_ref[p]) for p in range(3)]
    df = max(np.max(np.abs(a - c)) / np.max(np.abs(c)) for a, c in zip(f_gpu, f_ref))
    print(f"c0 open loop k={k}: pcg gpu={rep.iterations} ref={ref['iterations']} relres={res:.2e} "
          f"du={du:.2e} (ref's own tol-1e-8 error {ref_err:.2e}) dC={abs(c_gpu - c_ref) / c_ref:.2e} "
          f"dsens={ds:.2e} dfilt={df:.2e}")
    assert rep.converged and abs(rep.iterations - ref["iterations"]) <= (2 if k <= 25 else 0.05 * ref["iterations"])
    assert res <= 1.01e-8
    assert du <= 1e-8 + 2 * ref_err
    assert abs(c_gpu - c_ref) <= 1e-9 * c_ref + 2 * ref_err * c_ref
    assert ds <= 1e-8 + 4 * ref_err and df <= 1e-8 + 4 * ref_err

