"""GPU pCGMG vs the CPU checker on identical seeded inputs.

Bars (north star): relative L2 error of u <= 1e-8, compliance within 1e-9
relative, PCG iteration count within +-2. Kernel-level pins are tighter:
operator / Galerkin entries <= 1e-13 relative to the largest entry, one
V-cycle <= 1e-12 relative. The checker is oracle/liboracle.so, itself pinned
bit-for-bit to the reference (tests/test_oracle_pin.py).
"""
import numpy as np
import pytest

import paper_2301_07457_b200 as P
from helpers import MAT, moduli, pair, rel
from oracle import pyoracle as po

pytestmark = pytest.mark.gpu

SIZES = [(8, 8, 2), (16, 16, 3), (32, 16, 2), (24, 40, 3), (64, 64, 3), (128, 128, 4)]


@pytest.mark.parametrize("nx,ny,nc", SIZES)
def test_fine_apply_matches_assembled_matvec(nx, ny, nc):
    ops, sysc, b, _, _ = pair(nx, ny, nc)
    x = np.random.default_rng(3).standard_normal(sysc.n)
    y = ops.apply(nc, x)
    yr = sysc.matvec(nc, x)
    assert np.max(np.abs(y - yr)) <= 1e-13 * np.max(np.abs(yr))


@pytest.mark.parametrize("nx,ny,nc", SIZES)
def test_galerkin_hierarchy_matches_reference_entries(nx, ny, nc):
    ops, sysc, b, _, _ = pair(nx, ny, nc)
    for lvl in range(nc + 1):
        off, col, val = sysc.csr(lvl)
        got = ops.level_values(lvl, off, col)
        scale = np.max(np.abs(val))
        assert np.max(np.abs(got - val)) <= 1e-13 * scale, f"level {lvl}"


@pytest.mark.parametrize("nx,ny,nc", SIZES)
def test_coarse_level_apply(nx, ny, nc):
    ops, sysc, b, _, _ = pair(nx, ny, nc)
    rng = np.random.default_rng(4)
    for lvl in range(nc):
        x = rng.standard_normal(sysc.csr(lvl)[0].size - 1)
        y = ops.apply(lvl, x)
        yr = sysc.matvec(lvl, x)
        assert np.max(np.abs(y - yr)) <= 1e-13 * np.max(np.abs(yr)), f"level {lvl}"


@pytest.mark.parametrize("nx,ny,nc", [(16, 16, 3), (64, 32, 3)])
def test_jacobi_sweeps_match_csr_formula(nx, ny, nc):
    ops, sysc, b, _, _ = pair(nx, ny, nc)
    rng = np.random.default_rng(5)
    for lvl in range(1, nc + 1):
        off, col, val = sysc.csr(lvl)
        n = off.size - 1
        diag = np.array([val[off[i]:off[i + 1]][col[off[i]:off[i + 1]] == i][0] for i in range(n)])
        f = rng.standard_normal(n)
        u = rng.standard_normal(n)
        want = u.copy()
        for _ in range(2):
            want = want + 0.6 * (f - sysc.matvec(lvl, want)) / diag
        got = ops.smooth(lvl, f, u, 2)
        assert rel(got, want) <= 1e-13


@pytest.mark.parametrize("nx,ny,nc", SIZES)
@pytest.mark.parametrize("gamma", [1, 2])
def test_one_cycle_matches_mg_cycle(nx, ny, nc, gamma):
    ops, sysc, b, _, _ = pair(nx, ny, nc)
    rng = np.random.default_rng(6)
    f = rng.standard_normal(sysc.n)
    for u0 in (np.zeros(sysc.n), rng.standard_normal(sysc.n)):
        got = P.mg_cycle(ops, u0, f, gamma, 2, 2)
        want = sysc.vcycle(f, u0, gamma, 2, 2)
        # the device Ke is the symmetric 8-value form of the quadrature Ke
        # (<= 1 ulp per entry, tmg_device.cuh); one cycle amplifies that
        # through the coarsest solve to ~1e-12 at 128^2
        assert rel(got, want) <= 1e-11


def test_transfer_properties():
    """test_grid.cpp:106-155 restated for the device transfer kernels."""
    ops, sysc, b, _, _ = pair(16, 16, 2)
    fine = ops.level(2)
    coarse = ops.level(1)
    # prolongation reproduces linear fields exactly (test_grid.cpp:53-104)
    xs = np.array([[x, y] for x in range(coarse.nx + 1) for y in range(coarse.ny + 1)], float)
    uc = np.stack([2 * xs[:, 0] + 3 * xs[:, 1], -xs[:, 0] + 0.5 * xs[:, 1]], 1).ravel()
    uf = ops.prolongate(2, uc)
    xf = np.array([[x, y] for x in range(fine.nx + 1) for y in range(fine.ny + 1)], float) / 2
    want = np.stack([2 * xf[:, 0] + 3 * xf[:, 1], -xf[:, 0] + 0.5 * xf[:, 1]], 1).ravel()
    assert np.max(np.abs(uf - want)) < 1e-13
    # variational pairing <P u, v> = <u, 4 R v> (test_grid.cpp:140-155)
    rng = np.random.default_rng(7)
    u = rng.standard_normal(coarse.dof_count())
    v = rng.standard_normal(fine.dof_count())
    lhs = np.dot(ops.prolongate(2, u), v)
    rhs = np.dot(u, 4 * ops.restrict(2, v))
    assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))
    # interior coarse node of restricted ones = 1 (test_grid.cpp:106-120)
    rc = ops.restrict(2, np.ones(fine.dof_count()))
    k = coarse.node_index(3, 4)
    assert abs(rc[2 * k] - 1.0) < 1e-15 and abs(rc[2 * k + 1] - 1.0) < 1e-15


CASES = [
    (16, 16, 2, "iid", 0, "uniform"),
    (32, 32, 3, "iid", 1, "point"),
    (64, 64, 3, "uniform", 0, "uniform"),  # config 0 initial design
    (64, 64, 3, "checker", 2, "uniform"),
    (128, 64, 4, "iid", 3, "uniform"),
    (256, 256, 5, "iid", 0, "uniform"),
    (512, 512, 6, "iid", 0, "uniform"),  # BASELINE c1 exactly (7 levels, seed 0)
    (1024, 1024, 7, "uniform", 0, "uniform"),  # BASELINE c3's first solve (initial design)
]


@pytest.mark.parametrize("nx,ny,nc,recipe,seed,load", CASES)
def test_pcgmg_solve_parity(nx, ny, nc, recipe, seed, load):
    ops, sysc, b, _, _ = pair(nx, ny, nc, recipe, seed, load)
    cfg = P.SolverConfig(tol=1e-8, max_iter=2000, num_coarsenings=nc)
    rep = P.pcgmg_solve(ops, b, cfg)
    ref = sysc.solve(b, tol=1e-8, max_iter=2000)
    assert rep.converged and ref["converged"]
    assert abs(rep.iterations - ref["iterations"]) <= 2
    assert rel(rep.solution, ref["solution"]) <= 1e-8
    c_gpu = P.compliance(ops)
    c_ref = sysc.compliance(ref["solution"])
    assert abs(c_gpu - c_ref) <= 1e-9 * abs(c_ref)
    assert len(rep.residual_history) == rep.iterations + 1
    assert rep.residual_history[-1] == rep.final_residual <= 1e-8
    # relative residual of the GPU solution under the reference's assembled K
    r = b - sysc.matvec(nc, rep.solution)
    assert np.linalg.norm(r) / np.linalg.norm(b) <= 1e-8 * 1.0001


def test_reference_itself_when_available():
    if not po.available("ref"):
        pytest.skip("oracle/_ref not built")
    ops, sysc, b, _, _ = pair(64, 64, 3, kind="ref")
    rep = P.pcgmg_solve(ops, b, P.SolverConfig(tol=1e-8, max_iter=500))
    ref = sysc.solve(b, tol=1e-8, max_iter=500)
    assert abs(rep.iterations - ref["iterations"]) <= 2
    assert rel(rep.solution, ref["solution"]) <= 1e-8


@pytest.mark.parametrize("n,nc,recipe", [(16, 1, "uniform"), (32, 2, "uniform"), (64, 3, "iid"), (64, 3, "checker")])
def test_tight_tolerance_matches_direct_solution(n, nc, recipe):
    """acceptance.cpp:156-190: pCGMG at tol 1e-10 within 1e-8 of the direct
    solution on elasticity 16/32/64. The reference factors its assembled K
    with Cholesky; here the checker's assembled fine CSR (bit-identical to the
    reference's K, identity rows included) is factored by a sparse direct LU."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla

    ops, sysc, b, _, _ = pair(n, n, nc, recipe=recipe)
    rep = P.pcgmg_solve(ops, b, P.SolverConfig(tol=1e-10, max_iter=2000))
    assert rep.converged
    off, col, val = sysc.csr(nc)
    K = sp.csr_matrix((val, col, off), shape=(sysc.n, sysc.n)).tocsc()
    direct = spla.spsolve(K, b)
    assert rel(rep.solution, direct) <= 1e-8


def test_new_omega_on_a_live_handle_matches_a_fresh_handle():
    """omega is fixed when the operators are built (solvers.cpp:471): a setup
    with another omega on the same handle must solve exactly like a fresh
    handle built with it (the captured graphs carry omega by value). With
    omega = 0.9 the damped-Jacobi V-cycle is no longer positive definite on
    this problem: the reference raises PreconditionerError at iteration 3, and
    so must the live handle (stale omega-0.6 graphs would converge)."""
    nx = ny = 64
    nc = 3
    _, E = moduli(nx, ny)
    g = P.GridLevel(nx, ny)
    bc = P.wall_boundary_conditions(g, "uniform")
    b = P.assemble_rhs(g, bc)
    cfg = P.SolverConfig(tol=1e-8, max_iter=500)
    checker = lambda om: po.System("orc", nx, ny, E, 0.3, bc.fixed_dofs, bc.point_loads).build_mg(nc, om)  # noqa
    live = P.MultigridOperators(g, nc, 0.3, bc)
    live.set_moduli(E, 0.6)
    first = P.pcgmg_solve(live, b, cfg)
    live.set_moduli(E, 0.9)
    with pytest.raises(po.OracleError) as want_err:
        checker(0.9).solve(b, tol=1e-8)
    with pytest.raises(P.PreconditionerError) as got_err:
        P.pcgmg_solve(live, b, cfg)
    assert str(got_err.value) == want_err.value.msg
    live.set_moduli(E, 0.7)
    again = P.pcgmg_solve(live, b, cfg)
    fresh = P.MultigridOperators(g, nc, 0.3, bc)
    fresh.set_moduli(E, 0.7)
    want = P.pcgmg_solve(fresh, b, cfg)
    assert again.iterations == want.iterations
    assert np.array_equal(again.solution, want.solution)
    assert again.residual_history == want.residual_history
    ref = checker(0.7).solve(b, tol=1e-8)
    assert abs(again.iterations - ref["iterations"]) <= 2
    assert rel(again.solution, ref["solution"]) <= 1e-8
    assert first.residual_history != again.residual_history


def test_warm_start_and_zero_rhs_and_max_iter():
    ops, sysc, b, _, _ = pair(32, 32, 3)
    cfg = P.SolverConfig(tol=1e-8, max_iter=500)
    first = P.pcgmg_solve(ops, b, cfg)
    ref = sysc.solve(b, tol=1e-8, max_iter=500, x0=first.solution * 0.99)
    warm = P.pcgmg_solve(ops, b, cfg, x0=first.solution * 0.99)
    assert abs(warm.iterations - ref["iterations"]) <= 2
    assert rel(warm.solution, ref["solution"]) <= 1e-8
    # already converged warm start: 0 iterations (solvers.cpp:351-357)
    done = P.pcgmg_solve(ops, b, cfg, x0=first.solution)
    assert done.converged and done.iterations == 0 and len(done.residual_history) == 1
    # zero rhs: zero solution, converged, history {0} (solvers.cpp:338-344)
    z = P.pcgmg_solve(ops, np.zeros_like(b), cfg, x0=first.solution)
    assert z.converged and z.iterations == 0 and z.residual_history == [0.0]
    assert not np.any(z.solution)
    # max_iter exhausted: not converged, not an error
    short = P.pcgmg_solve(ops, b, P.SolverConfig(tol=1e-14, max_iter=3))
    rs = sysc.solve(b, tol=1e-14, max_iter=3)
    assert not short.converged and short.iterations == 3
    assert rel(short.solution, rs["solution"]) <= 1e-10


@pytest.mark.parametrize("sweeps", [1, 2, 3])
@pytest.mark.parametrize("max_iter", [1, 2, 5, 500])
def test_sweep_counts_and_iteration_caps(sweeps, max_iter):
    """pre = post = 1 takes the unfused x/r update; 2 and 3 finish each PCG
    iteration inside the next one's first smoothing pass (and after the loop
    when max_iter stops it): iterates, histories and caps must not tell."""
    ops, sysc, b, _, _ = pair(64, 32, 3, seed=4)
    rep = P.pcgmg_solve(ops, b, P.SolverConfig(tol=1e-8, max_iter=max_iter, pre_sweeps=sweeps,
                                               post_sweeps=sweeps))
    ref = sysc.solve(b, tol=1e-8, max_iter=max_iter, pre=sweeps, post=sweeps)
    assert rep.converged == ref["converged"]
    if not ref["converged"]:
        assert rep.iterations == ref["iterations"] == max_iter
        assert rel(rep.solution, ref["solution"]) <= 1e-10
    else:
        assert abs(rep.iterations - ref["iterations"]) <= 2
        assert rel(rep.solution, ref["solution"]) <= 1e-8
    assert len(rep.residual_history) == rep.iterations + 1
    n = min(len(rep.residual_history), len(ref["residual_history"]))
    np.testing.assert_allclose(rep.residual_history[:n], ref["residual_history"][:n], rtol=1e-6)


@pytest.mark.parametrize("nx,ny,nc", [(64, 64, 3), (128, 64, 4)])
def test_two_stage_coarse_passes_match_reference(monkeypatch, nx, ny, nc):
    """Small meshes normally keep the one-pass coarse kernels; lifting the
    size threshold runs the two-stage ones (tmg_smarch.cuh) on every coarse
    level, against the reference hierarchy."""
    monkeypatch.setenv("TMG_SMARCH_MIN_NODES", "0")
    ops, sysc, b, _, _ = pair(nx, ny, nc, seed=7)
    rng = np.random.default_rng(8)
    f = rng.standard_normal(b.size)
    u = P.mg_cycle(ops, np.zeros_like(f), f, 1, 2, 2)
    want = sysc.vcycle(f, np.zeros_like(f), 1, 2, 2)
    assert rel(u, want) <= 1e-11
    rep = P.pcgmg_solve(ops, b, P.SolverConfig(tol=1e-8, max_iter=500))
    ref = sysc.solve(b, tol=1e-8, max_iter=500)
    assert abs(rep.iterations - ref["iterations"]) <= 2
    assert rel(rep.solution, ref["solution"]) <= 1e-8


def test_single_level_hierarchy_solves_in_one_iteration():
    """test_solvers.cpp:328-342 for the elasticity system."""
    ops, sysc, b, _, _ = pair(8, 8, 0)
    rep = P.pcgmg_solve(ops, b, P.SolverConfig(tol=1e-6))
    assert rep.converged and rep.iterations == 1
    ref = sysc.solve(b, tol=1e-6)
    assert rel(rep.solution, ref["solution"]) <= 1e-12


def test_errors_mirror_reference():
    g = P.GridLevel(10, 8)
    with pytest.raises(P.ConfigError):
        P.MultigridOperators(g, 2, 0.3, P.wall_boundary_conditions(g, "uniform"))
    ops, sysc, b, _, _ = pair(16, 16, 2)
    with pytest.raises(P.ConfigError):
        P.pcgmg_solve(ops, b, P.SolverConfig(pre_sweeps=2, post_sweeps=3))
    with pytest.raises(P.DimensionError):
        ops.set_moduli(np.ones(5))
    with pytest.raises(P.ConfigError):
        P.MultigridOperators(P.GridLevel(8, 8), 1, 0.3, P.BoundaryConditions([1000], []))
    # unconstrained structure: singular coarsest operator (solvers.cpp:144-148)
    # the reference stops at row 14, the first dependent row (its pivot there
    # is a rounding residue); the device treats a pivot within 16 n eps of
    # the row's diagonal as zero and stops at the same row
    free = P.MultigridOperators(P.GridLevel(8, 8), 2, 0.3, P.BoundaryConditions([], []))
    with pytest.raises(P.DefinitenessError) as err:
        free.set_moduli(np.ones(64))
    with pytest.raises(po.OracleError) as want:
        po.System("orc", 8, 8, np.ones(64), 0.3, [], []).build_mg(2)
    assert err.value.row == want.value.row == 14


def test_duplicate_fixed_dofs_follow_finish_assembly():
    g = P.GridLevel(16, 16)
    bc = P.wall_boundary_conditions(g, "uniform")
    bc.fixed_dofs = bc.fixed_dofs + bc.fixed_dofs[:6]
    ops, sysc, b, _, _ = pair(16, 16, 2, bc=bc)
    x = np.random.default_rng(8).standard_normal(sysc.n)
    assert np.max(np.abs(ops.apply(2, x) - sysc.matvec(2, x))) <= 1e-13 * np.max(np.abs(sysc.matvec(2, x)))
    rep = P.pcgmg_solve(ops, b, P.SolverConfig(tol=1e-8))
    ref = sysc.solve(b, tol=1e-8)
    assert rel(rep.solution, ref["solution"]) <= 1e-8


def test_preconditioner_is_symmetric():
    """test_solvers.cpp:387-409 / acceptance criterion 6."""
    ops, sysc, b, _, _ = pair(8, 8, 2)
    n = sysc.n
    m = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        m[:, j] = P.mg_cycle(ops, np.zeros(n), e)
    assert np.max(np.abs(m - m.T)) < 1e-10 * max(1.0, np.max(np.abs(m)))


def test_bitwise_determinism():
    ops, sysc, b, _, _ = pair(64, 64, 3)
    cfg = P.SolverConfig(tol=1e-9)
    r1 = P.pcgmg_solve(ops, b, cfg)
    r2 = P.pcgmg_solve(ops, b, cfg)
    assert r1.iterations == r2.iterations
    assert r1.residual_history == r2.residual_history
    assert np.array_equal(r1.solution, r2.solution)


@pytest.mark.parametrize("nx,ny", [(16, 16), (40, 24)])
def test_consumers_match_reference(nx, ny):
    ops, sysc, b, alpha, E = pair(nx, ny, 2)
    rep = P.pcgmg_solve(ops, b, P.SolverConfig(tol=1e-10))
    u = rep.solution
    en = P.element_energies(ops)
    en_r = po.element_energies("orc", nx, ny, u, 0.3)
    assert np.max(np.abs(en - en_r)) <= 1e-13 * np.max(np.abs(en_r))
    s = P.sensitivities(ops, alpha, MAT)
    s_r = po.sensitivities("orc", nx, ny, alpha, MAT.phase_moduli, MAT.penalty, 0.3, u)
    assert np.max(np.abs(s - s_r)) <= 1e-13 * np.max(np.abs(s_r))
    # alpha_void can be exactly 0 in the iid recipe: the reference then divides
    # by zero (mto.cpp:114); both sides must agree on where that happens
    floored = np.maximum(alpha, 1e-3)
    for a in (alpha, floored):
        for radius in (1.0, 1.5, 3.0):
            for ph in range(4):
                f = P.filter_sensitivities(ops, s[ph], a, ph, radius)
                f_r = po.filter_sensitivities("orc", nx, ny, a, ph, radius, s_r[ph])
                fin = np.isfinite(f_r)
                assert np.array_equal(fin, np.isfinite(f))
                assert np.array_equal(np.isnan(f), np.isnan(f_r))
                if fin.any():
                    scale = np.max(np.abs(f_r[fin]))
                    assert np.max(np.abs(f[fin] - f_r[fin])) <= 1e-12 * scale


def test_device_simp_matches_host_moduli():
    nx = ny = 32
    from helpers import moduli
    alpha, E = moduli(nx, ny, "iid", 4)
    g = P.GridLevel(nx, ny)
    bc = P.wall_boundary_conditions(g, "uniform")
    a = P.MultigridOperators(g, 3, 0.3, bc)
    a.set_density(alpha, MAT)
    b_ = P.MultigridOperators(g, 3, 0.3, bc)
    b_.set_moduli(E)
    x = np.random.default_rng(9).standard_normal(g.dof_count())
    ya, yb = a.apply(3, x), b_.apply(3, x)
    assert np.max(np.abs(ya - yb)) <= 1e-14 * np.max(np.abs(yb))


@pytest.mark.parametrize("tol,max_iter", [(1e-8, 500), (1e-12, 6), (1e-12, 1), (1e-12, 2), (1e-3, 500)])
@pytest.mark.parametrize("switch", ["TMG_NO_COND_NODES", "TMG_NO_DEVICE_LOOP"])
def test_device_stopping_test_matches_host_loop(monkeypatch, switch, tol, max_iter):
    """The iteration graphs skip the speculative rest of an iteration on the
    device once r_{it-1} meets the stopping test (a conditional graph node).
    The results must be bitwise those of the plain graphs (TMG_NO_COND_NODES),
    at convergence, at the iteration cap and on an early stop. The same holds
    for the whole loop as one graph (a conditional WHILE node, the default)
    against the per-iteration host loop (TMG_NO_DEVICE_LOOP)."""
    nx = ny = 128
    _, E = moduli(nx, ny, "iid", 4)
    g = P.GridLevel(nx, ny)
    bc = P.wall_boundary_conditions(g, "uniform")
    b = P.assemble_rhs(g, bc)
    cfg = P.SolverConfig(tol=tol, max_iter=max_iter)
    reps = []
    for off in ("0", "1"):
        monkeypatch.setenv(switch, off)
        ops = P.MultigridOperators(g, 4, 0.3, bc)
        ops.set_moduli(E, 0.6)
        reps.append((P.pcgmg_solve(ops, b, cfg), P.compliance(ops)))
    (a, ca), (c, cc) = reps
    assert a.iterations == c.iterations and a.converged == c.converged
    assert a.residual_history == c.residual_history
    assert np.array_equal(a.solution, c.solution) and ca == cc


@pytest.mark.parametrize("omega", [1.2, 2.0])
@pytest.mark.parametrize("device_loop", ["0", "1"])
def test_breakdown_raises_like_reference(monkeypatch, omega, device_loop):
    """An over-relaxed smoother makes the V-cycle indefinite: the reference
    throws PreconditionerError with z^T r and the iteration (solvers.cpp:
    362-366), at iteration 2 for omega 1.2 and at iteration 1 for 2.0 on this
    mesh. The device loop (one graph) and the host loop raise the same."""
    import re

    monkeypatch.setenv("TMG_NO_DEVICE_LOOP", "0" if device_loop == "1" else "1")
    ops, sysc, b, _, _ = pair(32, 32, 2, seed=4, omega=omega)
    with pytest.raises(po.OracleError) as want:
        sysc.solve(b, tol=1e-8, max_iter=300)
    with pytest.raises(P.PreconditionerError) as got:
        P.pcgmg_solve(ops, b, P.SolverConfig(tol=1e-8, max_iter=300))
    pat = r"z\^T r = (-?[0-9.]+) at iteration (\d+)"
    (zw, iw), (zg, ig) = re.search(pat, str(want.value)).groups(), re.search(pat, str(got.value)).groups()
    assert iw == ig
    assert abs(float(zg) - float(zw)) <= 1e-6 * abs(float(zw))


@pytest.mark.parametrize("nx,ny,nc,recipe,gamma", [(64, 64, 3, "iid", 1), (256, 128, 5, "checker", 1),
                                                   (96, 160, 4, "iid", 2), (1024, 512, 7, "iid", 1)])
def test_tile_kernels_match_marching(monkeypatch, nx, ny, nc, recipe, gamma):
    """Small coarse levels run the V(2,2) halves as shared-memory tiles
    (tmg_stile.cuh) with the marching kernels' per-node arithmetic, so every
    result is bitwise that of the marching path (TMG_STILE_MAX_NODES=0)."""
    _, E = moduli(nx, ny, recipe, 3)
    g = P.GridLevel(nx, ny)
    bc = P.wall_boundary_conditions(g, "uniform")
    b = P.assemble_rhs(g, bc)
    cfg = P.SolverConfig(tol=1e-10, max_iter=500, gamma=gamma)
    f = np.random.default_rng(2).standard_normal(b.size)
    reps = []
    for lim in ("1000000000", "0"):
        monkeypatch.setenv("TMG_STILE_MAX_NODES", lim)
        ops = P.MultigridOperators(g, nc, 0.3, bc)
        ops.set_moduli(E, 0.6)
        rep = P.pcgmg_solve(ops, b, cfg)
        reps.append((rep, P.compliance(ops), P.mg_cycle(ops, np.zeros_like(f), f, gamma=gamma)))
    (a, ca, va), (c, cc, vc) = reps
    assert a.converged and a.iterations == c.iterations
    assert a.residual_history == c.residual_history
    assert np.array_equal(a.solution, c.solution) and ca == cc
    assert np.array_equal(va, vc)


@pytest.mark.parametrize("nx,ny,nc,recipe,gamma", [(64, 64, 3, "iid", 1), (256, 128, 5, "checker", 1),
                                                   (96, 160, 4, "iid", 2), (512, 512, 6, "iid", 1)])
def test_tile_sizes_and_dependent_launch_are_bitwise(monkeypatch, nx, ny, nc, recipe, gamma):
    """The tile kernels come in 1/2/4/8-node sizes (TMG_STILE_TC{1,2,4}_NODES)
    and the V-cycle bottom launches with programmatic stream serialization
    (TMG_NO_PDL=1 turns it off); every combination performs the same per-node
    arithmetic, so solves, histories and one cycle are bitwise equal."""
    _, E = moduli(nx, ny, recipe, 8)
    g = P.GridLevel(nx, ny)
    bc = P.wall_boundary_conditions(g, "uniform")
    b = P.assemble_rhs(g, bc)
    cfg = P.SolverConfig(tol=1e-10, max_iter=500, gamma=gamma)
    f = np.random.default_rng(9).standard_normal(b.size)
    reps = []
    for env in ({}, {"TMG_NO_PDL": "1", "TMG_STILE_TC2_NODES": "0", "TMG_STILE_TC4_NODES": "0"},
                {"TMG_STILE_TC1_NODES": "1000000"}, {"TMG_STILE_TC4_NODES": "1000000", "TMG_STILE_TC2_NODES": "0"}):
        for k in ("TMG_NO_PDL", "TMG_STILE_TC1_NODES", "TMG_STILE_TC2_NODES", "TMG_STILE_TC4_NODES"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        ops = P.MultigridOperators(g, nc, 0.3, bc)
        ops.set_moduli(E, 0.6)
        rep = P.pcgmg_solve(ops, b, cfg)
        reps.append((rep, P.compliance(ops), P.mg_cycle(ops, np.zeros_like(f), f, gamma=gamma)))
    a, ca, va = reps[0]
    assert a.converged
    for c, cc, vc in reps[1:]:
        assert a.iterations == c.iterations and a.residual_history == c.residual_history
        assert np.array_equal(a.solution, c.solution) and ca == cc
        assert np.array_equal(va, vc)


@pytest.mark.parametrize("nx,ny,nc,recipe,gamma", [(64, 64, 3, "iid", 1), (256, 128, 5, "checker", 1),
                                                   (96, 160, 4, "iid", 2), (1024, 512, 7, "iid", 1)])
def test_specialised_coarse_kernels_are_bitwise(monkeypatch, nx, ny, nc, recipe, gamma):
    """The two-stage coarse kernels with stage A and stage B on separate warps
    (tmg_smarch2.cuh) perform the lockstep kernels' per-node arithmetic in the
    same order: every result is bitwise that of TMG_SMARCH_LOCKSTEP=1. The
    marching kernels run on every coarse level (TMG_STILE_MAX_NODES=0)."""
    monkeypatch.setenv("TMG_STILE_MAX_NODES", "0")
    _, E = moduli(nx, ny, recipe, 5)
    g = P.GridLevel(nx, ny)
    bc = P.wall_boundary_conditions(g, "uniform")
    b = P.assemble_rhs(g, bc)
    cfg = P.SolverConfig(tol=1e-10, max_iter=500, gamma=gamma)
    f = np.random.default_rng(4).standard_normal(b.size)
    reps = []
    for lockstep in ("0", "1"):
        monkeypatch.setenv("TMG_SMARCH_LOCKSTEP", lockstep)
        ops = P.MultigridOperators(g, nc, 0.3, bc)
        ops.set_moduli(E, 0.6)
        rep = P.pcgmg_solve(ops, b, cfg)
        reps.append((rep, P.compliance(ops), P.mg_cycle(ops, np.zeros_like(f), f, gamma=gamma)))
    (a, ca, va), (c, cc, vc) = reps
    assert a.converged and a.iterations == c.iterations
    assert a.residual_history == c.residual_history
    assert np.array_equal(a.solution, c.solution) and ca == cc
    assert np.array_equal(va, vc)


@pytest.mark.parametrize("nx,ny,nc,recipe", [(128, 128, 2, "iid"), (256, 128, 2, "checker"), (256, 256, 2, "iid"),
                                              (128, 256, 1, "iid")])
def test_large_coarsest_level_matches_reference(nx, ny, nc, recipe):
    """Reference configs with few coarsenings (the default num_coarsenings = 2,
    solvers.hpp:25) leave a coarsest level of thousands of dofs, which
    CholeskyFactor (solvers.cpp:89-152) accepts at any size. Above 2048 dofs
    the device factors the band in L2 and forms the explicit inverse with the
    banded / tiled kernels: same cycle, same solve, same iteration count."""
    ops, sysc, b, _, _ = pair(nx, ny, nc, recipe, 5)
    assert 2 * (nx // 2**nc + 1) * (ny // 2**nc + 1) > 2048
    rng = np.random.default_rng(3)
    f = rng.standard_normal(sysc.n)
    got = P.mg_cycle(ops, np.zeros(sysc.n), f, 1, 2, 2)
    want = sysc.vcycle(f, np.zeros(sysc.n), 1, 2, 2)
    assert rel(got, want) <= 1e-10
    cfg = P.SolverConfig(tol=1e-8, max_iter=2000, num_coarsenings=nc)
    rep = P.pcgmg_solve(ops, b, cfg)
    ref = sysc.solve(b, tol=1e-8, max_iter=2000)
    assert rep.converged and ref["converged"]
    assert abs(rep.iterations - ref["iterations"]) <= 2
    assert rel(rep.solution, ref["solution"]) <= 1e-8
    c_ref = sysc.compliance(ref["solution"])
    assert abs(P.compliance(ops) - c_ref) <= 1e-9 * abs(c_ref)


def test_large_coarsest_level_singular_and_limit():
    """An unconstrained structure fails at the first dependent pivot of the
    large banded factor too (solvers.cpp:144-148); beyond the documented limit
    the handle is refused with ConfigError."""
    free = P.MultigridOperators(P.GridLevel(128, 128), 2, 0.3, P.BoundaryConditions([], []))
    with pytest.raises(P.DefinitenessError):
        free.set_moduli(np.ones(128 * 128))
    with pytest.raises(P.ConfigError):
        P.MultigridOperators(P.GridLevel(512, 512), 2, 0.3, P.BoundaryConditions([], []))
    # a tall coarsest level (2 x 2049 nodes): the one-CTA band factor would run for minutes
    with pytest.raises(P.ConfigError):
        P.MultigridOperators(P.GridLevel(2, 4096), 1, 0.3, P.BoundaryConditions([], []))


@pytest.mark.parametrize("nx,ny,nc", [(64, 64, 3), (128, 96, 3), (160, 96, 4)])
def test_banded_coarsest_factor_is_the_dense_one(monkeypatch, nx, ny, nc):
    """The banded one-warp Cholesky of the coarsest matrix performs, inside
    the band, the dense kernel's operations in the same order, so the solve is
    bitwise the same as with the dense factor (TMG_DENSE_COARSE_FACTOR=1);
    the singular (unsupported) structure fails at setup either way."""
    _, E = moduli(nx, ny, "iid", 7)
    g = P.GridLevel(nx, ny)
    bc = P.wall_boundary_conditions(g, "uniform")
    b = P.assemble_rhs(g, bc)
    reps = []
    for dense in ("0", "1"):
        monkeypatch.setenv("TMG_DENSE_COARSE_FACTOR", dense)
        ops = P.MultigridOperators(g, nc, 0.3, bc)
        ops.set_moduli(E, 0.6)
        reps.append(P.pcgmg_solve(ops, b, P.SolverConfig(tol=1e-10, max_iter=300)))
        free = P.MultigridOperators(P.GridLevel(8, 8), 2, 0.3, P.BoundaryConditions([], []))
        with pytest.raises(P.DefinitenessError):
            free.set_moduli(np.ones(64))
    a, c = reps
    assert a.iterations == c.iterations and a.residual_history == c.residual_history
    assert np.array_equal(a.solution, c.solution)


def test_restrict_prolongate_known_answers():
    """test_grid.cpp:106-137 on the device transfer kernels: zeros restrict to
    zeros, and restrict(prolongate(spike)) is 0.5625 at the spike (the
    hand-composed full-weighting stencil) with its maximum there."""
    ops, _, _, _, _ = pair(8, 8, 1)
    fine, coarse = ops.level(1), ops.level(0)
    assert not np.any(ops.restrict(1, np.zeros(fine.dof_count())))
    for comp in (0, 1):
        c = np.zeros(coarse.dof_count())
        spike = 2 * coarse.node_index(2, 2) + comp
        c[spike] = 1.0
        back = ops.restrict(1, ops.prolongate(1, c))
        assert abs(back[spike] - 0.5625) <= 1e-14
        assert np.argmax(back) == spike and np.sum(back == back[spike]) == 1


def test_one_vcycle_contracts_poisson_residual():
    """test_solvers.cpp:344-355: one V(2,2)-cycle from zero reduces the
    Poisson residual (64^2, 5 coarsenings) by 5x or better; the device cycle
    is measured under the checker's assembled matrix."""
    g, nc = 64, 5
    ops = P.PoissonMultigrid(P.GridLevel(g, g), nc)
    sysc = po.poisson_system("orc", g, g, 1.0).build_mg(nc, 0.6)
    b = sysc.rhs()
    u = ops.vcycle(np.zeros_like(b), b, 1, 2, 2)
    after = np.linalg.norm(b - sysc.matvec(nc, u))
    assert after < 0.2 * np.linalg.norm(b)


def test_device_sensitivities_known_answers():
    """test_mto.cpp:72-114 on the device consumers: sensitivities vanish at
    u = 0 and are never positive; the adjoint sensitivities match central
    finite differences of the compliance of device solves (void modulus kept
    finite so the difference stays above roundoff)."""
    n, nc = 8, 2
    mat = P.MaterialModel(phase_moduli=[9.0, 3.0, 1.0, 1e-3], poisson_ratio=0.3, penalty=3.0)
    rng = np.random.default_rng(33)
    a = rng.uniform(0.05, 1.0, (n * n, 4))
    a /= a.sum(1, keepdims=True)
    g = P.GridLevel(n, n)
    bc = P.wall_boundary_conditions(g, "uniform")
    b = P.assemble_rhs(g, bc)
    ops = P.MultigridOperators(g, nc, 0.3, bc)
    cfg = P.SolverConfig(tol=1e-13, max_iter=500)

    def compliance(alpha):
        ops.set_moduli(P.effective_moduli(alpha, mat), 0.6)
        rep = P.pcgmg_solve(ops, b, cfg)
        assert rep.converged
        return P.compliance(ops)

    compliance(a)
    assert not np.any(P.sensitivities(ops, a, mat, np.zeros(g.dof_count())))
    assert np.all(P.sensitivities(ops, a, mat, rng.uniform(-1, 1, g.dof_count())) <= 0.0)
    ad = P.sensitivities(ops, a, mat)  # at the resident solution
    h = 1e-5
    for e in range(0, n * n, 5):
        for i in range(4):
            up, dn = a.copy(), a.copy()
            up[e, i] += h
            dn[e, i] -= h
            fd = (compliance(up) - compliance(dn)) / (2 * h)
            assert abs(fd - ad[i, e]) <= 1e-3 * max(abs(ad[i, e]), 1e-12), (e, i, fd, ad[i, e])


def test_device_filter_known_answers():
    """test_mto.cpp:116-135 on the device filter: radius <= 1 is the identity
    (bitwise), and on a uniform design a uniform field stays uniform under a
    radius-3 cone."""
    n = 12
    g = P.GridLevel(n, n)
    ops = P.MultigridOperators(g, 2, 0.3, P.wall_boundary_conditions(g, "uniform"))
    rng = np.random.default_rng(5)
    a = rng.uniform(0.05, 1.0, (n * n, 4))
    a /= a.sum(1, keepdims=True)
    raw = -rng.uniform(0.0, 2.0, n * n)
    assert np.array_equal(P.filter_sensitivities(ops, raw, a, 0, 1.0), raw)
    assert np.array_equal(P.filter_sensitivities(ops, raw, a, 1, 0.5), raw)
    uni = np.tile([0.3, 0.7], (n * n, 1))  # DensityField::uniform(8, 8, {0.3, 0.7}) of the reference test
    f = P.filter_sensitivities(ops, np.full(n * n, -1.75), uni, 0, 3.0)
    np.testing.assert_allclose(f, -1.75, rtol=1e-13)
