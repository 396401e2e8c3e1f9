"""Parity at BASELINE sizes (SURVEY.md 8(c) protocol), where the reference
itself is too slow to run inside a test:

c2 (2048^2, 16x16-element phase checkerboard, 1e9 contrast, 9 levels): the
CPU checker (bit-exact to the reference) still assembles and builds the
hierarchy here, so the device is compared against it directly: Galerkin
levels, one V(2,2)-cycle, and the GPU solution's residual under the
checker's assembled K.

c3 (1024^2, r_f 3, warm start, 8 levels): the optimizer closed loop for its
first five outer iterations against the checker (bit-exact to the
reference's optimize()): compliance history to 1e-8 (warm-started tol-1e-8
solves fix it only to about the solver tolerance: 7e-9 measured at outer
iteration 4), PCG counts within +-2 and the design to the north-star 1e-6.

c4 recipe at 4096^2 (the largest mesh the reference can assemble: its CSR
offsets are int, sparse.hpp:53, and 8192^2 has ~2.42e9 nonzeros): against a
fixture generated once from the unmodified reference (oracle/_ref) by
tests/golden/make_c4_recipe_4096.py -- iteration count +-2, residual history,
compliance 1e-9, u on a fixed dof sample 1e-8, |u| and four random
projections of u.

c4 (8192^2, 134M DOFs, 11 levels, the bench workload): size-independent
properties only: the residual recomputed through a different kernel (the
plain K.u pass) against the host right-hand side, compliance = b.u at
convergence, bitwise run-to-run determinism and the symmetry of the
preconditioner (test_solvers.cpp:387-409)."""
import numpy as np
import pytest

import paper_2301_07457_b200 as P
from helpers import MAT, moduli, rel
from oracle import pyoracle as po

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c2():
    nx = ny = 2048
    nc = 8
    _, E = moduli(nx, ny, "checker", 2)
    g = P.GridLevel(nx, ny)
    bc = P.wall_boundary_conditions(g, "uniform")
    ops = P.MultigridOperators(g, nc, 0.3, bc)
    ops.set_moduli(E, 0.6)
    sysc = po.System("orc", nx, ny, E, 0.3, bc.fixed_dofs, bc.point_loads).build_mg(nc, 0.6)
    return ops, sysc, sysc.rhs(), nc


def test_c2_galerkin_levels(c2):
    ops, sysc, _, nc = c2
    for lvl in (nc - 1, nc - 4, 1):
        off, col, val = sysc.csr(lvl)
        dval = ops.level_values(lvl, off, col)
        assert np.max(np.abs(dval - val)) <= 1e-13 * np.max(np.abs(val)), lvl


def test_c2_one_vcycle(c2):
    ops, sysc, _, _ = c2
    f = np.random.default_rng(2).standard_normal(sysc.n)
    got = P.mg_cycle(ops, np.zeros_like(f), f, 1, 2, 2)
    want = sysc.vcycle(f, np.zeros_like(f), 1, 2, 2)
    # 1e9 contrast: the symmetric 8-value Ke (<= 1 ulp per entry, DESIGN.md
    # 2) is amplified through the void phase; the reference's own
    # reassociation moves a cycle by the same order
    assert rel(got, want) <= 1e-10


def test_c2_solution_residual_under_reference_K(c2):
    """SURVEY.md 8(c) protocol for the 1e9-contrast configs. Plain CG's
    recursively updated residual drifts from the true one at this contrast:
    the reference's own tol-1e-8 solutions have true residuals of 2e-6 -
    6e-6 under its own K (measured at 256^2 - 1024^2 with this recipe), and
    the iteration count at which the recursive residual crosses 1e-8 is
    chaotic (reported, not gated). Gated: the device solution's true residual
    under the checker's assembled K is at that attainable level, and its true
    residuals under the two operators agree to 5 %. (The naive rounding bound
    64 eps |||K||u|||/||b|| is ~3e-4 here, useless against 4e-6 residuals:
    K u cancels over nine orders of magnitude. Measured differences of the
    two residuals are 0.8-1.2 %, i.e. 3-6e-8 absolute.)"""
    ops, sysc, b, nc = c2
    rep = P.pcgmg_solve(ops, b, P.SolverConfig(tol=1e-8, max_iter=2000, num_coarsenings=nc))
    assert rep.converged
    nb = np.linalg.norm(b)
    r_ref = np.linalg.norm(b - sysc.matvec(nc, rep.solution)) / nb
    r_dev = np.linalg.norm(b - ops.apply(nc, rep.solution)) / nb
    assert r_ref <= 1e-5
    assert abs(r_ref - r_dev) <= 0.05 * r_ref, (r_ref, r_dev)


@pytest.fixture(scope="module")
def c4():
    nx = ny = 8192
    nc = 10
    g = P.GridLevel(nx, ny)
    bc = P.wall_boundary_conditions(g, "uniform")
    E = P.effective_moduli(P.density_iid(nx, ny, 1), MAT)
    ops = P.MultigridOperators(g, nc, 0.3, bc)
    ops.set_moduli(E, 0.6)
    return ops, P.assemble_rhs(g, bc), nc


def test_c4_residual_compliance_determinism(c4):
    ops, b, nc = c4
    cfg = P.SolverConfig(tol=1e-8, max_iter=500, num_coarsenings=nc)
    rep = P.pcgmg_solve(ops, b, cfg)
    # the reference cannot run this mesh (int CSR offsets, sparse.hpp:53), so
    # the count is not gated against it here; the c4 recipe is pinned against
    # the reference at 4096^2 (test_c4_recipe_4096_matches_the_reference)
    assert rep.converged
    print(f"c4: {rep.iterations} PCG iterations")
    u = rep.solution
    # residual through the plain K.u pass (not the fused PCG kernels)
    r = b - ops.apply(nc, u)
    assert np.linalg.norm(r) / np.linalg.norm(b) <= 1e-8 * 1.001
    # compliance u^T K u equals b^T u up to u^T r
    c = P.compliance(ops)
    bu = float(b @ u)
    assert abs(c - bu) <= abs(float(u @ r)) + 1e-12 * abs(bu)
    again = P.pcgmg_solve(ops, b, cfg)
    assert again.iterations == rep.iterations and np.array_equal(again.solution, u)


def test_c4_preconditioner_symmetric(c4):
    ops, b, _ = c4
    rng = np.random.default_rng(4)
    x, y = rng.standard_normal(b.size), rng.standard_normal(b.size)
    zero = np.zeros_like(b)
    mx = P.mg_cycle(ops, zero, x, 1, 2, 2)
    my = P.mg_cycle(ops, zero, y, 1, 2, 2)
    lhs, rhs = float(y @ mx), float(x @ my)
    assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), abs(rhs))


def test_c3_first_outer_iterations():
    n, nc, k = 1024, 7, 5
    g = P.GridLevel(n, n)
    bc = P.wall_boundary_conditions(g, "uniform")
    phases = [1.0, 0.5, 0.2, 1e-9]
    fr = [0.15, 0.15, 0.15, 0.55]
    mat = P.MaterialModel(phase_moduli=phases, poisson_ratio=0.3, penalty=3.0)
    cfg = P.OptimConfig(volume_fractions=fr, filter_radius=3.0, warm_start=True, tol=1e-12, max_outer=k,
                        solver=P.SolverConfig(tol=1e-8, max_iter=2000, num_coarsenings=nc))
    ops = P.MultigridOperators(g, nc, 0.3, bc)
    got = P.optimize(ops, mat, cfg)
    want = po.optimize("orc", n, n, list(bc.fixed_dofs), list(bc.point_loads), phases, 3.0, 0.3, fr,
                       num_coarsenings=nc, filter_radius=3.0, tol=1e-12, warm_start=True, max_outer=k)
    assert got.outer_iterations == want["outer_iterations"] == k
    np.testing.assert_allclose(got.compliance_history, want["compliance_history"], rtol=1e-8)
    assert all(abs(a - b) <= 2 for a, b in zip(got.solver_iteration_history, want["solver_iteration_history"]))
    d = float(np.max(np.abs(got.density - want["density"])))
    print(f"c3 closed loop, {k} outer iterations: max |design diff| = {d:.2e}")
    assert d <= 1e-6


def test_c4_recipe_4096_matches_the_reference():
    """BASELINE c4's recipe (iid U(0,1) densities from seed 1, 10 levels down
    to the 8x8 coarsest grid, tol 1e-8) at 4096^2 against the unmodified
    reference's own pcgmg_solve (acceptance.cpp:156-190 drives it the same
    way). The density generator is pinned bit for bit to the reference's
    (tests/test_oracle_pin.py::test_bench_input_recipe_is_pinned)."""
    import pathlib

    fx = np.load(pathlib.Path(__file__).resolve().parent / "golden" / "c4_recipe_4096.npz")
    n, nc, seed = int(fx["nx"]), int(fx["num_coarsenings"]), int(fx["seed"])
    g = P.GridLevel(n, n)
    bc = P.wall_boundary_conditions(g, "uniform")
    E = P.effective_moduli(P.density_iid(n, n, seed), MAT)
    ops = P.MultigridOperators(g, nc, 0.3, bc)
    ops.set_moduli(E, 0.6)
    b = P.assemble_rhs(g, bc)
    rep = P.pcgmg_solve(ops, b, P.SolverConfig(tol=1e-8, max_iter=5000, num_coarsenings=nc))
    assert rep.converged and bool(fx["converged"])
    ref_it = int(fx["iterations"])
    print(f"4096^2 c4 recipe: device {rep.iterations} vs reference {ref_it} PCG iterations")
    assert abs(rep.iterations - ref_it) <= 2
    h = np.asarray(rep.residual_history)
    hr = fx["residual_history"]
    k = min(h.size, hr.size)
    np.testing.assert_allclose(h[:k], hr[:k], rtol=1e-6)
    u = rep.solution
    idx = fx["sample_index"]
    assert rel(u[idx], fx["u_sample"]) <= 1e-8
    un = float(fx["u_norm"])
    # | |u| - |u_ref| | <= |u - u_ref|: the north-star bar on u (1.5e-9 measured)
    assert abs(np.linalg.norm(u) - un) <= 1e-8 * un
    assert abs(P.compliance(ops) - float(fx["compliance"])) <= 1e-9 * abs(float(fx["compliance"]))
    for s, p in zip(fx["proj_seeds"], fx["projections"]):
        r = np.random.default_rng(int(s)).integers(0, 2, u.size, dtype=np.int8).astype(np.float64) * 2.0 - 1.0
        # |r.(u - u_ref)| <= |r| |u - u_ref| = sqrt(n) |u - u_ref| <= sqrt(n) 1e-8 |u_ref|
        assert abs(float(r @ u) - float(p)) <= 1e-8 * np.sqrt(u.size) * un
