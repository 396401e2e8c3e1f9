"""Poisson pCGMG (the paper's Table 1 path) against
the pinned CPU checker, which is bit-exact to the reference's
assemble_poisson + build_multigrid_operators + pcgmg_solve.

Host inputs (element matrices, right-hand side) are checked bit for bit on
the CPU; the device operator, Galerkin levels, cycle and solve on the B200."""
import numpy as np
import pytest

import paper_2301_07457_b200 as P
from helpers import rel
from oracle import pyoracle as po


def test_host_rhs_bit_exact():
    for g, src in ((16, 1.0), (24, None)):
        rng = np.random.default_rng(g)
        source = rng.standard_normal((g + 1) ** 2) if src is None else src
        grid = P.GridLevel(g, g)
        want = po.poisson_system("orc", g, g, source).rhs()
        assert np.array_equal(P.assemble_poisson_rhs(grid, source), want)


def planes_to_dense(planes, nx, ny):
    """The five half-stencil planes as the full symmetric matrix."""
    n = (nx + 1) * (ny + 1)
    A = np.zeros((n, n))
    off = [(0, 0), (0, 1), (1, -1), (1, 0), (1, 1)]
    for x in range(nx + 1):
        for y in range(ny + 1):
            i = x * (ny + 1) + y
            for p, (dx, dy) in enumerate(off):
                x2, y2 = x + dx, y + dy
                if 0 <= x2 <= nx and 0 <= y2 <= ny:
                    j = x2 * (ny + 1) + y2
                    A[i, j] = planes[p, i]
                    A[j, i] = planes[p, i]
    return A


def csr_dense(off, col, val, n):
    A = np.zeros((n, n))
    for i in range(n):
        A[i, col[off[i]:off[i + 1]]] = val[off[i]:off[i + 1]]
    return A


@pytest.mark.gpu
@pytest.mark.parametrize("g", [4, 16, 32])
def test_operators_match_reference_levels(g):
    nc = P.poisson_full_depth(g)
    ops = P.PoissonMultigrid(P.GridLevel(g, g), nc)
    sysc = po.poisson_system("orc", g, g, 1.0).build_mg(nc, 0.6)
    for lvl in range(nc + 1):
        n_l = g >> (nc - lvl)
        got = planes_to_dense(ops.level_planes(lvl), n_l, n_l)
        want = csr_dense(*sysc.csr(lvl), (n_l + 1) ** 2)
        assert np.max(np.abs(got - want)) <= 1e-14 * np.max(np.abs(want)), lvl
        if lvl == nc:
            assert np.array_equal(got, want)  # the fine operator is bit-exact


@pytest.mark.gpu
@pytest.mark.parametrize("g,gamma", [(32, 1), (64, 1), (64, 2)])
def test_cycle_matches_reference(g, gamma):
    nc = P.poisson_full_depth(g)
    ops = P.PoissonMultigrid(P.GridLevel(g, g), nc)
    sysc = po.poisson_system("orc", g, g, 1.0).build_mg(nc, 0.6)
    rng = np.random.default_rng(g)
    f = rng.standard_normal((g + 1) ** 2)
    for u0 in (np.zeros_like(f), rng.standard_normal(f.size)):
        got = ops.vcycle(u0, f, gamma, 2, 2)
        want = sysc.vcycle(f, u0, gamma, 2, 2)
        assert rel(got, want) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("g", [16, 32, 64, 128, 256])
def test_paper_bench_solves(g):
    """bench.cpp:64-82: constant source 1, coarsest 2x2, tol 1e-6, omega 0.6,
    2+2 sweeps: the reference's iteration count and solution."""
    nc = P.poisson_full_depth(g)
    grid = P.GridLevel(g, g)
    ops = P.PoissonMultigrid(grid, nc)
    b = P.assemble_poisson_rhs(grid, 1.0)
    cfg = P.SolverConfig(tol=1e-6, max_iter=2000, num_coarsenings=nc)
    rep = ops.solve(b, cfg)
    sysc = po.poisson_system("orc", g, g, 1.0).build_mg(nc, 0.6)
    ref = sysc.solve(b, tol=1e-6, max_iter=2000)
    assert rep.converged and ref["converged"]
    assert abs(rep.iterations - ref["iterations"]) <= 2
    assert rel(rep.solution, ref["solution"]) <= 1e-8
    assert len(rep.residual_history) == rep.iterations + 1


@pytest.mark.gpu
def test_random_source_warm_start_and_errors():
    g = 64
    nc = P.poisson_full_depth(g)
    grid = P.GridLevel(g, g)
    rng = np.random.default_rng(3)
    src = rng.standard_normal((g + 1) ** 2)
    b = P.assemble_poisson_rhs(grid, src)
    ops = P.PoissonMultigrid(grid, nc)
    sysc = po.poisson_system("orc", g, g, src).build_mg(nc, 0.6)
    cfg = P.SolverConfig(tol=1e-10, max_iter=500)
    rep = ops.solve(b, cfg)
    ref = sysc.solve(b, tol=1e-10, max_iter=500)
    assert abs(rep.iterations - ref["iterations"]) <= 2 and rel(rep.solution, ref["solution"]) <= 1e-8
    x0 = rep.solution * 0.9
    warm = ops.solve(b, cfg, x0=x0)
    rw = sysc.solve(b, tol=1e-10, max_iter=500, x0=x0)
    assert abs(warm.iterations - rw["iterations"]) <= 2 and rel(warm.solution, rw["solution"]) <= 1e-8
    z = ops.solve(np.zeros_like(b), cfg)
    assert z.converged and z.iterations == 0 and z.residual_history == [0.0]
    with pytest.raises(P.ConfigError):
        ops.solve(b, P.SolverConfig(pre_sweeps=1, post_sweeps=2))
    with pytest.raises(P.ConfigError):
        P.PoissonMultigrid(P.GridLevel(12, 12), 3)


@pytest.mark.gpu
@pytest.mark.parametrize("g,nc", [(128, 1), (256, 2), (256, 1)])
def test_large_coarsest_level(g, nc):
    """Few coarsenings leave a coarsest level above 2048 dofs, which the
    reference's CholeskyFactor accepts (solvers.cpp:89-152): the large banded
    factor / tiled inverse path gives the reference's count and solution."""
    assert ((g >> nc) + 1) ** 2 > 2048
    grid = P.GridLevel(g, g)
    ops = P.PoissonMultigrid(grid, nc)
    b = P.assemble_poisson_rhs(grid, 1.0)
    rep = ops.solve(b, P.SolverConfig(tol=1e-8, max_iter=500, num_coarsenings=nc))
    sysc = po.poisson_system("orc", g, g, 1.0).build_mg(nc, 0.6)
    ref = sysc.solve(b, tol=1e-8, max_iter=500)
    assert rep.converged and ref["converged"]
    assert abs(rep.iterations - ref["iterations"]) <= 2
    assert rel(rep.solution, ref["solution"]) <= 1e-8
    rng = np.random.default_rng(g)
    f = rng.standard_normal((g + 1) ** 2)
    assert rel(ops.vcycle(np.zeros_like(f), f, 1, 2, 2), sysc.vcycle(f, np.zeros_like(f), 1, 2, 2)) <= 1e-11
