"""The x-slab decomposition run end to end on one B200:
several ranks in one process exchange halos by device copies and all-reduce
the reduction partials (LocalComm); the NCCL path differs only in the
transport. Every per-node formula is partition-independent and the
reductions sum a global tile layout in one fixed order (SURVEY.md 8(e)
"deterministic reductions"), so the decomposed solve must reproduce the
single-rank solve BITWISE: iterations, residual history, solution and
compliance."""
import numpy as np
import pytest

import paper_2301_07457_b200 as P
from helpers import MAT, moduli, rel
from oracle import pyoracle as po

pytestmark = pytest.mark.gpu


def build(nx, ny, nc, slabs, rep=-1, recipe="iid", seed=0):
    _, E = moduli(nx, ny, recipe, seed)
    g = P.GridLevel(nx, ny)
    bc = P.wall_boundary_conditions(g, "uniform")
    ops = P.MultigridOperators(g, nc, 0.3, bc, slabs=slabs, replicated_level=rep)
    ops.set_moduli(E, 0.6)
    return ops, E, bc, P.assemble_rhs(g, bc)


CASES = [
    # nx, ny, coarsenings, slabs, replicated level (-1 = auto)
    (64, 32, 3, 2, 1),
    (64, 64, 3, 2, -1),
    (128, 64, 4, 3, 1),
    (128, 128, 5, 4, 2),
    (256, 64, 5, 2, 3),
    (256, 128, 2, 2, 0),  # coarsest level above 2048 dofs (65 x 33 nodes), replicated on both slabs
]


@pytest.mark.parametrize("nx,ny,nc,slabs,rep", CASES)
def test_slab_solve_matches_single_rank_and_reference(nx, ny, nc, slabs, rep):
    one, E, bc, b = build(nx, ny, nc, 1)
    many, _, _, _ = build(nx, ny, nc, slabs, rep)
    cfg = P.SolverConfig(tol=1e-8, max_iter=500)
    r1 = P.pcgmg_solve(one, b, cfg)
    rn = P.pcgmg_solve(many, b, cfg)
    ref = po.System("orc", nx, ny, E, 0.3, bc.fixed_dofs, bc.point_loads).build_mg(nc).solve(b, tol=1e-8)
    assert rn.converged
    assert rn.iterations == r1.iterations
    assert rn.residual_history == r1.residual_history
    assert np.array_equal(rn.solution, r1.solution)
    assert abs(rn.iterations - ref["iterations"]) <= 2
    assert rel(rn.solution, ref["solution"]) <= 1e-8
    assert P.compliance(many) == P.compliance(one)


@pytest.mark.parametrize("gamma,sweeps", [(1, 2), (2, 1), (1, 1), (2, 2)])
def test_slab_cycle_matches_single_rank(gamma, sweeps):
    nx, ny, nc = 128, 64, 4
    one, _, _, _ = build(nx, ny, nc, 1)
    many, _, _, _ = build(nx, ny, nc, 3, 1)
    rng = np.random.default_rng(21)
    f = rng.standard_normal(2 * (nx + 1) * (ny + 1))
    for u0 in (np.zeros_like(f), rng.standard_normal(f.size)):
        a = P.mg_cycle(one, u0, f, gamma, sweeps, sweeps)
        b = P.mg_cycle(many, u0, f, gamma, sweeps, sweeps)
        assert np.array_equal(b, a)


@pytest.mark.parametrize("zero", [True, False])
def test_two_stage_passes_on_slabs(monkeypatch, zero):
    """With the size threshold lifted every coarse level runs the two-stage
    passes (tmg_smarch.cuh), which read two ghost columns of their inputs and
    of the coarse correction; a zero start takes them, as inside pcgmg."""
    monkeypatch.setenv("TMG_SMARCH_MIN_NODES", "0")
    nx, ny, nc = 128, 64, 4
    one, _, _, _ = build(nx, ny, nc, 1)
    for slabs, rep in ((2, 1), (3, 1), (4, 2), (2, 3)):
        many, _, _, _ = build(nx, ny, nc, slabs, rep)
        rng = np.random.default_rng(5)
        f = rng.standard_normal(2 * (nx + 1) * (ny + 1))
        u0 = np.zeros_like(f) if zero else rng.standard_normal(f.size)
        a = P.mg_cycle(one, u0, f, 1, 2, 2)
        b = P.mg_cycle(many, u0, f, 1, 2, 2)
        assert np.array_equal(b, a), (slabs, rep)
        cfg = P.SolverConfig(tol=1e-8, max_iter=500)
        s1, sn = P.pcgmg_solve(one, a, cfg), P.pcgmg_solve(many, a, cfg)
        assert sn.iterations == s1.iterations
        assert sn.residual_history == s1.residual_history
        assert np.array_equal(sn.solution, s1.solution)


def test_slab_warm_start_and_determinism():
    nx, ny, nc = 128, 64, 4
    many, E, bc, b = build(nx, ny, nc, 2, 2)
    cfg = P.SolverConfig(tol=1e-8, max_iter=500)
    first = P.pcgmg_solve(many, b, cfg)
    again = P.pcgmg_solve(many, b, cfg)
    assert first.residual_history == again.residual_history
    assert np.array_equal(first.solution, again.solution)
    warm = P.pcgmg_solve(many, b, cfg, x0=first.solution * 0.98)
    ref = po.System("orc", nx, ny, E, 0.3, bc.fixed_dofs, bc.point_loads).build_mg(nc).solve(
        b, tol=1e-8, x0=first.solution * 0.98)
    assert abs(warm.iterations - ref["iterations"]) <= 2
    assert rel(warm.solution, ref["solution"]) <= 1e-8


@pytest.mark.parametrize("slabs", [2, 3, 4, 5])
def test_partition_independent_bitwise(slabs):
    """1 rank vs 2-5 slabs at a mesh where the reduction tiles are wider than
    the slab granularity: warm start, W-cycle and a capped solve (the
    stand-alone x/r update of the last iteration) all bitwise equal."""
    nx, ny, nc = 512, 256, 5
    one, _, _, b = build(nx, ny, nc, 1, recipe="checker", seed=3)
    many, _, _, _ = build(nx, ny, nc, slabs, recipe="checker", seed=3)
    x0 = np.random.default_rng(8).standard_normal(b.size) * 1e-3
    for cfg, kw in ((P.SolverConfig(tol=1e-8, max_iter=500), {}),
                    (P.SolverConfig(tol=1e-8, max_iter=500), {"x0": x0}),
                    (P.SolverConfig(tol=1e-8, max_iter=500, gamma=2, pre_sweeps=1, post_sweeps=1), {}),
                    (P.SolverConfig(tol=1e-12, max_iter=7), {})):
        r1, rn = P.pcgmg_solve(one, b, cfg, **kw), P.pcgmg_solve(many, b, cfg, **kw)
        assert rn.iterations == r1.iterations and rn.converged == r1.converged
        assert rn.residual_history == r1.residual_history
        assert np.array_equal(rn.solution, r1.solution)
