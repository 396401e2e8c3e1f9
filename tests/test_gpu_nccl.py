"""The NCCL transport of the x-slab decomposition on the B200 (SURVEY.md
8(e)). A gpurun box has one GPU, and NCCL refuses two ranks on one device, so
the transport is driven as a one-rank communicator: tmg_gpu_create_nccl with
nranks = 1 turns the whole slab machinery on (partials all-reduced by
ncclAllReduce, ghost exchanges by grouped send/recv, the finest replicated
level and the stencil planes gathered by grouped ncclBroadcast, all captured
into the PCG graphs) and must solve BITWISE like the plain single-rank
handle, whose reductions finish the same global tile array in the same order.
Multi-rank NCCL runs are what bench.py --gpus N launches."""
import numpy as np
import pytest

import paper_2301_07457_b200 as P
from helpers import moduli

pytestmark = pytest.mark.gpu


def _pair(nx, ny, nc, rep=-1, recipe="iid", seed=0):
    _, E = moduli(nx, ny, recipe, seed)
    g = P.GridLevel(nx, ny)
    bc = P.wall_boundary_conditions(g, "uniform")
    one = P.MultigridOperators(g, nc, 0.3, bc)
    one.set_moduli(E, 0.6)
    nccl = P.MultigridOperators(g, nc, 0.3, bc, nccl=(1, 0, P.nccl_unique_id()), replicated_level=rep)
    nccl.set_moduli(E, 0.6)
    return one, nccl, P.assemble_rhs(g, bc)


def _same(a, b):
    assert a.iterations == b.iterations
    assert a.converged == b.converged
    assert a.residual_history == b.residual_history
    assert np.array_equal(a.solution, b.solution)


@pytest.mark.parametrize("rep", [-1, 3])
def test_nccl_one_rank_c1_solve_is_bitwise_the_single_rank_solve(rep):
    """BASELINE c1 exactly: 512^2, iid seed 0, 7 levels, tol 1e-8."""
    one, nccl, b = _pair(512, 512, 6, rep=rep)
    cfg = P.SolverConfig(tol=1e-8, max_iter=500, num_coarsenings=6)
    a = P.pcgmg_solve(one, b, cfg)
    c = P.pcgmg_solve(nccl, b, cfg)
    assert a.converged and a.iterations > 5
    _same(a, c)
    assert P.compliance(one) == P.compliance(nccl)
    # warm start and a W-cycle through the same communicator
    x0 = a.solution * 0.9
    _same(P.pcgmg_solve(one, b, cfg, x0=x0), P.pcgmg_solve(nccl, b, cfg, x0=x0))
    w = P.SolverConfig(tol=1e-8, max_iter=500, gamma=2, num_coarsenings=6)
    _same(P.pcgmg_solve(one, b, w), P.pcgmg_solve(nccl, b, w))


def test_nccl_one_rank_conditional_graphs(monkeypatch):
    """TMG_NCCL_COND_NODES=1: the device-side stopping test and the one-graph
    PCG loop with the NCCL collectives inside conditional bodies; bitwise the
    plain solve, including a capped one."""
    monkeypatch.setenv("TMG_NCCL_COND_NODES", "1")
    one, nccl, b = _pair(256, 256, 5, recipe="checker", seed=2)
    for cfg in (P.SolverConfig(tol=1e-8, max_iter=1000, num_coarsenings=5),
                P.SolverConfig(tol=1e-12, max_iter=7, num_coarsenings=5)):
        _same(P.pcgmg_solve(one, b, cfg), P.pcgmg_solve(nccl, b, cfg))


def test_nccl_one_rank_pipelined_solves_are_bitwise_the_single_rank_ones():
    """The bench's e2e leg at N > 1 runs the pipelined calls
    (tmg_gpu_stage_inputs / tmg_gpu_solve_staged / tmg_gpu_sync_outputs) on an
    NCCL handle: staged uploads of the rank's slab, the install, the setup with
    its plane gathers and the solve must give, problem for problem, bitwise
    the blocking single-rank solves."""
    g = P.GridLevel(256, 256)
    bc = P.wall_boundary_conditions(g, "uniform")
    cfg = P.SolverConfig(tol=1e-9, max_iter=2000)
    probs = []
    for k in range(3):
        _, E = moduli(256, 256, "iid" if k % 2 == 0 else "checker", 30 + k)
        probs.append((E, P.assemble_rhs(g, bc)))
    one = P.MultigridOperators(g, 5, 0.3, bc)
    want = []
    for E, b in probs:
        one.set_moduli(E, 0.6)
        want.append(P.pcgmg_solve(one, b, cfg))
    nccl = P.MultigridOperators(g, 5, 0.3, bc, nccl=(1, 0, P.nccl_unique_id()))
    got = P.pcgmg_solve_many(nccl, probs, cfg, 0.6)
    for r, w in zip(got, want):
        _same(r, w)
