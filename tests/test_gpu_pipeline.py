"""Pipelined solves (tmg_gpu_stage_inputs / tmg_gpu_solve_staged /
tmg_gpu_sync_outputs, include/tmg_gpu.h): a stream of independent problems
whose host<->device copies overlap the neighbouring solves must give, problem
for problem, bitwise the results of the blocking set_moduli + pcgmg_solve
pair (solvers.cpp:460-530) on the same handle geometry."""
import numpy as np
import pytest

import paper_2301_07457_b200 as P
from helpers import moduli

pytestmark = pytest.mark.gpu


def problems(nx, ny, n):
    g = P.GridLevel(nx, ny)
    out = []
    for k in range(n):
        _, E = moduli(nx, ny, "iid" if k % 2 == 0 else "checker", 20 + k)
        bc = P.wall_boundary_conditions(g, "uniform" if k % 3 else "point")
        out.append((E, P.assemble_rhs(g, bc)))
    return g, P.wall_boundary_conditions(g, "uniform"), out


@pytest.mark.parametrize("nx,ny,nc,slabs,pinned", [(128, 96, 4, 1, True), (256, 256, 5, 1, False),
                                                   (512, 512, 6, 2, True)])
def test_pipelined_solves_are_bitwise_the_blocking_ones(nx, ny, nc, slabs, pinned):
    g, bc, probs = problems(nx, ny, 5)
    cfg = P.SolverConfig(tol=1e-9, max_iter=2000)
    ops = P.MultigridOperators(g, nc, 0.3, bc, slabs=slabs)
    want = []
    for E, b in probs:
        ops.set_moduli(E, 0.6)
        want.append((P.pcgmg_solve(ops, b, cfg), P.compliance(ops)))
    if pinned:
        bufs = []
        staged = []
        for E, b in probs:
            pe, pb = P.PinnedArray(E.size), P.PinnedArray(b.size)
            pe.a[:] = E
            pb.a[:] = b
            bufs += [pe, pb]
            staged.append((pe.a, pb.a))
        outs = [P.PinnedArray(g.dof_count()) for _ in probs]
        got = P.pcgmg_solve_many(ops, staged, cfg, 0.6, outputs=[o.a for o in outs])
    else:
        got = P.pcgmg_solve_many(ops, probs, cfg, 0.6)
    # the last problem's operators stay resident
    assert P.compliance(ops) == want[-1][1]
    for r, (w, _) in zip(got, want):
        assert r.converged and r.iterations == w.iterations
        assert r.residual_history == w.residual_history
        assert np.array_equal(r.solution, w.solution)


def test_pipeline_errors_mirror_the_blocking_calls():
    g, bc, probs = problems(64, 64, 1)
    ops = P.MultigridOperators(g, 3, 0.3, bc)
    lib = ops.lib
    x = np.empty(g.dof_count())
    with pytest.raises(P.ConfigError, match="no inputs staged"):
        ops._check(lib.tmg_gpu_solve_staged(ops.h, 0, 0.6, 1e-8, 100, 1, 2, 2, P._lib.dptr(x), None, None, None,
                                            None, None, 0, None))
    E, b = probs[0]
    with pytest.raises(P.DimensionError, match="slot"):
        ops._check(lib.tmg_gpu_stage_inputs(ops.h, 2, P._lib.dptr(E), E.size, P._lib.dptr(b)))
    with pytest.raises(P.DimensionError, match="element modulus count"):
        P.pcgmg_solve_many(ops, [(E[:-1], b)], P.SolverConfig())
    # pre != post is rejected like pcgmg_solve (solvers.cpp:518-521)
    with pytest.raises(P.ConfigError):
        P.pcgmg_solve_many(ops, [(E, b)], P.SolverConfig(pre_sweeps=2, post_sweeps=1))
