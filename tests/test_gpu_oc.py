"""The OC exchange on the B200 (tmg_gpu_oc_update_pair, SURVEY.md 8(f)
item 1) against the pinned CPU checker: oc_update_pair (mto.cpp:142-227) on
the reference's own golden inputs and on densities and filtered sensitivities
taken from GPU solves.

The device sums the bisection means in a fixed tree instead of sequentially,
and its pow differs from glibc's by at most an ulp or two, so the densities
agree to ~1e-15, not bit for bit; the branch taken at every bisection step
(and so the multiplier) is the same. Pair sums are preserved exactly."""
import pathlib

import numpy as np
import pytest

import paper_2301_07457_b200 as P
from helpers import MAT, moduli
from oracle import pyoracle as po

pytestmark = pytest.mark.gpu
GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"


def ops_for(nx, ny, nc=2):
    g = P.GridLevel(nx, ny)
    ops = P.MultigridOperators(g, nc, 0.3, P.wall_boundary_conditions(g, "uniform"))
    return ops


def check_same(got, want, alpha, pa, pb):
    assert np.max(np.abs(got - want)) <= 1e-13
    # untouched phases are untouched, the pair sum is kept
    others = [i for i in range(alpha.shape[1]) if i not in (pa, pb)]
    assert np.array_equal(got[:, others], alpha[:, others])
    assert np.max(np.abs((got[:, pa] + got[:, pb]) - (alpha[:, pa] + alpha[:, pb]))) <= 1e-15


def test_golden_cases():
    d = np.load(GOLDEN / "oc_pair.npz")
    tags = sorted({k[: -len("_args")] for k in d.files if k.endswith("_args")})
    cache = {}
    for t in tags:
        pa, pb, target, damping, eps = d[t + "_args"]
        pa, pb = int(pa), int(pb)
        alpha = d[t + "_alpha"]
        ne = alpha.shape[0]
        nx = {"wall8_l2": 8, "wall16_l3_point": 16, "wall32x16_l2": 32, "wall24x40_l3": 24}[t.rsplit("_", 1)[0]]
        ny = ne // nx
        if (nx, ny) not in cache:
            cache[(nx, ny)] = ops_for(nx, ny, 1)
        ops = cache[(nx, ny)]
        got = np.array(alpha, copy=True)
        if int(d[t + "_status"]) == 8:
            with pytest.raises(P.MultiplierError):
                P.oc_update_pair(ops, got, pa, pb, d[t + "_sa"], d[t + "_sb"], float(target), d[t + "_move"],
                                 float(damping), float(eps))
            assert np.array_equal(got, alpha)  # unchanged on failure
            continue
        P.oc_update_pair(ops, got, pa, pb, d[t + "_sa"], d[t + "_sb"], float(target), d[t + "_move"],
                         float(damping), float(eps))
        check_same(got, d[t + "_out"], alpha, pa, pb)


@pytest.mark.parametrize("nx,ny,seed", [(64, 64, 0), (128, 96, 3), (256, 256, 1)])
def test_from_a_gpu_solve(nx, ny, seed):
    """One outer OC step's inputs: sensitivities and filtered sensitivities
    of a GPU solve, every phase pair, scalar and per-element move limits."""
    a, E = moduli(nx, ny, "iid", seed)
    a = np.maximum(a, 1e-3)
    a /= a.sum(1, keepdims=True)
    g = P.GridLevel(nx, ny)
    nc = int(np.log2(min(nx, ny) // 8))  # coarsest grid about 8 elements across
    ops = P.MultigridOperators(g, nc, 0.3, P.wall_boundary_conditions(g, "uniform"))
    ops.set_moduli(P.effective_moduli(a, MAT), 0.6)
    P.pcgmg_solve(ops, P.assemble_rhs(g, P.wall_boundary_conditions(g, "uniform")), P.SolverConfig())
    raw = P.sensitivities(ops, a, MAT)
    filt = [P.filter_sensitivities(ops, raw[i], a, i, 1.5) for i in range(4)]
    rng = np.random.default_rng(seed)
    steps = []
    for pa in range(3):
        for pb in range(pa + 1, 4):
            move = 0.2 if (pa + pb) % 2 else rng.uniform(0.02, 0.2, nx * ny)
            target = float(a[:, pa].mean() * (1.0 + 0.05 * (pb - 2)))
            want, st = po.oc_update_pair("orc", a, pa, pb, filt[pa], filt[pb], target, move, 0.5)
            got = np.array(a, copy=True)
            if st == 8:
                with pytest.raises(P.MultiplierError):
                    P.oc_update_pair(ops, got, pa, pb, filt[pa], filt[pb], target, move, 0.5)
                continue
            P.oc_update_pair(ops, got, pa, pb, filt[pa], filt[pb], target, move, 0.5)
            check_same(got, want, a, pa, pb)
            assert abs(got[:, pa].mean() - target) <= 1e-6
            steps.append(P.oc_timings(ops)[1])
    assert steps and all(1 <= s <= 101 for s in steps)


def test_errors():
    ops = ops_for(16, 16)
    a = np.full((256, 4), 0.25)
    s = np.zeros(256)
    with pytest.raises(P.ConfigError):
        P.oc_update_pair(ops, a, 1, 1, s, s, 0.25, 0.2, 0.5)
    with pytest.raises(P.DimensionError):
        P.oc_update_pair(ops, a, 0, 4, s, s, 0.25, 0.2, 0.5)
    with pytest.raises(P.DimensionError):
        P.oc_update_pair(ops, a[:100].copy(), 0, 1, s[:100], s[:100], 0.25, 0.2, 0.5)
