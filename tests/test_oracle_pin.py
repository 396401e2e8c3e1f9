"""Pin the CPU checker (oracle/liboracle.so) before trusting it.

1. Against the committed golden fixtures tests/golden/*.npz, generated from
   the unmodified reference by tests/golden/make_golden.py: every quantity
   must match BIT FOR BIT (the restatement performs the reference's floating
   point operations in the reference's order).
2. Against the reference itself (oracle/_ref, compiled from /root/reference
   by oracle/Makefile) on fresh random cases, when it is built.
3. Against the reference's own known-answer tests: the closed-form Q4
   stiffness (proj/tests/test_fem.cpp:19-34, oracles.hpp:193-215) and the
   filter identity / uniformity / conservation properties
   (proj/tests/test_mto.cpp:116-184).
"""
import pathlib

import numpy as np
import pytest

from oracle import pyoracle as po

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"
CASES = sorted(p for p in GOLDEN.glob("wall*.npz"))
PHASES = np.array([1.0, 0.5, 0.2, 1e-9])


def closed_form_q4(e, nu):
    """proj/tests/oracles.hpp:193-215 (the reference's own oracle)."""
    k = [0.5 - nu / 6.0, 0.125 + nu / 8.0, -0.25 - nu / 12.0, -0.125 + 3.0 * nu / 8.0,
         -0.25 + nu / 12.0, -0.125 - nu / 8.0, nu / 6.0, 0.125 - 3.0 * nu / 8.0]
    idx = [[0, 1, 2, 3, 4, 5, 6, 7], [1, 0, 7, 6, 5, 4, 3, 2], [2, 7, 0, 5, 6, 3, 4, 1],
           [3, 6, 5, 0, 7, 2, 1, 4], [4, 5, 6, 7, 0, 1, 2, 3], [5, 4, 3, 2, 1, 0, 7, 6],
           [6, 3, 4, 1, 2, 7, 0, 5], [7, 2, 1, 4, 3, 6, 5, 0]]
    c = e / (1.0 - nu * nu)
    return np.array([[c * k[idx[i][j]] for j in range(8)] for i in range(8)])


def test_golden_fixtures_exist():
    assert len(CASES) >= 4
    assert (GOLDEN / "element_stiffness.npz").exists()


def test_element_stiffness_bitwise_and_closed_form():
    g = np.load(GOLDEN / "element_stiffness.npz")
    for nu in (0.3, 0.42):
        k = po.element_stiffness("orc", 1.0, nu)
        assert np.array_equal(k, g[f"ke_nu{nu}"])
        assert np.max(np.abs(k - closed_form_q4(1.0, nu))) <= 1e-12 * np.max(np.abs(k))
        assert np.array_equal(k, k.T)
        # rigid translations produce no force (test_fem.cpp:49-61)
        for c in range(2):
            assert np.max(np.abs(k[:, c::2].sum(axis=1))) < 1e-12


@pytest.mark.parametrize("path", CASES, ids=lambda p: p.stem)
def test_oracle_matches_reference_golden_bitwise(path):
    g = np.load(path)
    nx, ny, nc = int(g["nx"]), int(g["ny"]), int(g["nc"])
    loads = list(zip(g["load_dofs"].tolist(), g["load_vals"].tolist()))
    E = po.effective_moduli("orc", nx, ny, g["alpha"], PHASES, 3.0)
    assert np.array_equal(E, g["E"])
    s = po.System("orc", nx, ny, E, 0.3, g["fixed"], loads).build_mg(nc, 0.6)
    assert np.array_equal(s.rhs(), g["b"])
    for lvl in range(nc + 1):
        off, col, val = s.csr(lvl)
        assert np.array_equal(off, g[f"L{lvl}_off"])
        assert np.array_equal(col, g[f"L{lvl}_col"])
        assert np.array_equal(val, g[f"L{lvl}_val"]), f"level {lvl}"
    x0 = g["x0"] if g["x0"].size else None
    r = s.solve(g["b"], tol=1e-8, max_iter=500, x0=x0)
    assert r["iterations"] == int(g["iterations"])
    assert np.array_equal(r["residual_history"], g["hist"])
    assert np.array_equal(r["solution"], g["x"])
    assert s.compliance(g["x"]) == float(g["compliance"])
    f = g["f"]
    assert np.array_equal(s.vcycle(f, np.zeros_like(f), 1, 2, 2), g["vcycle_v22"])
    assert np.array_equal(s.vcycle(f, np.zeros_like(f), 2, 1, 1), g["vcycle_w11"])
    assert np.array_equal(po.element_energies("orc", nx, ny, g["x"], 0.3), g["energies"])
    sens = po.sensitivities("orc", nx, ny, g["alpha"], PHASES, 3.0, 0.3, g["x"])
    assert np.array_equal(sens, g["sens"])
    for radius in (1.5, 3.0):
        filt = np.stack([po.filter_sensitivities("orc", nx, ny, g["alpha_floored"], ph, radius, sens[ph])
                         for ph in range(4)])
        assert np.array_equal(filt, g[f"filter_r{radius}"])


@pytest.mark.skipif(not po.available("ref"), reason="oracle/_ref not built (no /root/reference)")
@pytest.mark.parametrize("nx,ny,nc,seed", [(8, 16, 1, 11), (20, 12, 2, 12), (40, 40, 3, 13)])
def test_oracle_matches_live_reference_bitwise(nx, ny, nc, seed):
    rng = np.random.default_rng(seed)
    E = rng.uniform(1e-3, 2.0, nx * ny)
    fixed = [2 * x * (ny + 1) for x in range(nx + 1)] + [2 * x * (ny + 1) + 1 for x in range(0, nx + 1, 2)]
    loads = [(2 * (x * (ny + 1) + ny) + 1, -rng.uniform()) for x in range(nx + 1)]
    out = {}
    for kind in ("orc", "ref"):
        s = po.System(kind, nx, ny, E, 0.27, fixed, loads).build_mg(nc, 0.7)
        b = s.rhs()
        r = s.solve(b, tol=1e-10, max_iter=400, gamma=2, pre=1, post=1)
        out[kind] = (b, r, [s.csr(l)[2] for l in range(nc + 1)], s.compliance(r["solution"]))
    (b0, r0, c0, k0), (b1, r1, c1, k1) = out["orc"], out["ref"]
    assert np.array_equal(b0, b1)
    assert r0["iterations"] == r1["iterations"]
    assert np.array_equal(r0["solution"], r1["solution"])
    assert all(np.array_equal(a, b) for a, b in zip(c0, c1))
    assert k0 == k1


@pytest.mark.skipif(not po.available("ref"), reason="oracle/_ref not built (no /root/reference)")
def test_error_behaviour_matches_reference():
    nx = ny = 8
    E = np.ones(nx * ny)
    for kind in ("orc", "ref"):
        # unconstrained structure: singular coarsest matrix (solvers.cpp:144-148)
        s = po.System(kind, nx, ny, E, 0.3, [], [(2 * ((nx // 2) * (ny + 1) + ny) + 1, -1.0)])
        with pytest.raises(po.OracleError) as ei:
            s.build_mg(2)
        assert ei.value.code == 3 and ei.value.row == 14
        # fixed and loaded dof (fem.cpp:122-124)
        with pytest.raises(po.OracleError) as ei:
            po.System(kind, nx, ny, E, 0.3, [1], [(1, 1.0)])
        assert ei.value.code == 1
        # divisibility (grid.cpp:66-73)
        s = po.System(kind, nx, ny, E, 0.3, [0, 1], [(5, 1.0)])
        with pytest.raises(po.OracleError) as ei:
            s.build_mg(4)
        assert ei.value.code == 1


def test_filter_properties_of_the_reference_tests():
    """test_mto.cpp:116-184 (identity for r <= 1, uniform field, conservation)."""
    nx, ny = 7, 7
    rng = np.random.default_rng(8)
    a = np.tile([0.4, 0.6], (nx * ny, 1))
    raw = -rng.uniform(0.0, 1.0, nx * ny)
    assert np.array_equal(po.filter_sensitivities("orc", nx, ny, a, 0, 1.0, raw), raw)
    uni = np.full(nx * ny, -1.75)
    assert np.allclose(po.filter_sensitivities("orc", nx, ny, a, 0, 3.0, uni), -1.75, rtol=1e-13)
    rf = 2.5
    f = po.filter_sensitivities("orc", nx, ny, a, 0, rf, raw)
    for ex in range(nx):
        for ey in range(ny):
            ws = wr = 0.0
            for jx in range(nx):
                for jy in range(ny):
                    w = rf - np.sqrt((ex - jx) ** 2 + (ey - jy) ** 2)
                    if w > 0:
                        ws += w
                        wr += w * raw[jx * ny + jy]
            assert abs(f[ex * ny + ey] * ws - wr) <= 1e-12 * abs(wr)


def _oc_runs():
    d = np.load(GOLDEN / "oc_pair.npz")
    tags = sorted({k[: -len("_args")] for k in d.files if k.endswith("_args")})
    return d, tags


def test_oc_update_pair_golden_bit_exact():
    """oc_update_pair (mto.cpp:142-227): both bisection branches and the
    MultiplierError path, against the reference's own outputs."""
    d, tags = _oc_runs()
    assert len(tags) >= 20
    for t in tags:
        pa, pb, target, damping, eps = d[t + "_args"]
        out, st = po.oc_update_pair("orc", d[t + "_alpha"], int(pa), int(pb), d[t + "_sa"], d[t + "_sb"],
                                    float(target), d[t + "_move"], float(damping), float(eps))
        assert st == int(d[t + "_status"]), t
        assert np.array_equal(out, d[t + "_out"]), t


def test_oc_update_pair_matches_live_reference():
    if not po.available("ref"):
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(11)
    for trial in range(8):
        ne, nph = 300 + 91 * trial, 3 + trial % 2
        a = rng.uniform(0.05, 1.0, (ne, nph))
        a /= a.sum(1, keepdims=True)
        sa, sb = -rng.uniform(0, 2, ne), -rng.uniform(0, 2, ne)
        if trial == 5:
            sb = sa - rng.uniform(0.1, 1, ne)  # uniform-shift branch
        move = rng.uniform(0.01, 0.2, ne) if trial % 3 else np.full(ne, 0.2)
        target = a[:, 0].mean() + (0.02 if trial % 2 else -0.02)
        r1, s1 = po.oc_update_pair("ref", a, 0, nph - 1, sa, sb, target, move, 0.3 + 0.1 * trial)
        r2, s2 = po.oc_update_pair("orc", a, 0, nph - 1, sa, sb, target, move, 0.3 + 0.1 * trial)
        assert s1 == s2 and np.array_equal(r1, r2)


def _wall(n):
    fixed, loads = [], []
    for x in range(n + 1):
        node = x * (n + 1)
        fixed += [2 * node, 2 * node + 1]
        loads.append((2 * (x * (n + 1) + n) + 1, -1.0 / (n + 1)))
    return fixed, loads


def test_optimize_golden_bit_exact():
    """The whole optimizer loop (mto.cpp:229-354) against the reference's own
    OptimReport: density and every history bit for bit."""
    d = np.load(GOLDEN / "optimize.npz")
    for tag in ("n16", "n24_warm"):
        n, radius, max_outer, nc, warm, sweeps = d[tag + "_args"]
        fixed, loads = _wall(int(n))
        r = po.optimize("orc", int(n), int(n), fixed, loads, PHASES, 3.0, 0.3, [0.15, 0.15, 0.15, 0.55],
                        filter_radius=float(radius), tol=1e-12, max_outer=int(max_outer), num_coarsenings=int(nc),
                        warm_start=bool(warm), inner_sweeps=int(sweeps))
        for k in ("density", "compliance_history", "change_history", "solver_iteration_history",
                  "outer_iterations", "total_solver_iterations", "converged"):
            assert np.array_equal(np.asarray(r[k]), d[f"{tag}_{k}"]), (tag, k)


def test_optimize_matches_live_reference():
    if not po.available("ref"):
        pytest.skip("oracle/_ref not built")
    fixed, loads = _wall(20)
    kw = dict(filter_radius=2.0, tol=1e-3, max_outer=5, num_coarsenings=1, move_limit=0.1, oc_damping=0.7)
    a = po.optimize("ref", 20, 20, fixed, loads, PHASES, 3.0, 0.3, [0.2, 0.1, 0.1, 0.6], **kw)
    b = po.optimize("orc", 20, 20, fixed, loads, PHASES, 3.0, 0.3, [0.2, 0.1, 0.1, 0.6], **kw)
    for k in a:
        assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k


def _full_depth(g):
    d = 0
    while g > 2:
        g //= 2
        d += 1
    return d


@pytest.mark.parametrize("tag,g", [("g16", 16), ("g64", 64), ("g32_rand", 32)])
def test_poisson_golden_bit_exact(tag, g):
    """assemble_poisson + the Galerkin hierarchy + pcgmg on a 1-dof grid
    (fem.cpp:232-276, bench.cpp:64-82) against the reference's own outputs."""
    d = np.load(GOLDEN / "poisson.npz")
    s = po.poisson_system("orc", g, g, d[tag + "_source"]).build_mg(_full_depth(g), 0.6)
    assert np.array_equal(s.rhs(), d[tag + "_b"])
    for lvl in range(_full_depth(g) + 1):
        for got, key in zip(s.csr(lvl), ("off", "col", "val")):
            assert np.array_equal(got, d[f"{tag}_L{lvl}_{key}"]), (lvl, key)
    r = s.solve(d[tag + "_b"], tol=1e-6, max_iter=2000)
    assert r["iterations"] == int(d[tag + "_iterations"])
    assert np.array_equal(r["solution"], d[tag + "_x"])
    assert np.array_equal(r["residual_history"], d[tag + "_hist"])
    assert np.array_equal(s.vcycle(d[tag + "_f"], np.zeros(s.n), 1, 2, 2), d[tag + "_vcycle"])


def _make_golden():
    import importlib.util

    spec = importlib.util.spec_from_file_location("make_golden", GOLDEN / "make_golden.py")
    mg = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mg)
    return mg


@pytest.mark.parametrize("nx,ny,seed", [(8, 8, 0), (16, 12, 1), (24, 40, 7)])
def test_bench_input_recipe_is_pinned(nx, ny, seed):
    """The BASELINE density recipe (std::mt19937_64 with the
    oracles.hpp:21-23 bit recipe) four ways, bit for bit: the product's host
    generator (tmg_inputs_density_iid, which feeds every bench input), the
    independent pure-Python restatement in make_golden.py, the C checker and
    the reference's own oracle::Rng through oracle/_ref."""
    import paper_2301_07457_b200 as P

    mg = _make_golden()
    want = mg.density(nx, ny, seed)
    assert np.array_equal(P.density_iid(nx, ny, seed), want)
    assert np.array_equal(po.density_iid("orc", nx, ny, seed), want)
    if po.available("ref"):
        assert np.array_equal(po.density_iid("ref", nx, ny, seed), want)
        E = po.effective_moduli("ref", nx, ny, want, PHASES, 3.0)
        assert np.array_equal(P.effective_moduli(want, P.MaterialModel()), E)


def test_bench_input_recipe_at_scale():
    """c1 (512^2, seed 0) and a 1024^2 seed-1 prefix of the c4 recipe: product,
    C checker and reference generators agree bit for bit; the checkerboard
    likewise (c2 recipe, 16x16 blocks)."""
    import paper_2301_07457_b200 as P

    kinds = ["orc"] + (["ref"] if po.available("ref") else [])
    for nx, seed in ((512, 0), (1024, 1)):
        a = P.density_iid(nx, nx, seed)
        for k in kinds:
            assert np.array_equal(po.density_iid(k, nx, nx, seed), a), (k, nx)
    c = P.density_checker(256, 256, 16, 2)
    for k in kinds:
        assert np.array_equal(po.density_checker(k, 256, 256, 16, 2), c), k


def test_bench_supports_and_load_match_the_product():
    import paper_2301_07457_b200 as P

    for nx, ny in ((8, 8), (16, 32)):
        bc = P.wall_boundary_conditions(P.GridLevel(nx, ny), "uniform")
        fixed, loads = po.wall_uniform_bc(nx, ny)
        assert fixed == bc.fixed_dofs
        assert loads == bc.point_loads
