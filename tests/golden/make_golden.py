#!/usr/bin/env python3
"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

The reference (topopt-mg) ships no golden vectors, so the
fixtures are produced by running its own code path -- assemble_from_moduli,
build_multigrid_operators, mg_cycle, pcgmg_solve, compliance,
element_energies, sensitivities, filter_sensitivities, oc_update_pair -- through the C-ABI
shim oracle/ref_shim.cpp on small seeded inputs. tests/test_oracle_pin.py
then pins the committed plain-C oracle to these files bit for bit, so the
oracle stays pinned even where /root/reference is absent (the GPU box).

Run from the repo root (needs /root/reference and `make -C oracle ref`):
    python tests/golden/make_golden.py
"""
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import pyoracle as po  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent
PHASES = np.array([1.0, 0.5, 0.2, 1e-9])


def mt_uniform(seed, n):
    """std::mt19937_64 with the oracles.hpp:21-23 bit recipe, in pure Python
    (independent of the product's input generator)."""
    mt = [0] * 312
    mt[0] = seed & 0xFFFFFFFFFFFFFFFF
    for i in range(1, 312):
        mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
    idx = 312
    out = []
    for _ in range(n):
        if idx >= 312:
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            idx = 0
        y = mt[idx]
        idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        out.append((y >> 11) * 2.0 ** -53)
    return np.array(out)


def density(nx, ny, seed):
    u = mt_uniform(seed, 3 * nx * ny).reshape(nx * ny, 3)
    a = np.zeros((nx * ny, 4))
    for e in range(nx * ny):
        r = u[e].copy()
        s = r[0] + r[1] + r[2]
        if s > 1.0:
            r = r / s
            s = r[0] + r[1] + r[2]
        a[e, :3] = r
        a[e, 3] = max(0.0, 1.0 - s)
    return a


def wall(nx, ny, load):
    fixed = []
    for x in range(nx + 1):
        node = x * (ny + 1)
        fixed += [2 * node, 2 * node + 1]
    if load == "point":
        loads = [(2 * ((nx // 2) * (ny + 1) + ny) + 1, -1.0)]
    else:
        loads = [(2 * (x * (ny + 1) + ny) + 1, -1.0 / (nx + 1)) for x in range(nx + 1)]
    return fixed, loads


CASES = [
    # name, nx, ny, coarsenings, seed, load, with x0
    ("wall8_l2", 8, 8, 2, 0, "uniform", False),
    ("wall16_l3_point", 16, 16, 3, 1, "point", False),
    ("wall32x16_l2", 32, 16, 2, 4, "uniform", True),
    ("wall24x40_l3", 24, 40, 3, 5, "uniform", False),
]


def main():
    if not po.available("ref"):
        raise SystemExit("oracle/_ref/libtopmg_ref.so missing: run `make -C oracle ref`")
    ke = {f"ke_nu{nu}": po.element_stiffness("ref", 1.0, nu) for nu in (0.3, 0.42)}
    oc = {}
    np.savez_compressed(OUT / "element_stiffness.npz", **ke)
    for name, nx, ny, nc, seed, load, with_x0 in CASES:
        alpha = density(nx, ny, seed)
        E = po.effective_moduli("ref", nx, ny, alpha, PHASES, 3.0)
        fixed, loads = wall(nx, ny, load)
        s = po.System("ref", nx, ny, E, 0.3, fixed, loads).build_mg(nc, 0.6)
        b = s.rhs()
        rng = np.random.default_rng(seed)
        x0 = rng.standard_normal(s.n) * 1e-2 if with_x0 else None
        r = s.solve(b, tol=1e-8, max_iter=500, gamma=1, pre=2, post=2, x0=x0)
        f = rng.standard_normal(s.n)
        v1 = s.vcycle(f, np.zeros(s.n), 1, 2, 2)
        v2 = s.vcycle(f, np.zeros(s.n), 2, 1, 1)
        d = dict(nx=nx, ny=ny, nc=nc, alpha=alpha, E=E, fixed=np.array(fixed, np.int32),
                 load_dofs=np.array([l[0] for l in loads], np.int32),
                 load_vals=np.array([l[1] for l in loads]), b=b, x=r["solution"],
                 iterations=r["iterations"], hist=r["residual_history"],
                 compliance=s.compliance(r["solution"]), f=f, vcycle_v22=v1, vcycle_w11=v2,
                 x0=x0 if x0 is not None else np.zeros(0))
        for lvl in range(nc + 1):
            off, col, val = s.csr(lvl)
            d[f"L{lvl}_off"], d[f"L{lvl}_col"], d[f"L{lvl}_val"] = off, col, val
        u = r["solution"]
        d["energies"] = po.element_energies("ref", nx, ny, u, 0.3)
        sens = po.sensitivities("ref", nx, ny, alpha, PHASES, 3.0, 0.3, u)
        d["sens"] = sens
        floored = np.maximum(alpha, 1e-3)
        for radius in (1.5, 3.0):
            d[f"filter_r{radius}"] = np.stack(
                [po.filter_sensitivities("ref", nx, ny, floored, ph, radius, sens[ph]) for ph in range(4)])
        d["alpha_floored"] = floored
        s.close()
        np.savez_compressed(OUT / f"{name}.npz", **d)
        print(name, "iterations", r["iterations"])
        oc_cases(name, floored, d["filter_r1.5"], seed, oc)
    np.savez_compressed(OUT / "oc_pair.npz", **oc)
    optim_cases()
    poisson_cases()


def full_depth(g):
    d = 0
    while g > 2:
        g //= 2
        d += 1
    return d


def poisson_cases():
    """assemble_poisson + pcgmg (fem.cpp:232-276, bench.cpp:30-111): the
    paper's Poisson bench setting (constant source 1, coarsest 2x2, omega 0.6,
    2+2 sweeps, tol 1e-6) and a seeded random source."""
    out = {}
    for tag, g, src in (("g16", 16, 1.0), ("g64", 64, 1.0), ("g32_rand", 32, None)):
        rng = np.random.default_rng(g)
        source = rng.standard_normal((g + 1) ** 2) if src is None else np.full((g + 1) ** 2, src)
        s = po.poisson_system("ref", g, g, source).build_mg(full_depth(g), 0.6)
        b = s.rhs()
        r = s.solve(b, tol=1e-6, max_iter=2000)
        f = rng.standard_normal(s.n)
        out[f"{tag}_source"], out[f"{tag}_b"] = source, b
        out[f"{tag}_x"], out[f"{tag}_hist"] = r["solution"], r["residual_history"]
        out[f"{tag}_iterations"] = np.array(r["iterations"])
        out[f"{tag}_f"], out[f"{tag}_vcycle"] = f, s.vcycle(f, np.zeros(s.n), 1, 2, 2)
        for lvl in range(full_depth(g) + 1):
            off, col, val = s.csr(lvl)
            out[f"{tag}_L{lvl}_off"], out[f"{tag}_L{lvl}_col"], out[f"{tag}_L{lvl}_val"] = off, col, val
        s.close()
    np.savez_compressed(OUT / "poisson.npz", **out)


def optim_cases():
    """optimize() with Method::pcgmg (mto.cpp:229-354) on two c0-style wall
    problems: BASELINE config-0 materials and fractions, uniform top load."""
    out = {}
    for tag, n, kw in (("n16", 16, dict(filter_radius=1.5, max_outer=8, num_coarsenings=1)),
                       ("n24_warm", 24, dict(filter_radius=3.0, max_outer=6, num_coarsenings=1, warm_start=True,
                                             inner_sweeps=2))):
        fixed, loads = wall(n, n, "uniform")
        r = po.optimize("ref", n, n, fixed, loads, PHASES, 3.0, 0.3, [0.15, 0.15, 0.15, 0.55], tol=1e-12, **kw)
        for k, v in r.items():
            out[f"{tag}_{k}"] = np.asarray(v)
        out[f"{tag}_args"] = np.array([n, kw["filter_radius"], kw["max_outer"], kw["num_coarsenings"],
                                       int(kw.get("warm_start", False)), kw.get("inner_sweeps", 1)])
    np.savez_compressed(OUT / "optimize.npz", **out)


def oc_cases(name, alpha, filt, seed, out):
    """oc_update_pair (mto.cpp:142-227) on the case's floored density and
    filtered sensitivities: the multiplicative branch for three phase pairs,
    the uniform-shift branch (no element prefers phase a) and an unreachable
    target (MultiplierError, status 8)."""
    rng = np.random.default_rng(100 + seed)
    ne = alpha.shape[0]
    move = rng.uniform(0.02, 0.2, ne)
    runs = [("mul01", 0, 1, filt[0], filt[1], +0.01), ("mul03", 0, 3, filt[0], filt[3], -0.02),
            ("mul23", 2, 3, filt[2], filt[3], +0.005),
            ("shift", 1, 2, filt[2] + np.abs(filt[1]) + 1e-3, filt[2], -0.01),
            ("unreach", 0, 1, filt[0], filt[1], +0.5)]
    for tag, pa, pb, sa, sb, dt in runs:
        target = float(alpha[:, pa].mean() + dt)
        new, st = po.oc_update_pair("ref", alpha, pa, pb, sa, sb, target, move, 0.5)
        k = f"{name}_{tag}"
        out[k + "_alpha"], out[k + "_sa"], out[k + "_sb"], out[k + "_move"] = alpha, sa, sb, move
        out[k + "_args"] = np.array([pa, pb, target, 0.5, 1e-3])
        out[k + "_out"], out[k + "_status"] = new, np.array(st)


if __name__ == "__main__":
    main()
