"""Measure the device OC exchange (tmg_gpu_oc_update_pair, SURVEY.md 8(f)
item 1) at a BASELINE mesh size, beside the unmodified reference on the host.

  python tools/bench_oc.py [--nx 8192] [--ny 8192] [--reps 3]

Inputs: the c4-recipe density (mt19937_64 iid, seed 1, floored at 1e-3 and
renormalised) and seeded synthetic filtered sensitivities with the sign and
scale of real ones (-U(0, 2) per phase); per-element move limits U(0.02,
0.2); phases (0, 3), target = current phase-0 fraction + 0.01, damping 0.5.
Prints one JSON line: element-steps/s on the device (bisection steps x
elements / device time), the e2e time through the C ABI with host arrays,
the roofline of the bisection (32 B per element and step: a, gain, lo, hi)
and the reference's rate on a 512^2 sample (1 host thread)."""
import argparse
import json
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def inputs(nx, ny, seed):
    import paper_2301_07457_b200 as P

    a = np.maximum(P.density_iid(nx, ny, seed), 1e-3)
    a /= a.sum(1, keepdims=True)
    rng = np.random.default_rng(seed)
    ne = nx * ny
    sa, sb = -rng.uniform(0, 2, ne), -rng.uniform(0, 2, ne)
    move = rng.uniform(0.02, 0.2, ne)
    return np.ascontiguousarray(a), sa, sb, move


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=8192)
    ap.add_argument("--ny", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import paper_2301_07457_b200 as P

    nx, ny = args.nx, args.ny
    a, sa, sb, move = inputs(nx, ny, 1)
    target = float(a[:, 0].mean() + 0.01)
    g = P.GridLevel(nx, ny)
    nc = int(np.log2(min(nx, ny) // 8))  # a valid hierarchy for the handle
    ops = P.MultigridOperators(g, nc, 0.3, P.wall_boundary_conditions(g, "uniform"))
    runs = []
    for _ in range(args.reps + 1):  # first run warms up
        work = a.copy()
        t0 = time.perf_counter()
        P.oc_update_pair(ops, work, 0, 3, sa, sb, target, move, 0.5)
        t1 = time.perf_counter()
        ms, steps = P.oc_timings(ops)
        runs.append((ms, steps, (t1 - t0) * 1e3))
    runs = runs[1:]
    ms = float(np.median([r[0] for r in runs]))
    steps = runs[0][1]
    e2e_ms = float(np.median([r[2] for r in runs]))
    ne = nx * ny
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() \
        else 6650.0
    # prep reads 2 density phases + sa, sb, move (40 B) and writes a, gain, lo,
    # hi (32 B); each step reads 32 B; the final pass reads 40 and writes 16
    algo = ne * (72 + 32 * steps + 56)
    out = {"metric": "OC exchange element-steps/s (elements x bisection steps / device s)",
           "value": ne * steps / (ms * 1e-3), "unit": "element-steps/s", "elements": ne, "phases": 4,
           "bisection_steps": steps, "device_ms": ms, "e2e_ms": e2e_ms,
           "e2e_note": "host arrays through tmg_gpu_oc_update_pair: density up and down, sens a/b and move up",
           "roofline": {"bound": "hbm", "achieved": algo / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                        "frac": algo / (ms * 1e-3) / 1e9 / peak,
                        "algorithmic_bytes": algo},
           "data": "synthetic (c4-recipe density; seeded sensitivities -U(0,2), move U(0.02,0.2))"}
    from oracle import pyoracle as po  # reference leg only

    kind = "ref" if po.available("ref") else "orc"
    sx = 512
    a2, sa2, sb2, mv2 = inputs(sx, sx, 1)
    t2 = float(a2[:, 0].mean() + 0.01)
    t0 = time.perf_counter()
    _, st = po.oc_update_pair(kind, a2, 0, 3, sa2, sb2, t2, mv2, 0.5)
    dt = time.perf_counter() - t0
    # the device run on the same sample takes the same bisection branches;
    # its step count puts the reference in the same unit
    work = a2.copy()
    g2 = P.GridLevel(sx, sx)
    ops2 = P.MultigridOperators(g2, int(np.log2(sx // 8)), 0.3, P.wall_boundary_conditions(g2, "uniform"))
    P.oc_update_pair(ops2, work, 0, 3, sa2, sb2, t2, mv2, 0.5)
    steps2 = P.oc_timings(ops2)[1]
    out["cpu_baseline"] = {"value": sx * sx * steps2 / dt, "unit": "element-steps/s",
                           "kind": "reference" if kind == "ref" else "port", "cores": 1,
                           "sample": f"{sx}x{sx} elements, same recipe, one oc_update_pair "
                                     f"({steps2} bisection steps, status {st}, {dt:.2f} s)"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
