"""H2D / D2H rates of the e2e leg's copies on the box (c4 sizes): the pitched
copies the C ABI makes vs plain contiguous pinned copies of the same bytes.

  python tools/copy_rates.py"""
import ctypes as C
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_07457_b200 as P  # noqa: E402

n = 8192
g = P.GridLevel(n, n)
bc = P.wall_boundary_conditions(g, "uniform")
ops = P.MultigridOperators(g, 10, 0.3, bc)
lib = P._lib.load()
nE, nb = n * n, 2 * (n + 1) * (n + 1)
pE, pb = lib.tmg_host_alloc(8 * nE), lib.tmg_host_alloc(8 * nb)
hE = np.ctypeslib.as_array((C.c_double * nE).from_address(pE))
hb = np.ctypeslib.as_array((C.c_double * nb).from_address(pb))
hE[:] = 1.0
hb[:] = 0.0
D = P._lib.dptr


def t(fn, bytes_, name, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    m = min(ts)
    print(f"{name:40s} {bytes_ / 1e9:6.3f} GB  {m * 1e3:7.2f} ms  {bytes_ / m / 1e9:6.1f} GB/s", flush=True)


t(lambda: ops._check(lib.tmg_gpu_upload_moduli(ops.h, D(hE), nE)), 8 * nE, "E upload (pitched 2D, C ABI)")
t(lambda: ops._check(lib.tmg_gpu_upload_rhs(ops.h, D(hb))), 8 * nb, "b upload (pitched 2D, C ABI)")
hp = torch.empty(nb, dtype=torch.float64, pin_memory=True)
dv = torch.empty(nb, dtype=torch.float64, device="cuda")
t(lambda: dv.copy_(hp, non_blocking=True), 8 * nb, "contiguous pinned H2D (torch)")
t(lambda: hp.copy_(dv, non_blocking=True), 8 * nb, "contiguous pinned D2H (torch)")
