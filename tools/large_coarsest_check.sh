# Large coarsest levels (n > 2048 dofs: k_cholesky_band_g, k_lower_inverse_band,
# k_gram_tiled): the GPU parity tests and setup / solve times (under gpurun).
mkdir -p gpurun_out/lc
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "large_coarsest or banded_coarsest" > gpurun_out/lc/test.log 2>&1; echo rc=$?
tail -3 gpurun_out/lc/test.log
timeout 600 python - <<'PY' 2>&1 | tee gpurun_out/lc/times.txt | tail -20
import sys, time, numpy as np
sys.path.insert(0, "tests")
import paper_2301_07457_b200 as P
from helpers import moduli
for nx, ny, nc in [(128,128,2),(256,256,2),(512,256,2)]:
    _, E = moduli(nx, ny, "iid", 5)
    g = P.GridLevel(nx, ny); bc = P.wall_boundary_conditions(g, "uniform"); b = P.assemble_rhs(g, bc)
    ops = P.MultigridOperators(g, nc, 0.3, bc)
    ops.set_moduli(E, 0.6)
    t0 = time.time(); ops.set_moduli(E, 0.6); t1 = time.time()
    rep = P.pcgmg_solve(ops, b, P.SolverConfig(tol=1e-8, max_iter=2000, num_coarsenings=nc)); t2 = time.time()
    print(nx, ny, nc, "coarsest dofs", 2*(nx//2**nc+1)*(ny//2**nc+1), "setup s", round(t1-t0,4), "solve s", round(t2-t1,4), "its", rep.iterations, ops.last_timings())
PY
