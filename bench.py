#!/usr/bin/env python3
"""Benchmark of the B200 pCGMG solve (BASELINE.json metric) -- one JSON line.

A step is one pass of the hot path over one synthetic input: the device setup
that replaces assemble_elasticity + build_multigrid_operators (Galerkin
hierarchy + coarsest inverse) followed by pcgmg_solve to tol 1e-8 -- exactly
what optimize() runs per outer iteration (mto.cpp:267-283).

  value : inputs (moduli, rhs) resident in HBM, timed with CUDA events on the
          library's stream; MDOF/s = DOFs x PCG iterations / step seconds.
  e2e   : the same metric through the C-ABI calls a user makes with HOST
          buffers: H2D of moduli and rhs and D2H of the solution inside the
          timed region, every step. Headline form: the pipelined calls
          (tmg_gpu_stage_inputs / tmg_gpu_solve_staged), whose copies run on
          a copy stream beside the neighbouring steps' solves; `e2e.serial`
          is the blocking tmg_gpu_set_moduli + tmg_gpu_solve pair.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4|c2|c1]
  python bench.py --impl reference ...   # the reference's own CPU path

Default workload: BASELINE configs[4] ("c4"), 8192x8192 Q4 (134.25M DOFs),
iid U(0,1) densities from seed 1, 11 levels, the largest single-GPU config
the metric is quoted on. Every vector is 1.07 GB, far above the 126 MB L2, so
no L2 flush is needed between steps.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import pathlib
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (nx, ny, coarsenings, recipe, seed, description)
    "c4": (8192, 8192, 10, "iid", 1,
           "c4: 8192x8192 Q4 wall, iid U(0,1) densities seed 1, 11 levels, tol 1e-8"),
    "c2": (2048, 2048, 8, "checker", 2,
           "c2: 2048x2048 Q4 wall, 16x16-element phase checkerboard seed 2 (1e9 contrast), 9 levels, tol 1e-8"),
    "c1": (512, 512, 6, "iid", 0,
           "c1: 512x512 Q4 wall, iid U(0,1) densities seed 0, 7 levels, tol 1e-8"),
    # the optimizer configs' meshes and hierarchies, one solve (latency-bound sizes)
    "c0": (64, 64, 3, "iid", 0,
           "c0 mesh: 64x64 Q4 wall, iid U(0,1) densities seed 0, 4 levels, tol 1e-8"),
    "c3": (1024, 1024, 7, "iid", 0,
           "c3 mesh: 1024x1024 Q4 wall, iid U(0,1) densities seed 0, 8 levels, tol 1e-8"),
    # weak scaling: a (1024 N) x 8192 wall on N GPUs, 11 levels
    "weak": (1024, 8192, 10, "iid", 1,
             "weak: (1024 N)x8192 Q4 wall on N GPUs, iid U(0,1) densities seed 1, 11 levels, tol 1e-8"),
}


def config_of(name, ws):
    """The CONFIGS entry, with the weak-scaling mesh widened to 1024 per GPU."""
    nx, ny, nc, recipe, seed, desc = CONFIGS[name]
    if name == "weak":
        nx *= ws
    return nx, ny, nc, recipe, seed, desc
TOL, OMEGA, SWEEPS, MAX_ITER = 1e-8, 0.6, 2, 5000
MATERIAL = dict(phase_moduli=[1.0, 0.5, 0.2, 1e-9], poisson_ratio=0.3, penalty=3.0)
METRIC = "pCGMG MDOF/s (DOFs x PCG iterations / s, per solve incl. device setup)"
# bounded CPU sample (same recipe as the workload, 512x512, one full solve)
CPU_SAMPLE = (512, 512, 6)
SAMPLE_WHY = ("the reference cannot run c4 itself: its CSR row offsets are int (sparse.hpp:53, sparse.cpp:44-45) "
              "and 8192^2 needs ~2.42e9 nonzeros > INT_MAX, plus >100 GB of assembly triplets; a 512^2 solve of "
              "the same recipe is ~5 s of single-threaded work, one per host core")


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_inputs(nx, ny, recipe, seed):
    import paper_2301_07457_b200 as P

    if recipe == "iid":
        alpha = P.density_iid(nx, ny, seed)
    else:
        alpha = P.density_checker(nx, ny, 16, seed)
    mat = P.MaterialModel(**MATERIAL)
    E = P.effective_moduli(alpha, mat)
    del alpha
    g = P.GridLevel(nx, ny)
    bc = P.wall_boundary_conditions(g, "uniform")
    b = P.assemble_rhs(g, bc)
    return g, bc, E, b


class Clocks:
    """nvidia-smi sampler for the timed region (clocks + throttle reasons)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        load = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel_key):
    """dram bytes per launch from the committed ncu --set full summary."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        return d.get(kernel_key)
    except Exception:
        return None


def run_reference_sample(nx, ny, nc, recipe, seed, kind):
    """One full reference solve (assemble + build_multigrid_operators +
    pcgmg_solve) on the host, 1 thread; returns (MDOF*it/s, iterations, s)."""
    from oracle import pyoracle as po  # CPU checker / reference -- bench CPU leg only

    # inputs through the reference side only (its oracle::Rng recipe and its
    # effective_moduli; nothing of the product library is loaded here)
    if recipe == "iid":
        alpha = po.density_iid(kind, nx, ny, seed)
    else:
        alpha = po.density_checker(kind, nx, ny, 16, seed)
    E = po.effective_moduli(kind, nx, ny, alpha, MATERIAL["phase_moduli"], MATERIAL["penalty"])
    fixed, loads = po.wall_uniform_bc(nx, ny)
    t0 = time.perf_counter()
    s = po.System(kind, nx, ny, E, MATERIAL["poisson_ratio"], fixed, loads)
    s.build_mg(nc, OMEGA)
    r = s.solve(s.rhs(), tol=TOL, max_iter=MAX_ITER, gamma=1, pre=SWEEPS, post=SWEEPS)
    dt = time.perf_counter() - t0
    s.close()
    dofs = 2 * (nx + 1) * (ny + 1)
    return dofs * r["iterations"] / dt / 1e6, r["iterations"], dt


def _ref_noop(sec):
    time.sleep(sec)  # keeps each task on its own worker while the pool starts
    return os.getpid()


def _ref_worker(job):
    """One reference sample in a worker process (bench CPU leg only)."""
    _, it, dt = run_reference_sample(*job)
    return it, dt


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


class ReferencePool:
    """The reference's pcgmg path is single-threaded, so the
    host's throughput is one independent sample per core, run concurrently in
    `cores` worker processes (they share the host's memory bandwidth, which the
    aggregate rate reflects)."""

    def __init__(self, cores):
        import concurrent.futures as cf
        import multiprocessing as mp

        self.cores = cores
        # spawn: the GPU arm forks nothing after CUDA and its threads are initialised
        self.ex = cf.ProcessPoolExecutor(max_workers=cores, mp_context=mp.get_context("spawn"))
        # start every worker (interpreter + imports) before anything is timed
        list(self.ex.map(_ref_noop, [0.2] * cores))

    def step(self, job):
        """All cores run one sample; returns (MDOF*it/s aggregate, iterations, wall s)."""
        t0 = time.perf_counter()
        res = list(self.ex.map(_ref_worker, [job] * self.cores))
        el = time.perf_counter() - t0
        its = sum(r[0] for r in res)
        dofs = 2 * (job[0] + 1) * (job[1] + 1)
        return dofs * its / el / 1e6, its, el

    def close(self):
        self.ex.shutdown()


def reference_arm(args, cfg_name):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import pyoracle as po

    kind = "ref" if po.available("ref") else "orc"
    nx, ny, nc, recipe, seed, desc = config_of(cfg_name, dist_env()[0])
    sx, sy, snc = CPU_SAMPLE
    job = (sx, sy, snc, recipe, seed, kind)
    pool = ReferencePool(host_cores())
    for _ in range(args.warmup):
        pool.step(job)
    t0 = time.perf_counter()
    its = []
    for _ in range(args.steps):
        _, it, _ = pool.step(job)
        its.append(it)
    el = time.perf_counter() - t0
    pool.close()
    dofs = 2 * (sx + 1) * (sy + 1)
    value = dofs * sum(its) / el / 1e6
    sample = (f"{sx}x{sy} mesh, same recipe ({recipe}, seed {seed}), {snc + 1} levels, tol {TOL}: per step, "
              f"{pool.cores} concurrent single-threaded samples (one per host core), each one full "
              f"assemble_from_moduli + build_multigrid_operators + pcgmg_solve "
              f"({'oracle/_ref = unmodified reference sources' if kind == 'ref' else 'oracle port'})")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "MDOF/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": desc, "sample": f"{sx}x{sy}", "samples_per_step": pool.cores,
                                         "pcg_iterations_per_step": its, "why_sample": SAMPLE_WHY,
                                         "inputs": "generated by oracle/_ref (the reference's oracle::Rng recipe "
                                                   "and effective_moduli); the product library is not loaded"},
        "cpu_baseline": {"value": value, "unit": "MDOF/s", "cores": pool.cores,
                         "kind": "reference" if kind == "ref" else "port", "sample": sample},
        "e2e": {"value": value, "unit": "MDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def gpu_arm(args, cfg_name):
    import paper_2301_07457_b200 as P

    ws, rank, local = dist_env()
    dist = None
    nccl = None
    if ws > 1:
        # control plane (barriers, max over ranks) on gloo; the solver's own
        # halo exchanges and PCG all-reduces run on an NCCL communicator
        import torch.distributed as td

        td.init_process_group("gloo")
        dist = td
        print(f"[bench] rank {rank}/{ws} (local {local}): control plane up, NCCL solver communicator next",
              file=sys.stderr, flush=True)
        uid = [P.nccl_unique_id() if rank == 0 else None]
        td.broadcast_object_list(uid, src=0)
        nccl = (ws, rank, uid[0])
    nx, ny, nc, recipe, seed, desc = config_of(cfg_name, dist_env()[0])
    g, bc, E, b = make_inputs(nx, ny, recipe, seed)
    dofs = g.dof_count()
    lib = P._lib.load()
    ops = P.MultigridOperators(g, nc, MATERIAL["poisson_ratio"], bc, device=local, nccl=nccl)

    # pinned host buffers for the e2e leg
    nE, nb = E.size, b.size
    pE = lib.tmg_host_alloc(8 * nE)
    pb = lib.tmg_host_alloc(8 * nb)
    px = lib.tmg_host_alloc(8 * nb)
    px2 = lib.tmg_host_alloc(8 * nb)
    hE = np.ctypeslib.as_array((C.c_double * nE).from_address(pE))
    hb = np.ctypeslib.as_array((C.c_double * nb).from_address(pb))
    hx = np.ctypeslib.as_array((C.c_double * nb).from_address(px))
    hx2 = np.ctypeslib.as_array((C.c_double * nb).from_address(px2))
    hE[:] = E
    hb[:] = b
    del E

    D = P._lib.dptr
    itc, fr, cv, sec, hl = C.c_int(), C.c_double(), C.c_int(), C.c_double(), C.c_int()
    hist = np.empty(MAX_ITER + 1)

    def resident_step():
        ops._check(lib.tmg_gpu_setup(ops.h, OMEGA))
        ops._check(lib.tmg_gpu_solve_resident(ops.h, 0, TOL, MAX_ITER, 1, SWEEPS, SWEEPS, C.byref(itc), C.byref(fr),
                                              C.byref(cv), C.byref(sec), D(hist), hist.size, C.byref(hl)))
        if not cv.value:
            raise RuntimeError("solve did not converge")
        return itc.value

    def e2e_step():
        ops._check(lib.tmg_gpu_set_moduli(ops.h, D(hE), nE, OMEGA))
        ops._check(lib.tmg_gpu_solve(ops.h, D(hb), None, TOL, MAX_ITER, 1, SWEEPS, SWEEPS, D(hx), C.byref(itc),
                                     C.byref(fr), C.byref(cv), C.byref(sec), D(hist), hist.size, C.byref(hl)))
        return itc.value

    def e2e_pipelined(n):
        # the serving form of the same C-ABI path: step k+1's inputs are
        # staged (H2D on the library's copy stream) while step k solves, and
        # step k's solution is downloaded while step k+1 solves
        # (tmg_gpu_stage_inputs / tmg_gpu_solve_staged, include/tmg_gpu.h)
        outs = (hx, hx2)
        its_ = []
        ops._check(lib.tmg_gpu_stage_inputs(ops.h, 0, D(hE), nE, D(hb)))
        for k in range(n):
            if k + 1 < n:
                ops._check(lib.tmg_gpu_stage_inputs(ops.h, (k + 1) & 1, D(hE), nE, D(hb)))
            ops._check(lib.tmg_gpu_solve_staged(ops.h, k & 1, OMEGA, TOL, MAX_ITER, 1, SWEEPS, SWEEPS, D(outs[k & 1]),
                                                C.byref(itc), C.byref(fr), C.byref(cv), C.byref(sec), D(hist),
                                                hist.size, C.byref(hl)))
            its_.append(itc.value)
        ops._check(lib.tmg_gpu_sync_outputs(ops.h))
        return its_

    def barrier():
        if dist:
            dist.barrier()

    def max_over_ranks(v):
        if not dist:
            return v
        import torch

        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up (also uploads the resident inputs)
    ops.upload_moduli(hE)
    ops._check(lib.tmg_gpu_upload_rhs(ops.h, D(hb)))
    for _ in range(max(args.warmup, 3)):
        resident_step()
    e2e_step()
    e2e_pipelined(2)

    # ---- value: inputs resident in HBM
    clocks = Clocks(local)
    clocks.start()
    barrier()
    ops._check(lib.tmg_gpu_event_record(ops.h, 0))
    l0 = ops.launch_count()
    its = [resident_step() for _ in range(args.steps)]
    ops._check(lib.tmg_gpu_event_record(ops.h, 1))
    ms = C.c_double()
    ops._check(lib.tmg_gpu_event_elapsed(ops.h, 0, 1, C.byref(ms)))
    launches = ops.launch_count() - l0
    barrier()
    clk = clocks.stop()
    t_res = max_over_ranks(ms.value)
    setup_ms, pcg_ms = ops.last_timings()

    # ---- e2e: host buffers through the C ABI, pipelined (the headline) and
    # one blocking solve at a time
    barrier()
    ops._check(lib.tmg_gpu_event_record(ops.h, 2))
    e_its = e2e_pipelined(args.steps)
    ops._check(lib.tmg_gpu_event_record(ops.h, 3))
    ops._check(lib.tmg_gpu_event_elapsed(ops.h, 2, 3, C.byref(ms)))
    barrier()
    t_e2e = max_over_ranks(ms.value)
    barrier()
    ops._check(lib.tmg_gpu_event_record(ops.h, 2))
    s_its = [e2e_step() for _ in range(args.steps)]
    ops._check(lib.tmg_gpu_event_record(ops.h, 3))
    ops._check(lib.tmg_gpu_event_elapsed(ops.h, 2, 3, C.byref(ms)))
    barrier()
    t_ser = max_over_ranks(ms.value)

    # ---- dominant-kernel roofline, live CUDA events on the library's stream:
    # the fused PCG update + two pre-sweeps (the largest share of a PCG
    # iteration), with the plain K.u apply and one sweep beside it
    dom_ms, dom_bytes = ops.time_kernel(2, 20)
    ku_ms, ku_bytes = ops.time_kernel(0, 20)
    sw_ms, sw_bytes = ops.time_kernel(1, 20)
    peak, peak_src = hbm_peak()
    gbs = lambda b, t: b / (t * 1e-3) / 1e9  # noqa: E731
    dom_gbs, ku_gbs, sw_gbs = gbs(dom_bytes, dom_ms), gbs(ku_bytes, ku_ms), gbs(sw_bytes, sw_ms)

    result = None
    if rank == 0:
        # strong scaling: the same global solve at every N (weak: 1024 columns per GPU)
        value = dofs * sum(its) / (t_res * 1e-3) / 1e6
        e2e_value = dofs * sum(e_its) / (t_e2e * 1e-3) / 1e6
        ser_value = dofs * sum(s_its) / (t_ser * 1e-3) / 1e6
        result = {
            "metric": METRIC, "value": value, "unit": "MDOF/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_res / args.steps, "higher_is_better": True,
            "scaling": "weak" if cfg_name == "weak" else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded densities with the BASELINE recipe; no dataset exists)",
            "config": {"workload": desc, "nx": nx, "ny": ny, "dofs": dofs, "levels": nc + 1, "tol": TOL,
                       "omega": OMEGA, "smoother": f"damped Jacobi {SWEEPS}+{SWEEPS}", "cycle": "V",
                       "pcg_iterations": its,
                       "parallelism": "single GPU" if ws == 1 else f"x-slab decomposition over {ws} GPUs (NCCL)",
                       "l2": "inputs larger than L2 (1.07 GB per fine vector); no flush needed"
                       if cfg_name in ("c4", "weak") else "working set partly L2-resident; no flush",
                       "solves_per_s": args.steps / (t_res * 1e-3),
                       "setup_ms_last": setup_ms, "pcg_ms_last": pcg_ms,
                       "pcg_only_mdof_s": dofs * its[-1] / (pcg_ms * 1e-3) / 1e6},
            "e2e": {"value": e2e_value, "unit": "MDOF/s", "h2d_bytes_per_step": 8 * nE + 8 * nb,
                    "d2h_bytes_per_step": 8 * nb, "ms_per_step": t_e2e / args.steps,
                    "mode": "pipelined: each step copies its moduli and rhs from pinned host memory to the device "
                            "and its solution back, on the library's copy stream, overlapping the neighbouring "
                            "steps' solves (tmg_gpu_stage_inputs / tmg_gpu_solve_staged / tmg_gpu_sync_outputs); "
                            "the timed region runs from before the first upload to after the last download",
                    "pcg_iterations": e_its,
                    "serial": {"value": ser_value, "ms_per_step": t_ser / args.steps, "pcg_iterations": s_its,
                               "mode": "one blocking tmg_gpu_set_moduli + tmg_gpu_solve per step"}},
            "gpu_launches": launches,
            "clocks": clk,
            "roofline": {"bound": "hbm",
                         "kernel": "k_march<StSweep01U> (PCG x/r update + two damped-Jacobi sweeps from zero, "
                                   "121 B/node)",
                         "achieved": dom_gbs, "peak": peak, "unit": "GB/s", "frac": dom_gbs / peak,
                         "peak_source": peak_src, "traffic": ncu_traffic("k_march<StSweep01T<1>, 1>"),
                         "bytes_per_launch": dom_bytes, "avg_launch_ms": dom_ms,
                         "share_of_pcg_iteration": dom_ms / (pcg_ms / its[-1]),
                         "others": [
                             {"kernel": "k_march<StApply> (K.u, 41 B/node)", "achieved": ku_gbs,
                              "frac": ku_gbs / peak, "bytes_per_launch": ku_bytes, "avg_launch_ms": ku_ms},
                             {"kernel": "k_march<StSweep> (one sweep, 57 B/node)", "achieved": sw_gbs,
                              "frac": sw_gbs / peak, "bytes_per_launch": sw_bytes, "avg_launch_ms": sw_ms}]},
        }
        if not args.no_cpu_baseline and ws == 1:
            from oracle import pyoracle as po

            kind = "ref" if po.available("ref") else "orc"
            sx, sy, snc = CPU_SAMPLE
            pool = ReferencePool(host_cores())
            rate, it, dt = pool.step((sx, sy, snc, recipe, seed, kind))
            pool.close()
            result["cpu_baseline"] = {
                "value": rate, "unit": "MDOF/s", "cores": pool.cores, "kind": "reference" if kind == "ref" else "port",
                "sample": f"{sx}x{sy} mesh, {recipe} seed {seed}, {snc + 1} levels: {pool.cores} concurrent "
                          f"single-threaded samples (the reference has no threading; one per host core), each "
                          f"one full assemble + build_multigrid_operators + pcgmg_solve ({it} PCG iterations in "
                          f"total, {dt:.1f} s wall); {SAMPLE_WHY}"}
    lib.tmg_host_free(C.c_void_p(pE))
    lib.tmg_host_free(C.c_void_p(pb))
    lib.tmg_host_free(C.c_void_p(px))
    ops.close()
    if dist:
        dist.destroy_process_group()
    if result:
        print(json.dumps(result), flush=True)
    return 0


def free_port():
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def launch_ranks(n):
    """--gpus N without a torchrun environment: start N ranks (one process per
    GPU) through torch.distributed.run on 127.0.0.1 and return its exit code;
    rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", str(pathlib.Path(__file__).resolve()),
           *sys.argv[1:]]
    print(f"[bench] launching {n} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def arm_watchdog():
    """A rank that has not finished after TMG_BENCH_WATCHDOG_S seconds (default
    1800) exits with code 124 and a message instead of waiting forever on a
    peer: multi-rank NCCL runs of the solver have not been exercised on a
    multi-GPU box yet (every gpurun box has one GPU), so a hang there ends the
    rank rather than the driver's whole time slot."""
    limit = float(os.environ.get("TMG_BENCH_WATCHDOG_S", "1800"))

    def fire():
        print(f"[bench] rank {dist_env()[1]}: no result after {limit:.0f} s, exiting (watchdog)", file=sys.stderr,
              flush=True)
        os._exit(124)

    t = threading.Timer(limit, fire)
    t.daemon = True
    t.start()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return launch_ranks(args.gpus)
    ws = dist_env()[0]
    if ws > 1:
        arm_watchdog()
    if ws != args.gpus:
        print(f"[bench] --gpus {args.gpus} but WORLD_SIZE={ws}: running {ws} ranks", file=sys.stderr, flush=True)
    if args.impl == "reference":
        return reference_arm(args, args.config)
    return gpu_arm(args, args.config)


if __name__ == "__main__":
    sys.exit(main())
