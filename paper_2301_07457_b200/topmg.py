"""Python mirror of the reference topopt-mg interface for the pCGMG hot path.

Names, argument meaning and error types follow the reference so that code and
tests written against it read the same (citations: /root/reference/proj):

  GridLevel, BoundaryConditions       grid.hpp:10-24, fem.hpp:14-19
  SolverConfig, SolveReport           solvers.hpp:17-37
  element_stiffness                   fem.cpp:131-169
  effective_moduli                    density.cpp:78-85
  wall_boundary_conditions            fem.cpp:320-336
  build_multigrid_operators           solvers.cpp:460-481  (GPU: matrix-free)
  pcgmg_solve                         solvers.cpp:516-530
  mg_cycle                            solvers.cpp:483-514
  compliance / element_energies       fem.cpp:284-318
  sensitivities / filter_sensitivities mto.cpp:61-117
  ConfigError ... MultiplierError     errors.hpp:9-47

Everything that computes runs in libtmg_gpu.so on an sm_100 GPU; this module
only marshals arrays. There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import dptr, iptr


# ----------------------------------------------------------------- errors --
class TopmgError(RuntimeError):
    pass


class ConfigError(TopmgError):
    pass


class DimensionError(TopmgError):
    pass


class NumericError(TopmgError):
    pass


class DefinitenessError(NumericError):
    def __init__(self, what: str, row: int = -1):
        super().__init__(what)
        self.row = row


class SplittingError(NumericError):
    pass


class PreconditionerError(NumericError):
    pass


class MultiplierError(NumericError):
    pass


class CudaError(TopmgError):
    pass


def _raise(code: int, msg: str, row: int = -1):
    if code == 1:
        raise ConfigError(msg)
    if code == 2:
        raise DimensionError(msg)
    if code == 3:
        raise DefinitenessError(msg, row)
    if code == 4:
        raise PreconditionerError(msg)
    if code == 5:
        raise SplittingError(msg)
    if code == 8:
        raise MultiplierError(msg)
    raise CudaError(msg or f"tmg_gpu status {code}")


# ------------------------------------------------------------------ types --
@dataclass
class GridLevel:
    nx: int = 0
    ny: int = 0
    dofs_per_node: int = 2
    level_index: int = 0

    def node_count(self) -> int:
        return (self.nx + 1) * (self.ny + 1)

    def dof_count(self) -> int:
        return self.dofs_per_node * self.node_count()

    def element_count(self) -> int:
        return self.nx * self.ny

    def node_index(self, x: int, y: int) -> int:
        return x * (self.ny + 1) + y

    def dof_index(self, x: int, y: int, c: int) -> int:
        return self.node_index(x, y) * self.dofs_per_node + c

    def element_index(self, ex: int, ey: int) -> int:
        return ex * self.ny + ey


@dataclass
class BoundaryConditions:
    fixed_dofs: list = field(default_factory=list)
    point_loads: list = field(default_factory=list)  # (dof, value)


@dataclass
class SolverConfig:
    method: str = "pcgmg"
    tol: float = 1e-6
    max_iter: int = 1000
    omega: float = 0.6
    gamma: int = 1
    pre_sweeps: int = 2
    post_sweeps: int = 2
    num_coarsenings: int = 2

    def validate(self):
        """SolverConfig::validate (solvers.cpp:72-88)."""
        if not self.tol > 0.0:
            raise ConfigError("solver tol must be positive")
        if self.max_iter < 1:
            raise ConfigError("max_iter must be >= 1")
        if not (0.0 < self.omega <= 1.0):
            raise ConfigError(f"omega must lie in (0, 1], got {self.omega:f}")
        if self.gamma not in (1, 2):
            raise ConfigError("gamma must be 1 (V-cycle) or 2 (W-cycle)")
        if self.pre_sweeps < 0 or self.post_sweeps < 0:
            raise ConfigError("smoothing sweep counts must be non-negative")
        if self.num_coarsenings < 0:
            raise ConfigError("num_coarsenings must be non-negative")
        if self.method == "pcgmg" and self.pre_sweeps != self.post_sweeps:
            raise ConfigError("pcgmg needs pre_sweeps == post_sweeps for a symmetric preconditioner")


@dataclass
class SolveReport:
    solution: np.ndarray = None
    iterations: int = 0
    final_residual: float = 0.0
    converged: bool = False
    seconds: float = 0.0
    residual_history: list = field(default_factory=list)


@dataclass
class MaterialModel:
    phase_moduli: list = field(default_factory=lambda: [1.0, 0.5, 0.2, 1e-9])
    poisson_ratio: float = 0.3
    penalty: float = 3.0

    def num_phases(self) -> int:
        return len(self.phase_moduli)


# --------------------------------------------------------- host producers --
def element_stiffness(modulus: float, poisson_ratio: float) -> np.ndarray:
    """8x8 Q4 plane-stress Ke (fem.cpp:131-169), row-major."""
    k = np.zeros(64)
    _lib.load().tmg_element_stiffness(modulus, poisson_ratio, dptr(k))
    return k.reshape(8, 8)


def effective_moduli(alpha: np.ndarray, material: MaterialModel) -> np.ndarray:
    """E_e = sum_i alpha_i^p E_i (density.cpp:68-85); alpha is [ne, nphases]."""
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    ne, npn = a.shape
    pm = np.ascontiguousarray(material.phase_moduli, dtype=np.float64)
    out = np.empty(ne)
    _lib.load().tmg_inputs_effective_moduli(ne, npn, dptr(a), dptr(pm), material.penalty, dptr(out))
    return out


def density_iid(nx: int, ny: int, seed: int, nmat: int = 3) -> np.ndarray:
    a = np.empty((nx * ny, nmat + 1))
    _lib.load().tmg_inputs_density_iid(nx, ny, nmat, seed, dptr(a))
    return a


def density_checker(nx: int, ny: int, block: int, seed: int, nphases: int = 4) -> np.ndarray:
    a = np.empty((nx * ny, nphases))
    _lib.load().tmg_inputs_density_checker(nx, ny, block, nphases, seed, dptr(a))
    return a


def wall_boundary_conditions(grid: GridLevel, load: str = "point") -> BoundaryConditions:
    """Bottom edge clamped (fem.cpp:320-336). load='point' is the reference's
    unit load at the top-mid node; load='uniform' is BASELINE's unit total
    load spread as -1/(nx+1) over every top node."""
    if load == "point" and grid.nx % 2:
        raise ConfigError("wall load sits on the top-edge midpoint; nx must be even")
    nx, ny = grid.nx, grid.ny
    fixed = np.empty(2 * (nx + 1), np.int32)
    nf = C.c_int()
    ld = np.empty(nx + 1, np.int32)
    lv = np.empty(nx + 1)
    nl = C.c_int()
    _lib.load().tmg_inputs_wall_bc(nx, ny, 0 if load == "point" else 1, iptr(fixed), C.byref(nf),
                                   iptr(ld), dptr(lv), C.byref(nl))
    return BoundaryConditions(fixed_dofs=fixed[: nf.value].tolist(),
                              point_loads=list(zip(ld[: nl.value].tolist(), lv[: nl.value].tolist())))


def validate_boundary_conditions(bc: BoundaryConditions, dof_count: int) -> None:
    """BoundaryConditions::validate (fem.cpp:110-129), message for message."""
    is_fixed = np.zeros(dof_count, dtype=bool)
    for d in bc.fixed_dofs:
        if d < 0 or d >= dof_count:
            raise ConfigError(f"fixed dof {d} outside [0, {dof_count})")
        is_fixed[d] = True
    for d, _ in bc.point_loads:
        if d < 0 or d >= dof_count:
            raise ConfigError(f"loaded dof {d} outside [0, {dof_count})")
        if is_fixed[d]:
            raise ConfigError(f"dof {d} is both fixed and loaded")


def assemble_rhs(grid: GridLevel, bc: BoundaryConditions) -> np.ndarray:
    """rhs of assemble_from_moduli: loads summed, fixed entries zeroed
    (fem.cpp:214-218), after BoundaryConditions::validate."""
    validate_boundary_conditions(bc, grid.dof_count())
    fixed = np.ascontiguousarray(bc.fixed_dofs, dtype=np.int32)
    ld = np.ascontiguousarray([d for d, _ in bc.point_loads], dtype=np.int32)
    lv = np.ascontiguousarray([v for _, v in bc.point_loads], dtype=np.float64)
    b = np.empty(grid.dof_count())
    st = _lib.load().tmg_inputs_rhs(grid.nx, grid.ny, iptr(fixed), len(fixed), iptr(ld), dptr(lv), len(lv),
                                    dptr(b))
    if st != 0:
        raise ConfigError("invalid boundary conditions")
    return b


def _check_dofs(what: str, v: np.ndarray | None, n: int, fmt: str):
    if v is not None and v.size != n:
        raise DimensionError(fmt.format(what=what, got=v.size, n=n))


def _check_density(alpha: np.ndarray, grid: GridLevel, nphases: int | None, what: str):
    if alpha.ndim != 2 or alpha.shape[0] != grid.element_count():
        raise DimensionError(f"{what}: density grid does not match level")
    if nphases is not None and alpha.shape[1] != nphases:
        raise DimensionError(f"{what}: phase count mismatch")


# ------------------------------------------------------------- GPU solver --
class MultigridOperators:
    """GPU-resident counterpart of MultigridOperators (solvers.hpp:93-102).

    Holds the matrix-free fine operator (moduli, Ke, Dirichlet mask), the
    device Galerkin hierarchy and the coarsest inverse; rebuilt by
    ``set_moduli`` each outer iteration while the mesh stays resident.
    """

    def __init__(self, grid: GridLevel, num_coarsenings: int, poisson_ratio: float,
                 bc: BoundaryConditions, device: int = 0, slabs: int = 1, replicated_level: int = -1,
                 nccl: tuple | None = None):
        """slabs > 1: the x-slab decomposition driven from this process on one
        device; nccl=(nranks, rank, unique_id_bytes): one rank of a
        multi-process (torchrun) solve."""
        self.lib = _lib.load()
        self.grid = grid
        self.num_coarsenings = num_coarsenings
        self.omega = 0.6
        h = C.c_void_p()
        if nccl is not None:
            nranks, rank, uid = nccl
            buf = C.create_string_buffer(bytes(uid), 128)
            st = self.lib.tmg_gpu_create_nccl(grid.nx, grid.ny, num_coarsenings, grid.dofs_per_node, device,
                                              nranks, rank, buf, replicated_level, C.byref(h))
        elif slabs > 1:
            st = self.lib.tmg_gpu_create_local_slabs(grid.nx, grid.ny, num_coarsenings, grid.dofs_per_node,
                                                     device, slabs, replicated_level, C.byref(h))
        else:
            st = self.lib.tmg_gpu_create(grid.nx, grid.ny, num_coarsenings, grid.dofs_per_node, device,
                                         C.byref(h))
        self.h = h
        if st != 0:
            msg, row = self._err()
            self.close()
            _raise(st, msg, row)
        fixed = np.ascontiguousarray(bc.fixed_dofs, dtype=np.int32)
        self._check(self.lib.tmg_gpu_set_problem(self.h, poisson_ratio, iptr(fixed), len(fixed)))

    # ---- plumbing
    def _err(self):
        buf = C.create_string_buffer(512)
        row = C.c_int(-1)
        if self.h:
            self.lib.tmg_gpu_last_error(self.h, buf, 512, C.byref(row))
        return buf.value.decode(errors="replace"), row.value

    def _check(self, st: int):
        if st != 0:
            msg, row = self._err()
            _raise(st, msg, row)

    def close(self):
        if getattr(self, "h", None):
            self.lib.tmg_gpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return self.lib.tmg_gpu_stream(self.h) or 0

    def launch_count(self) -> int:
        return self.lib.tmg_gpu_launch_count(self.h)

    def level(self, index: int) -> GridLevel:
        s = 1 << (self.num_coarsenings - index)
        return GridLevel(self.grid.nx // s, self.grid.ny // s, 2, index)

    # ---- setup (assemble_elasticity + build_multigrid_operators)
    def set_moduli(self, moduli: np.ndarray, omega: float = 0.6):
        e = np.ascontiguousarray(moduli, dtype=np.float64)
        self.omega = omega
        self._check(self.lib.tmg_gpu_set_moduli(self.h, dptr(e), e.size, omega))

    def upload_moduli(self, moduli: np.ndarray):
        e = np.ascontiguousarray(moduli, dtype=np.float64)
        self._check(self.lib.tmg_gpu_upload_moduli(self.h, dptr(e), e.size))

    def setup(self, omega: float = 0.6):
        self.omega = omega
        self._check(self.lib.tmg_gpu_setup(self.h, omega))

    def set_density(self, alpha: np.ndarray, material: MaterialModel, omega: float = 0.6):
        a = np.ascontiguousarray(alpha, dtype=np.float64)
        pm = np.ascontiguousarray(material.phase_moduli, dtype=np.float64)
        self.omega = omega
        self._check(self.lib.tmg_gpu_set_density(self.h, dptr(a), a.shape[1], dptr(pm), material.penalty, omega))

    # ---- kernel-level entry points
    def apply(self, level: int, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x)
        self._check(self.lib.tmg_gpu_apply(self.h, level, dptr(x), dptr(y)))
        return y

    def level_values(self, level: int, offsets: np.ndarray, cols: np.ndarray) -> np.ndarray:
        off = np.ascontiguousarray(offsets, dtype=np.int32)
        col = np.ascontiguousarray(cols, dtype=np.int32)
        vals = np.empty(len(col))
        self._check(self.lib.tmg_gpu_level_values(self.h, level, iptr(off), iptr(col), dptr(vals)))
        return vals

    def prolongate(self, level: int, coarse: np.ndarray) -> np.ndarray:
        c = np.ascontiguousarray(coarse, dtype=np.float64)
        out = np.empty(self.level(level).dof_count())
        self._check(self.lib.tmg_gpu_prolongate(self.h, level, dptr(c), dptr(out)))
        return out

    def restrict(self, level: int, fine: np.ndarray) -> np.ndarray:
        f = np.ascontiguousarray(fine, dtype=np.float64)
        out = np.empty(self.level(level - 1).dof_count())
        self._check(self.lib.tmg_gpu_restrict(self.h, level, dptr(f), dptr(out)))
        return out

    def smooth(self, level: int, f: np.ndarray, u: np.ndarray, sweeps: int) -> np.ndarray:
        f = np.ascontiguousarray(f, dtype=np.float64)
        u = np.array(u, dtype=np.float64, copy=True)
        self._check(self.lib.tmg_gpu_smooth(self.h, level, dptr(f), dptr(u), sweeps))
        return u

    def time_kernel(self, which: int, reps: int):
        ms = C.c_double()
        by = C.c_double()
        self._check(self.lib.tmg_gpu_time_kernel(self.h, which, reps, C.byref(ms), C.byref(by)))
        return ms.value, by.value

    def last_timings(self):
        s = C.c_double()
        p = C.c_double()
        self.lib.tmg_gpu_last_timings(self.h, C.byref(s), C.byref(p))
        return s.value, p.value


def slab_partition(nx: int, ny: int, num_coarsenings: int, nranks: int, replicated_level: int = -1):
    """(first fine node column of every rank + [nx+1], replicated level)."""
    x0s = np.zeros(nranks + 1, np.int32)
    rep = C.c_int()
    st = _lib.load().tmg_partition(nx, ny, num_coarsenings, nranks, replicated_level, iptr(x0s), C.byref(rep))
    if st != 0:
        _raise(st, "tmg_partition failed")
    return x0s.tolist(), rep.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = _lib.load().tmg_nccl_unique_id(buf)
    if st != 0:
        _raise(st, "ncclGetUniqueId failed")
    return buf.raw


def build_multigrid_operators(grid: GridLevel, moduli: np.ndarray, poisson_ratio: float,
                              bc: BoundaryConditions, num_coarsenings: int, omega: float = 0.6,
                              device: int = 0) -> MultigridOperators:
    """assemble_from_moduli + build_hierarchy + build_multigrid_operators
    (fem.cpp:181, grid.cpp:53, solvers.cpp:460) as one device setup."""
    ops = MultigridOperators(grid, num_coarsenings, poisson_ratio, bc, device)
    ops.set_moduli(moduli, omega)
    return ops


def mg_cycle(ops: MultigridOperators, u: np.ndarray, f: np.ndarray, gamma: int = 1,
             pre_sweeps: int = 2, post_sweeps: int = 2) -> np.ndarray:
    """One gamma-cycle at the finest level (solvers.cpp:483-514); returns u."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    u = np.array(u, dtype=np.float64, copy=True)
    ops._check(ops.lib.tmg_gpu_vcycle(ops.h, dptr(f), dptr(u), gamma, pre_sweeps, post_sweeps))
    return u


def pcgmg_solve(ops: MultigridOperators, b: np.ndarray, cfg: SolverConfig,
                x0: np.ndarray | None = None) -> SolveReport:
    """pcgmg_solve (solvers.cpp:516-530): PCG with one gamma-cycle as M^-1."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    if b.size != ops.grid.dof_count():
        raise DimensionError(f"rhs length {b.size} != dof count {ops.grid.dof_count()}")
    x0c = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
    # r = b - A x0 (solvers.cpp:346-350): the reference's matvec length check
    _check_dofs("matvec", x0c, b.size, "{what}: vector length {got} does not match matrix size {n}")
    x = np.empty_like(b)
    it = C.c_int()
    fr = C.c_double()
    cv = C.c_int()
    sec = C.c_double()
    hist = np.empty(cfg.max_iter + 1)
    hl = C.c_int()
    ops._check(ops.lib.tmg_gpu_solve(ops.h, dptr(b), dptr(x0c), cfg.tol, cfg.max_iter, cfg.gamma,
                                     cfg.pre_sweeps, cfg.post_sweeps, dptr(x), C.byref(it), C.byref(fr),
                                     C.byref(cv), C.byref(sec), dptr(hist), hist.size, C.byref(hl)))
    return SolveReport(solution=x, iterations=it.value, final_residual=fr.value, converged=bool(cv.value),
                       seconds=sec.value, residual_history=hist[: hl.value].tolist())


class PinnedArray:
    """A float64 array in page-locked host memory (tmg_host_alloc), the kind
    of buffer the pipelined solves overlap their copies with; ``.a`` is the
    numpy view. Freed with the object."""

    def __init__(self, n: int):
        self.lib = _lib.load()
        self.ptr = self.lib.tmg_host_alloc(8 * max(1, n))
        if not self.ptr:
            raise CudaError("tmg_host_alloc failed")
        buf = (C.c_double * max(1, n)).from_address(self.ptr)
        buf._owner = self  # the numpy view keeps the pinned block alive
        self.a = np.ctypeslib.as_array(buf)[:n]

    def __del__(self):
        if getattr(self, "ptr", None):
            self.lib.tmg_host_free(self.ptr)
            self.ptr = None


def pcgmg_solve_many(ops: MultigridOperators, problems, cfg: SolverConfig, omega: float = 0.6,
                     outputs=None) -> list:
    """A stream of independent solves on one mesh: problem k = (moduli_k,
    b_k) gets set_moduli(moduli_k, omega) + pcgmg_solve(b_k) semantics
    (solvers.cpp:460-530; bitwise the same results), with the host<->device
    copies of problem k+1's inputs and problem k-1's solution overlapping
    solve k (tmg_gpu_stage_inputs / tmg_gpu_solve_staged, include/tmg_gpu.h).
    Inputs in PinnedArray buffers overlap; plain arrays work, serialised.
    ``outputs``: optional per-problem float64 arrays (pinned to overlap) that
    receive the solutions; by default each report gets a fresh array."""
    probs = [(np.ascontiguousarray(e, dtype=np.float64), np.ascontiguousarray(b, dtype=np.float64))
             for e, b in problems]
    n = ops.grid.dof_count()
    ne = ops.grid.element_count()
    for e, b in probs:
        if e.size != ne:
            raise DimensionError(f"element modulus count {e.size} does not match grid with {ne} elements")
        if b.size != n:
            raise DimensionError(f"rhs length {b.size} != dof count {n}")
    outs = outputs if outputs is not None else [np.empty(n) for _ in probs]
    ops.omega = omega
    lib = ops.lib

    def stage(k):
        e, b = probs[k]
        ops._check(lib.tmg_gpu_stage_inputs(ops.h, k & 1, dptr(e), e.size, dptr(b)))

    reports = []
    if probs:
        stage(0)
    for k in range(len(probs)):
        if k + 1 < len(probs):
            stage(k + 1)
        it, fr, cv, sec, hl = C.c_int(), C.c_double(), C.c_int(), C.c_double(), C.c_int()
        hist = np.empty(cfg.max_iter + 1)
        ops._check(lib.tmg_gpu_solve_staged(ops.h, k & 1, omega, cfg.tol, cfg.max_iter, cfg.gamma,
                                            cfg.pre_sweeps, cfg.post_sweeps, dptr(outs[k]), C.byref(it),
                                            C.byref(fr), C.byref(cv), C.byref(sec), dptr(hist), hist.size,
                                            C.byref(hl)))
        reports.append(SolveReport(solution=outs[k], iterations=it.value, final_residual=fr.value,
                                   converged=bool(cv.value), seconds=sec.value,
                                   residual_history=hist[: hl.value].tolist()))
    ops._check(lib.tmg_gpu_sync_outputs(ops.h))
    return reports


def compliance(ops: MultigridOperators, u: np.ndarray | None = None) -> float:
    """u^T K u (fem.cpp:284-290); u=None uses the resident solution."""
    uc = None if u is None else np.ascontiguousarray(u, dtype=np.float64)
    _check_dofs("compliance", uc, ops.grid.dof_count(), "{what}: vector length {got} != matrix size {n}")
    out = C.c_double()
    ops._check(ops.lib.tmg_gpu_compliance(ops.h, dptr(uc), C.byref(out)))
    return out.value


def element_energies(ops: MultigridOperators, u: np.ndarray | None = None) -> np.ndarray:
    uc = None if u is None else np.ascontiguousarray(u, dtype=np.float64)
    _check_dofs("element_energies", uc, ops.grid.dof_count(), "{what}: vector length {got} != dof count {n}")
    out = np.empty(ops.grid.element_count())
    ops._check(ops.lib.tmg_gpu_element_energies(ops.h, dptr(uc), dptr(out)))
    return out


def sensitivities(ops: MultigridOperators, alpha: np.ndarray, material: MaterialModel,
                  u: np.ndarray | None = None) -> np.ndarray:
    """[nphases, ne] dC/dalpha (mto.cpp:61-85)."""
    uc = None if u is None else np.ascontiguousarray(u, dtype=np.float64)
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    pm = np.ascontiguousarray(material.phase_moduli, dtype=np.float64)
    # mto.cpp:65-70, then element_energies' length check (fem.cpp:295-298)
    _check_density(a, ops.grid, pm.size, "sensitivities")
    _check_dofs("element_energies", uc, ops.grid.dof_count(), "{what}: vector length {got} != dof count {n}")
    out = np.empty((a.shape[1], a.shape[0]))
    ops._check(ops.lib.tmg_gpu_sensitivities(ops.h, dptr(uc), a.shape[1], dptr(a), dptr(pm),
                                             material.penalty, dptr(out)))
    return out


def filter_sensitivities(ops: MultigridOperators, raw: np.ndarray, alpha: np.ndarray, phase: int,
                         radius: float) -> np.ndarray:
    """Density-weighted cone sensitivity filter (mto.cpp:87-117)."""
    r = np.ascontiguousarray(raw, dtype=np.float64)
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    if r.size != ops.grid.element_count():
        raise DimensionError("filter: field length does not match element count")
    if radius > 1.0:  # the density is read only then (mto.cpp:93)
        _check_density(a, ops.grid, None, "filter")
    out = np.empty_like(r)
    ops._check(ops.lib.tmg_gpu_filter(ops.h, a.shape[1], dptr(a), phase, radius, dptr(r), dptr(out)))
    return out


def oc_update_pair(ops: MultigridOperators, alpha: np.ndarray, phase_a: int, phase_b: int,
                   filtered_sens_a: np.ndarray, filtered_sens_b: np.ndarray, target_fraction: float,
                   move, damping: float, floor_eps: float = 1e-3) -> np.ndarray:
    """One OC exchange between two phases (oc_update_pair, mto.cpp:142-227)
    on the device. alpha is the element-major density [ne, nphases] and is
    updated in place (and returned); move is a scalar or a per-element move
    limit (both overloads of mto.hpp:66-77). Raises MultiplierError when the
    volume target cannot be met, ConfigError when the phases coincide."""
    if not (isinstance(alpha, np.ndarray) and alpha.dtype == np.float64 and alpha.flags.c_contiguous
            and alpha.ndim == 2):
        raise DimensionError("oc_update_pair: alpha must be a C-contiguous float64 [ne, nphases] array")
    ne, nph = alpha.shape
    sa = np.ascontiguousarray(filtered_sens_a, dtype=np.float64)
    sb = np.ascontiguousarray(filtered_sens_b, dtype=np.float64)
    mv = np.ascontiguousarray(np.broadcast_to(np.asarray(move, dtype=np.float64), (ne,)))
    if ne != ops.grid.element_count() or sa.size != ne or sb.size != ne:
        raise DimensionError("oc_update_pair: field length does not match grid")
    ops._check(ops.lib.tmg_gpu_oc_update_pair(ops.h, dptr(alpha), nph, floor_eps, phase_a, phase_b, dptr(sa),
                                              dptr(sb), target_fraction, dptr(mv), damping))
    return alpha


def oc_timings(ops: MultigridOperators):
    """(device ms, bisection steps) of the last oc_update_pair."""
    ms, steps = C.c_double(), C.c_int()
    ops._check(ops.lib.tmg_gpu_oc_timings(ops.h, C.byref(ms), C.byref(steps)))
    return ms.value, steps.value


@dataclass
class OptimConfig:
    """OptimConfig (mto.hpp:12-27); the solver method is pcgmg."""
    volume_fractions: list = field(default_factory=lambda: [0.15, 0.15, 0.15, 0.55])
    filter_radius: float = 8.0
    filter_tol: float = 0.05
    tol: float = 1e-3
    inner_sweeps: int = 1
    move_limit: float = 0.2
    oc_damping: float = 0.5
    warm_start: bool = False
    max_outer: int = 2000
    density_floor: float = 1e-3
    solver: SolverConfig = field(default_factory=SolverConfig)


@dataclass
class OptimReport:
    """OptimReport (mto.hpp:29-39); density is element-major [ne, nphases]."""
    density: np.ndarray
    compliance_history: list
    change_history: list
    solver_iteration_history: list
    seconds_history: list
    outer_iterations: int
    total_solver_iterations: int
    seconds: float
    converged: bool


def optimize(ops: MultigridOperators, material: MaterialModel, cfg: OptimConfig,
             rhs: np.ndarray | None = None) -> OptimReport:
    """optimize() with Method::pcgmg (mto.cpp:229-354), every per-iteration
    step on the device. ops carries the grid, the supports and Poisson's
    ratio; rhs defaults to the wall problem's uniform top load."""
    if rhs is None:
        rhs = assemble_rhs(ops.grid, wall_boundary_conditions(ops.grid, "uniform"))
    b = np.ascontiguousarray(rhs, dtype=np.float64)
    if b.size != ops.grid.dof_count():
        raise DimensionError("optimize: rhs length does not match the grid")
    pm = np.ascontiguousarray(material.phase_moduli, dtype=np.float64)
    fr = np.ascontiguousarray(cfg.volume_fractions, dtype=np.float64)
    if fr.size != pm.size:
        raise ConfigError(f"volume fraction count {fr.size} does not match phase count {pm.size}")
    from ._lib import OptimConfigC
    s = cfg.solver
    c = OptimConfigC(pm.size, dptr(pm), material.penalty, dptr(fr), cfg.filter_radius, cfg.filter_tol, cfg.tol,
                     cfg.inner_sweeps, cfg.move_limit, cfg.oc_damping, int(cfg.warm_start), cfg.max_outer,
                     cfg.density_floor, s.tol, s.max_iter, s.gamma, s.pre_sweeps, s.post_sweeps, s.omega)
    ne, m = ops.grid.element_count(), max(cfg.max_outer, 1)
    dens = np.empty((ne, pm.size))
    ch, dh, sh = np.zeros(m), np.zeros(m), np.zeros(m)
    ih = np.zeros(m, dtype=np.int32)
    oi, cv = C.c_int(), C.c_int()
    ti, sec = C.c_long(), C.c_double()
    ops._check(ops.lib.tmg_gpu_optimize(ops.h, C.byref(c), dptr(b), dptr(dens), dptr(ch), dptr(dh), iptr(ih),
                                        dptr(sh), C.byref(oi), C.byref(ti), C.byref(cv), C.byref(sec)))
    k = oi.value
    return OptimReport(dens, list(ch[:k]), list(dh[:k]), [int(v) for v in ih[:k]], list(sh[:k]), k, ti.value,
                       sec.value, bool(cv.value))


# ------------------------------------------------------------- Poisson --
# The paper's Poisson path (fem.cpp:232-276, bench.cpp:30-111; SURVEY.md 8(f)
# item 3): 1 dof per node, every boundary node fixed.

def poisson_element_matrices():
    """(k_lap, m_mass), the 4x4 element matrices of fem.cpp:37-81."""
    k, m = np.empty(16), np.empty(16)
    _lib.load().tmg_poisson_element_matrices(dptr(k), dptr(m))
    return k.reshape(4, 4), m.reshape(4, 4)


def assemble_poisson_rhs(grid: GridLevel, source) -> np.ndarray:
    """The right-hand side of assemble_poisson for a per-node (or constant)
    source: -M f assembled element by element, boundary entries 0."""
    n = (grid.nx + 1) * (grid.ny + 1)
    f = np.ascontiguousarray(np.broadcast_to(np.asarray(source, dtype=np.float64), (n,)))
    b = np.empty(n)
    _lib.load().tmg_inputs_poisson_rhs(grid.nx, grid.ny, dptr(f), dptr(b))
    return b


def poisson_full_depth(grid: int) -> int:
    """Coarsenings down to a 2x2 coarsest grid (bench.cpp:17-24)."""
    d = 0
    while grid > 2:
        grid //= 2
        d += 1
    return d


class PoissonMultigrid:
    """build_hierarchy(nx, ny, nc, 1) + build_multigrid_operators of the
    Poisson system, resident on the GPU."""

    def __init__(self, grid: GridLevel, num_coarsenings: int, omega: float = 0.6, device: int = 0):
        self.lib = _lib.load()
        self.grid, self.nc = grid, num_coarsenings
        h = C.c_void_p()
        st = self.lib.tmg_poisson_create(grid.nx, grid.ny, num_coarsenings, device, C.byref(h))
        if st:
            _raise(st, "tmg_poisson_create: invalid hierarchy or CUDA failure")
        self.h = h
        self._check(self.lib.tmg_poisson_setup(self.h, omega))

    def _check(self, st):
        if st:
            buf = C.create_string_buffer(512)
            self.lib.tmg_poisson_last_error(self.h, buf, 512)
            _raise(st, buf.value.decode())

    def close(self):
        if getattr(self, "h", None):
            self.lib.tmg_poisson_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def level_planes(self, level: int) -> np.ndarray:
        """[5, (nx_l+1)(ny_l+1)]: centre, N, SE, E, NE stencil entries per node."""
        nx, ny = self.grid.nx >> (self.nc - level), self.grid.ny >> (self.nc - level)
        out = np.empty((5, (nx + 1) * (ny + 1)))
        self._check(self.lib.tmg_poisson_level_values(self.h, level, dptr(out)))
        return out

    def vcycle(self, u: np.ndarray, f: np.ndarray, gamma: int = 1, pre: int = 2, post: int = 2) -> np.ndarray:
        out = np.array(u, dtype=np.float64, copy=True)
        ff = np.ascontiguousarray(f, dtype=np.float64)
        self._check(self.lib.tmg_poisson_vcycle(self.h, dptr(ff), dptr(out), gamma, pre, post))
        return out

    def solve(self, b: np.ndarray, cfg: SolverConfig, x0: np.ndarray | None = None) -> SolveReport:
        bb = np.ascontiguousarray(b, dtype=np.float64)
        x0c = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
        x = np.empty_like(bb)
        hist = np.empty(cfg.max_iter + 1)
        it, cv, hl = C.c_int(), C.c_int(), C.c_int()
        fr, sec = C.c_double(), C.c_double()
        self._check(self.lib.tmg_poisson_solve(self.h, dptr(bb), dptr(x0c), cfg.tol, cfg.max_iter, cfg.gamma,
                                               cfg.pre_sweeps, cfg.post_sweeps, dptr(x), C.byref(it), C.byref(fr),
                                               C.byref(cv), C.byref(sec), dptr(hist), hist.size, C.byref(hl)))
        return SolveReport(x, it.value, fr.value, bool(cv.value), sec.value, list(hist[: hl.value]))


# ------------------------------------------------------------- outputs --
# Byte-compatible with the reference writers (report.cpp:34-97, 153-168);
# host-side, like the reference's.

def _fmt(v: float) -> str:
    return "%.17g" % v  # report.cpp:17-19


def _to_byte(a: np.ndarray) -> np.ndarray:
    """report.cpp:28-31: clamp(lround(255 a), 0, 255), lround = half away from zero."""
    x = 255.0 * np.asarray(a, dtype=np.float64)
    fl = np.floor(x)
    r = np.where(x - fl >= 0.5, fl + 1.0, fl)  # x >= 0 here; negatives clamp to 0 anyway
    return np.clip(r, 0, 255).astype(np.uint8)


def write_history_csv(report: OptimReport, path) -> None:
    with open(path, "w", newline="") as out:
        out.write("iteration,compliance,max_change,solver_iterations,seconds\n")
        for i in range(len(report.compliance_history)):
            out.write(f"{i + 1},{_fmt(report.compliance_history[i])},{_fmt(report.change_history[i])},"
                      f"{int(report.solver_iteration_history[i])},{_fmt(report.seconds_history[i])}\n")


def write_residual_csv(report: SolveReport, path) -> None:
    with open(path, "w", newline="") as out:
        out.write("iteration,relative_residual\n")
        for i, v in enumerate(report.residual_history):
            out.write(f"{i},{_fmt(v)}\n")


def _image_rows(alpha: np.ndarray, nx: int, ny: int) -> np.ndarray:
    """[ny, nx, nphases], top row first (report.cpp:55-57: ey = ny-1 .. 0)."""
    return np.asarray(alpha, dtype=np.float64).reshape(nx, ny, -1).transpose(1, 0, 2)[::-1]


def write_phase_pgm(alpha: np.ndarray, nx: int, ny: int, phase: int, path) -> None:
    img = _to_byte(_image_rows(alpha, nx, ny)[:, :, phase])
    with open(path, "wb") as out:
        out.write(f"P5\n{nx} {ny}\n255\n".encode())
        out.write(img.tobytes())


def write_composite_ppm(alpha: np.ndarray, nx: int, ny: int, path) -> None:
    a = _image_rows(alpha, nx, ny)
    nph = a.shape[2]
    rgb = np.zeros(a.shape[:2] + (3,))
    for i in range(nph):  # void (last) and phases beyond the third render gray
        if i < 3 and i != nph - 1:
            rgb[:, :, i] += a[:, :, i]
        else:
            rgb += a[:, :, i:i + 1]
    img = _to_byte(np.minimum(1.0, rgb))
    with open(path, "wb") as out:
        out.write(f"P6\n{nx} {ny}\n255\n".encode())
        out.write(img.tobytes())


def emit_outputs(report: OptimReport, grid: GridLevel, out_dir, images: bool = True, csv: bool = True) -> None:
    """emit_outputs (report.cpp:153-168): history.csv, phase_<i>.pgm, composite.ppm."""
    import os

    os.makedirs(out_dir, exist_ok=True)
    if csv:
        write_history_csv(report, os.path.join(out_dir, "history.csv"))
    if images:
        for i in range(report.density.shape[1]):
            write_phase_pgm(report.density, grid.nx, grid.ny, i, os.path.join(out_dir, f"phase_{i + 1}.pgm"))
        write_composite_ppm(report.density, grid.nx, grid.ny, os.path.join(out_dir, "composite.ppm"))


__all__ = [n for n in dir() if not n.startswith("_") and n not in ("C", "dataclasses", "np", "dataclass", "field")]
