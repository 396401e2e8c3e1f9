"""TEST INFRASTRUCTURE ONLY -- ctypes access to the CPU checkers.

``Checker('orc')`` loads oracle/liboracle.so (the committed plain-C
restatement); ``Checker('ref')`` loads oracle/_ref/libtopmg_ref.so (the
unmodified reference compiled from /root/reference by oracle/Makefile). Both
export the same function set (topmg_oracle.h / ref_shim.cpp). Only tests/,
__graft_entry__.smoke() and bench.py's CPU legs import this module.
"""
from __future__ import annotations

import ctypes as C
import pathlib

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
PATHS = {"orc": HERE / "liboracle.so", "ref": HERE / "_ref" / "libtopmg_ref.so"}

_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)


class OracleError(RuntimeError):
    def __init__(self, code, msg, row=-1):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg
        self.row = row


def available(kind: str) -> bool:
    return PATHS[kind].exists()


def _d(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def _i(a):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_I)


_cache = {}


def lib(kind: str):
    if kind in _cache:
        return _cache[kind]
    L = C.CDLL(str(PATHS[kind]))
    p = kind + "_"
    sig = {
        "element_stiffness": (None, [C.c_double, C.c_double, _D]),
        "system_create": (C.c_void_p, [C.c_int, C.c_int, _D, C.c_double, _I, C.c_int, _I, _D, C.c_int,
                                       C.c_char_p, C.c_int, _I]),
        "system_build_mg": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_char_p, C.c_int, _I]),
        "system_num_levels": (C.c_int, [C.c_void_p]),
        "system_rhs": (None, [C.c_void_p, _D]),
        "system_level_nnz": (C.c_long, [C.c_void_p, C.c_int]),
        "system_level_size": (C.c_int, [C.c_void_p, C.c_int]),
        "system_level_csr": (C.c_int, [C.c_void_p, C.c_int, _I, _I, _D]),
        "system_matvec": (C.c_int, [C.c_void_p, C.c_int, _D, _D]),
        "system_vcycle": (C.c_int, [C.c_void_p, _D, _D, C.c_int, C.c_int, C.c_int]),
        "system_solve": (C.c_int, [C.c_void_p, _D, _D, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, _D,
                                   _I, _D, _I, _D, _I, C.c_char_p, C.c_int]),
        "system_times": (None, [C.c_void_p, _D]),
        "system_compliance": (C.c_double, [C.c_void_p, _D]),
        "system_destroy": (None, [C.c_void_p]),
        "element_energies": (C.c_int, [C.c_int, C.c_int, _D, C.c_double, _D]),
        "effective_moduli": (None, [C.c_int, C.c_int, C.c_int, _D, _D, C.c_double, _D]),
        "density_iid": (None, [C.c_int, C.c_int, C.c_int, C.c_ulonglong, _D]),
        "density_checker": (None, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_ulonglong, _D]),
        "sensitivities": (C.c_int, [C.c_int, C.c_int, C.c_int, _D, _D, C.c_double, C.c_double, _D, _D]),
        "filter": (C.c_int, [C.c_int, C.c_int, C.c_int, _D, C.c_int, C.c_double, _D, _D]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, p + name)
        f.restype = res
        f.argtypes = args
    _cache[kind] = L
    return L


def density_iid(kind, nx, ny, seed, nmat=3):
    """BASELINE c1/c4 densities [nx*ny, nmat+1] (oracles.hpp:21-23 recipe)."""
    a = np.empty((nx * ny, nmat + 1))
    getattr(lib(kind), kind + "_density_iid")(nx, ny, nmat, seed, _d(a))
    return a


def density_checker(kind, nx, ny, block, seed, nphases=4):
    """BASELINE c2 one-hot checkerboard [nx*ny, nphases]."""
    a = np.empty((nx * ny, nphases))
    getattr(lib(kind), kind + "_density_checker")(nx, ny, block, nphases, seed, _d(a))
    return a


def effective_moduli(kind, nx, ny, alpha, phase_moduli, penalty):
    """effective_moduli (density.cpp:68-85)."""
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    pm = np.ascontiguousarray(phase_moduli, dtype=np.float64)
    out = np.empty(nx * ny)
    getattr(lib(kind), kind + "_effective_moduli")(nx, ny, a.shape[1], _d(a), _d(pm), penalty, _d(out))
    return out


def wall_uniform_bc(nx, ny):
    """BASELINE supports and load: both dofs of every bottom
    node fixed (fem.cpp:328-332), -1/(nx+1) on the v-dof of every top node."""
    x = np.arange(nx + 1)
    fixed = np.stack([2 * x * (ny + 1), 2 * x * (ny + 1) + 1], axis=1).ravel().tolist()
    loads = [(int(2 * (xi * (ny + 1) + ny) + 1), -1.0 / (nx + 1)) for xi in x]
    return fixed, loads


class System:
    """assemble_from_moduli (+ build_multigrid_operators on demand)."""

    def __init__(self, kind, nx, ny, moduli, nu, fixed, loads):
        self.kind, self.L, self.p = kind, lib(kind), kind + "_"
        self.nx, self.ny = nx, ny
        self.n = 2 * (nx + 1) * (ny + 1)
        e = np.ascontiguousarray(moduli, dtype=np.float64)
        fx = np.ascontiguousarray(fixed, dtype=np.int32)
        ld = np.ascontiguousarray([d for d, _ in loads], dtype=np.int32)
        lv = np.ascontiguousarray([v for _, v in loads], dtype=np.float64)
        err = C.create_string_buffer(256)
        st = C.c_int()
        self.h = self._f("system_create")(nx, ny, _d(e), nu, _i(fx), len(fx), _i(ld), _d(lv), len(lv), err, 256,
                                          C.byref(st))
        if st.value:
            raise OracleError(st.value, err.value.decode())
        self.levels = 1

    def _f(self, name):
        return getattr(self.L, self.p + name)

    def build_mg(self, num_coarsenings, omega=0.6):
        err = C.create_string_buffer(256)
        row = C.c_int(-1)
        st = self._f("system_build_mg")(self.h, num_coarsenings, omega, err, 256, C.byref(row))
        if st:
            raise OracleError(st, err.value.decode(), row.value)
        self.levels = num_coarsenings + 1
        return self

    def rhs(self):
        b = np.empty(self.n)
        self._f("system_rhs")(self.h, _d(b))
        return b

    def csr(self, level):
        n = self._f("system_level_size")(self.h, level)
        nnz = self._f("system_level_nnz")(self.h, level)
        off = np.empty(n + 1, np.int32)
        col = np.empty(nnz, np.int32)
        val = np.empty(nnz)
        st = self._f("system_level_csr")(self.h, level, _i(off), _i(col), _d(val))
        if st:
            raise OracleError(st, "level_csr")
        return off, col, val

    def matvec(self, level, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x)
        st = self._f("system_matvec")(self.h, level, _d(x), _d(y))
        if st:
            raise OracleError(st, "matvec")
        return y

    def vcycle(self, f, u, gamma=1, pre=2, post=2):
        f = np.ascontiguousarray(f, dtype=np.float64)
        u = np.array(u, dtype=np.float64, copy=True)
        st = self._f("system_vcycle")(self.h, _d(f), _d(u), gamma, pre, post)
        if st:
            raise OracleError(st, "vcycle")
        return u

    def solve(self, b, tol=1e-8, max_iter=1000, gamma=1, pre=2, post=2, x0=None):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x0c = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
        x = np.empty(self.n)
        it, cv, hl = C.c_int(), C.c_int(), C.c_int()
        fr = C.c_double()
        hist = np.empty(max_iter + 1)
        err = C.create_string_buffer(256)
        st = self._f("system_solve")(self.h, _d(b), _d(x0c), tol, max_iter, gamma, pre, post, _d(x), C.byref(it),
                                     C.byref(fr), C.byref(cv), _d(hist), C.byref(hl), err, 256)
        if st:
            raise OracleError(st, err.value.decode())
        return dict(solution=x, iterations=it.value, final_residual=fr.value, converged=bool(cv.value),
                    residual_history=hist[: hl.value].copy())

    def times(self):
        t = np.empty(3)
        self._f("system_times")(self.h, _d(t))
        return dict(assemble=t[0], setup=t[1], pcg=t[2])

    def compliance(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        return self._f("system_compliance")(self.h, _d(u))

    def close(self):
        if self.h:
            self._f("system_destroy")(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def poisson_system(kind, nx, ny, source):
    """assemble_poisson (fem.cpp:232-276) as a System (1 dof per node); source is
    a per-node array or a constant."""
    src = np.ascontiguousarray(np.broadcast_to(np.asarray(source, dtype=np.float64), ((nx + 1) * (ny + 1),)))
    s = System.__new__(System)
    s.kind, s.p, s.nx, s.ny = kind, kind + "_", nx, ny
    s.L = lib(kind)
    s.n = (nx + 1) * (ny + 1)
    s.levels = 1
    err = C.create_string_buffer(256)
    st = C.c_int()
    f = getattr(s.L, kind + "_poisson_create")
    f.restype = C.c_void_p
    s.h = f(nx, ny, _d(src), err, 256, C.byref(st))
    if st.value:
        raise OracleError(st.value, err.value.decode())
    return s


def element_stiffness(kind, modulus, nu):
    k = np.empty(64)
    getattr(lib(kind), kind + "_element_stiffness")(modulus, nu, _d(k))
    return k.reshape(8, 8)


def element_energies(kind, nx, ny, u, nu):
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty(nx * ny)
    getattr(lib(kind), kind + "_element_energies")(nx, ny, _d(u), nu, _d(out))
    return out


def effective_moduli(kind, nx, ny, alpha, phase_moduli, penalty):
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    pm = np.ascontiguousarray(phase_moduli, dtype=np.float64)
    out = np.empty(nx * ny)
    getattr(lib(kind), kind + "_effective_moduli")(nx, ny, a.shape[1], _d(a), _d(pm), penalty, _d(out))
    return out


def sensitivities(kind, nx, ny, alpha, phase_moduli, penalty, nu, u):
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    pm = np.ascontiguousarray(phase_moduli, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty((a.shape[1], nx * ny))
    getattr(lib(kind), kind + "_sensitivities")(nx, ny, a.shape[1], _d(a), _d(pm), penalty, nu, _d(u), _d(out))
    return out


def filter_sensitivities(kind, nx, ny, alpha, phase, radius, raw):
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    raw = np.ascontiguousarray(raw, dtype=np.float64)
    out = np.empty(nx * ny)
    getattr(lib(kind), kind + "_filter")(nx, ny, a.shape[1], _d(a), phase, radius, _d(raw), _d(out))
    return out


def oc_update_pair(kind, alpha, phase_a, phase_b, sens_a, sens_b, target, move, damping, floor_eps=1e-3):
    """One OC exchange (mto.cpp:142-227) on a copy of the element-major density
    alpha [ne, nphases]; returns (new alpha, status) -- status 8 is the
    reference's MultiplierError (alpha is then unchanged)."""
    a = np.array(alpha, dtype=np.float64, copy=True, order="C")
    ne, nph = a.shape
    sa = np.ascontiguousarray(sens_a, dtype=np.float64)
    sb = np.ascontiguousarray(sens_b, dtype=np.float64)
    mv = np.ascontiguousarray(np.broadcast_to(np.asarray(move, dtype=np.float64), (ne,)))
    f = getattr(lib(kind), kind + "_oc_update_pair")
    f.restype = C.c_int
    f.argtypes = [C.c_long, C.c_int, C.c_double, _D, C.c_int, C.c_int, _D, _D, C.c_double, _D, C.c_double]
    st = f(ne, nph, floor_eps, _d(a), phase_a, phase_b, _d(sa), _d(sb), target, _d(mv), damping)
    return a, st


def optimize(kind, nx, ny, fixed, loads, phase_moduli, penalty, nu, fractions, filter_radius=1.5,
             filter_tol=0.05, tol=1e-3, inner_sweeps=1, move_limit=0.2, oc_damping=0.5, warm_start=False,
             max_outer=10, density_floor=1e-3, num_coarsenings=2, omega=0.6, solver_tol=1e-8,
             solver_max_iter=2000, gamma=1, pre=2, post=2):
    """optimize() with Method::pcgmg (mto.cpp:229-354). Returns a dict with the
    OptimReport fields; raises OracleError on a reference exception."""
    np_ = len(phase_moduli)
    fx = np.ascontiguousarray(fixed, dtype=np.int32)
    ld = np.ascontiguousarray([l[0] for l in loads], dtype=np.int32)
    lv = np.ascontiguousarray([l[1] for l in loads], dtype=np.float64)
    pm = np.ascontiguousarray(phase_moduli, dtype=np.float64)
    fr = np.ascontiguousarray(fractions, dtype=np.float64)
    dens = np.empty(nx * ny * np_)
    ch, dh = np.zeros(max_outer), np.zeros(max_outer)
    ih = np.zeros(max_outer, dtype=np.int32)
    oi, cv = C.c_int(), C.c_int()
    ti = C.c_long()
    err = C.create_string_buffer(256)
    f = getattr(lib(kind), kind + "_optimize")
    f.restype = C.c_int
    st = f(nx, ny, np_, _d(pm), C.c_double(penalty), C.c_double(nu), fx.ctypes.data_as(_I), len(fx),
           ld.ctypes.data_as(_I), _d(lv), len(lv), _d(fr), C.c_double(filter_radius), C.c_double(filter_tol),
           C.c_double(tol), inner_sweeps, C.c_double(move_limit), C.c_double(oc_damping), int(warm_start),
           max_outer, C.c_double(density_floor), num_coarsenings, C.c_double(omega), C.c_double(solver_tol),
           solver_max_iter, gamma, pre, post, _d(dens), _d(ch), _d(dh), ih.ctypes.data_as(_I), C.byref(oi),
           C.byref(ti), C.byref(cv), err, 256)
    if st:
        raise OracleError(st, err.value.decode())
    k = oi.value
    return dict(density=dens.reshape(nx * ny, np_), compliance_history=ch[:k], change_history=dh[:k],
                solver_iteration_history=ih[:k], outer_iterations=k, total_solver_iterations=ti.value,
                converged=bool(cv.value))


def ref_write_history_csv(report, path):
    """The reference's write_history_csv (report.cpp:34-43) on an OptimReport-like object."""
    n = len(report.compliance_history)
    c = np.ascontiguousarray(report.compliance_history, dtype=np.float64)
    d = np.ascontiguousarray(report.change_history, dtype=np.float64)
    it = np.ascontiguousarray(report.solver_iteration_history, dtype=np.int32)
    s = np.ascontiguousarray(report.seconds_history, dtype=np.float64)
    st = lib("ref").ref_write_history_csv(n, _d(c), _d(d), it.ctypes.data_as(_I), _d(s), str(path).encode())
    if st:
        raise OracleError(st, "write_history_csv")


def ref_write_residual_csv(hist, path):
    h = np.ascontiguousarray(hist, dtype=np.float64)
    st = lib("ref").ref_write_residual_csv(len(h), _d(h), str(path).encode())
    if st:
        raise OracleError(st, "write_residual_csv")


def ref_write_density_images(nx, ny, alpha, directory):
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    st = lib("ref").ref_write_density_images(nx, ny, a.shape[1], _d(a), str(directory).encode())
    if st:
        raise OracleError(st, "write images")
