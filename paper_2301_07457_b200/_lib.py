"""ctypes binding of libtmg_gpu.so (the C ABI declared in include/tmg_gpu.h).

The shared library is built in-tree by ``paper_2301_07457_b200.build`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``). There is no fallback: if the
library is missing, loading raises instead of routing anywhere else.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib

import numpy as np

PKG_DIR = pathlib.Path(__file__).resolve().parent
# TMG_LIB_PATH points the loader at another build of the same library (A/B
# timing of kernel variants within one GPU session); the default is in-tree
LIB_PATH = pathlib.Path(os.environ.get("TMG_LIB_PATH", PKG_DIR / "libtmg_gpu.so"))

_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)
_H = C.c_void_p

# (name, restype, argtypes) for every symbol include/tmg_gpu.h declares
class OptimConfigC(C.Structure):
    """tmg_optim_config (include/tmg_gpu.h): OptimConfig + SolverConfig flattened."""
    _fields_ = [("nphases", C.c_int), ("phase_moduli", _D), ("penalty", C.c_double),
                ("volume_fractions", _D), ("filter_radius", C.c_double), ("filter_tol", C.c_double),
                ("tol", C.c_double), ("inner_sweeps", C.c_int), ("move_limit", C.c_double),
                ("oc_damping", C.c_double), ("warm_start", C.c_int), ("max_outer", C.c_int),
                ("density_floor", C.c_double), ("solver_tol", C.c_double), ("solver_max_iter", C.c_int),
                ("gamma", C.c_int), ("pre_sweeps", C.c_int), ("post_sweeps", C.c_int), ("omega", C.c_double)]


SIGNATURES = [
    ("tmg_gpu_create", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(_H)]),
    ("tmg_gpu_destroy", None, [_H]),
    ("tmg_partition", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _I, _I]),
    ("tmg_gpu_create_local_slabs", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                             C.POINTER(_H)]),
    ("tmg_gpu_create_nccl", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                      C.c_int, C.POINTER(_H)]),
    ("tmg_nccl_unique_id", C.c_int, [C.c_void_p]),
    ("tmg_gpu_last_error", C.c_int, [_H, C.c_char_p, C.c_int, _I]),
    ("tmg_gpu_set_problem", C.c_int, [_H, C.c_double, _I, C.c_int]),
    ("tmg_gpu_set_moduli", C.c_int, [_H, _D, C.c_long, C.c_double]),
    ("tmg_gpu_upload_moduli", C.c_int, [_H, _D, C.c_long]),
    ("tmg_gpu_setup", C.c_int, [_H, C.c_double]),
    ("tmg_gpu_set_density", C.c_int, [_H, _D, C.c_int, _D, C.c_double, C.c_double]),
    ("tmg_gpu_solve", C.c_int, [_H, _D, _D, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, _D, _I,
                                _D, _I, _D, _D, C.c_int, _I]),
    ("tmg_gpu_upload_rhs", C.c_int, [_H, _D]),
    ("tmg_gpu_upload_x0", C.c_int, [_H, _D]),
    ("tmg_gpu_solve_resident", C.c_int, [_H, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                         _I, _D, _I, _D, _D, C.c_int, _I]),
    ("tmg_gpu_download_solution", C.c_int, [_H, _D]),
    ("tmg_gpu_solution_to_x0", C.c_int, [_H]),
    ("tmg_gpu_stage_inputs", C.c_int, [_H, C.c_int, _D, C.c_long, _D]),
    ("tmg_gpu_solve_staged", C.c_int, [_H, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                       _D, _I, _D, _I, _D, _D, C.c_int, _I]),
    ("tmg_gpu_sync_outputs", C.c_int, [_H]),
    ("tmg_gpu_compliance", C.c_int, [_H, _D, _D]),
    ("tmg_gpu_element_energies", C.c_int, [_H, _D, _D]),
    ("tmg_gpu_sensitivities", C.c_int, [_H, _D, C.c_int, _D, _D, C.c_double, _D]),
    ("tmg_gpu_filter", C.c_int, [_H, C.c_int, _D, C.c_int, C.c_double, _D, _D]),
    ("tmg_gpu_oc_update_pair", C.c_int,
     [_H, _D, C.c_int, C.c_double, C.c_int, C.c_int, _D, _D, C.c_double, _D, C.c_double]),
    ("tmg_gpu_oc_timings", C.c_int, [_H, _D, _I]),
    ("tmg_poisson_create", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(_H)]),
    ("tmg_poisson_destroy", None, [_H]),
    ("tmg_poisson_last_error", C.c_int, [_H, C.c_char_p, C.c_int]),
    ("tmg_poisson_setup", C.c_int, [_H, C.c_double]),
    ("tmg_poisson_level_values", C.c_int, [_H, C.c_int, _D]),
    ("tmg_poisson_vcycle", C.c_int, [_H, _D, _D, C.c_int, C.c_int, C.c_int]),
    ("tmg_poisson_solve", C.c_int, [_H, _D, _D, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, _D, _I, _D, _I,
                                    _D, _D, C.c_int, _I]),
    ("tmg_poisson_element_matrices", None, [_D, _D]),
    ("tmg_inputs_poisson_rhs", None, [C.c_int, C.c_int, _D, _D]),
    ("tmg_gpu_optimize", C.c_int, [_H, C.POINTER(OptimConfigC), _D, _D, _D, _D, _I, _D, _I,
                                   C.POINTER(C.c_long), _I, _D]),
    ("tmg_gpu_apply", C.c_int, [_H, C.c_int, _D, _D]),
    ("tmg_gpu_level_values", C.c_int, [_H, C.c_int, _I, _I, _D]),
    ("tmg_gpu_vcycle", C.c_int, [_H, _D, _D, C.c_int, C.c_int, C.c_int]),
    ("tmg_gpu_prolongate", C.c_int, [_H, C.c_int, _D, _D]),
    ("tmg_gpu_restrict", C.c_int, [_H, C.c_int, _D, _D]),
    ("tmg_gpu_smooth", C.c_int, [_H, C.c_int, _D, _D, C.c_int]),
    ("tmg_gpu_stream", C.c_void_p, [_H]),
    ("tmg_gpu_launch_count", C.c_long, [_H]),
    ("tmg_gpu_time_kernel", C.c_int, [_H, C.c_int, C.c_int, _D, _D]),
    ("tmg_gpu_last_timings", C.c_int, [_H, _D, _D]),
    ("tmg_gpu_event_record", C.c_int, [_H, C.c_int]),
    ("tmg_gpu_event_elapsed", C.c_int, [_H, C.c_int, C.c_int, _D]),
    ("tmg_host_alloc", C.c_void_p, [C.c_ulong]),
    ("tmg_host_free", None, [C.c_void_p]),
    ("tmg_element_stiffness", None, [C.c_double, C.c_double, _D]),
    ("tmg_inputs_effective_moduli", None, [C.c_long, C.c_int, _D, _D, C.c_double, _D]),
    ("tmg_inputs_density_iid", None, [C.c_int, C.c_int, C.c_int, C.c_ulonglong, _D]),
    ("tmg_inputs_density_checker", None, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_ulonglong, _D]),
    ("tmg_inputs_wall_bc", None, [C.c_int, C.c_int, C.c_int, _I, _I, _I, _D, _I]),
    ("tmg_inputs_rhs", C.c_int, [C.c_int, C.c_int, _I, C.c_int, _I, _D, C.c_int, _D]),
]

_lib = None


def load():
    """Load libtmg_gpu.so once; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (the GPU path has no CPU fallback)")
    lib = C.CDLL(os.fspath(LIB_PATH))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def iptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_I)
