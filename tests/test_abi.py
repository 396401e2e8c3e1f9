"""The C-ABI library: loads on a CPU-only host, exports every symbol that
include/tmg_gpu.h declares, its host-side input producers are exact, and the
GPU entry points fail loudly (no CPU fallback) when no sm_100 device exists."""
import ctypes as C
import pathlib
import re

import numpy as np
import pytest

import paper_2301_07457_b200 as P
from paper_2301_07457_b200 import _lib
from oracle import pyoracle as po

ROOT = pathlib.Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "tmg_gpu.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tmg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_symbols()
    for must in ("tmg_gpu_create", "tmg_gpu_set_problem", "tmg_gpu_set_moduli", "tmg_gpu_solve",
                 "tmg_gpu_compliance", "tmg_gpu_element_energies", "tmg_gpu_sensitivities", "tmg_gpu_filter",
                 "tmg_gpu_destroy", "tmg_gpu_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes table covers the header exactly
    assert sorted(n for n, _, _ in _lib.SIGNATURES) == declared_symbols()


def test_library_is_built_for_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "-lelf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_host_element_stiffness_is_bit_identical_to_the_reference_oracle():
    for nu in (0.1, 0.3, 0.42):
        assert np.array_equal(P.element_stiffness(1.0, nu), po.element_stiffness("orc", 1.0, nu))


def test_host_moduli_match_effective_moduli():
    a = P.density_iid(12, 9, 3)
    assert np.all(a >= 0) and np.allclose(a.sum(1), 1.0)
    E = P.effective_moduli(a, P.MaterialModel())
    assert np.array_equal(E, po.effective_moduli("orc", 12, 9, a, [1.0, 0.5, 0.2, 1e-9], 3.0))
    c = P.density_checker(32, 32, 16, 2)
    assert set(np.unique(c)) <= {0.0, 1.0} and np.all(c.sum(1) == 1.0)
    # one phase per 16x16 block
    blk = c.reshape(32, 32, 4)[:16, :16]
    assert np.all(blk == blk[0, 0])


def test_wall_bc_and_rhs_match_assembly():
    g = P.GridLevel(8, 6)
    for load in ("point", "uniform"):
        bc = P.wall_boundary_conditions(g, load)
        assert len(bc.fixed_dofs) == 2 * (g.nx + 1)
        b = P.assemble_rhs(g, bc)
        s = po.System("orc", g.nx, g.ny, np.ones(g.element_count()), 0.3, bc.fixed_dofs, bc.point_loads)
        assert np.array_equal(b, s.rhs())
        assert abs(b.sum() + 1.0) < 1e-15
    with pytest.raises(P.ConfigError):
        P.wall_boundary_conditions(P.GridLevel(7, 4), "point")


def test_solver_config_validation_mirrors_reference():
    """test_solvers.cpp:510-523."""
    cfg = P.SolverConfig(pre_sweeps=2, post_sweeps=3)
    with pytest.raises(P.ConfigError):
        cfg.validate()
    cfg.post_sweeps = 2
    cfg.validate()
    cfg.omega = 1.5
    with pytest.raises(P.ConfigError):
        cfg.validate()
    cfg.omega = 0.6
    cfg.gamma = 3
    with pytest.raises(P.ConfigError):
        cfg.validate()


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_a_gpu():
    g = P.GridLevel(8, 8)
    with pytest.raises(P.CudaError):
        P.MultigridOperators(g, 2, 0.3, P.wall_boundary_conditions(g, "uniform"))


def test_config_errors_precede_device_work():
    # build_hierarchy validation happens before any device call (grid.cpp:55-80)
    with pytest.raises(P.ConfigError):
        P.MultigridOperators(P.GridLevel(10, 8), 2, 0.3, P.BoundaryConditions())
    with pytest.raises(P.ConfigError):
        P.MultigridOperators(P.GridLevel(0, 8), 0, 0.3, P.BoundaryConditions())
    # the documented limits of the device coarse solve (include/tmg_gpu.h): at
    # most 16,900 coarsest dofs, and above 2048 dofs node columns of <= 148 nodes
    with pytest.raises(P.ConfigError, match="16900"):
        P.MultigridOperators(P.GridLevel(512, 512), 2, 0.3, P.BoundaryConditions())
    with pytest.raises(P.ConfigError, match="148 nodes"):
        P.MultigridOperators(P.GridLevel(2, 4096), 1, 0.3, P.BoundaryConditions())


def test_boundary_condition_validation_mirrors_reference():
    """BoundaryConditions::validate (fem.cpp:110-129), in the Python mirror and
    in the C entry point itself (which leaves b untouched)."""
    g = P.GridLevel(4, 4)
    n = g.dof_count()
    cases = [
        (P.BoundaryConditions([n], []), f"fixed dof {n} outside [0, {n})"),
        (P.BoundaryConditions([-1], []), f"fixed dof -1 outside [0, {n})"),
        (P.BoundaryConditions([0], [(n + 3, 1.0)]), f"loaded dof {n + 3} outside [0, {n})"),
        (P.BoundaryConditions([0, 7], [(7, -1.0)]), "dof 7 is both fixed and loaded"),
    ]
    lib = P._lib.load()
    for bc, msg in cases:
        with pytest.raises(P.ConfigError, match=msg.replace("[", r"\[").replace("(", r"\(").replace(")", r"\)")):
            P.assemble_rhs(g, bc)
        fixed = np.ascontiguousarray(bc.fixed_dofs, dtype=np.int32)
        ld = np.ascontiguousarray([d for d, _ in bc.point_loads], dtype=np.int32)
        lv = np.ascontiguousarray([v for _, v in bc.point_loads], dtype=np.float64)
        b = np.full(n, 7.0)
        from paper_2301_07457_b200._lib import dptr, iptr
        assert lib.tmg_inputs_rhs(g.nx, g.ny, iptr(fixed), len(fixed), iptr(ld), dptr(lv), len(lv), dptr(b)) == 1
        assert np.all(b == 7.0)


def test_host_length_checks_precede_device_work():
    """Length / shape checks of the Python mirror raise the reference's
    DimensionError before any device call (sparse.cpp:72-75, fem.cpp:286-289,
    fem.cpp:295-298, mto.cpp:65-70)."""
    import types

    g = P.GridLevel(4, 4)
    ops = types.SimpleNamespace(grid=g, lib=None, h=None)  # never reached
    b = np.zeros(g.dof_count())
    with pytest.raises(P.DimensionError, match="matvec: vector length 3 does not match matrix size 50"):
        P.pcgmg_solve(ops, b, P.SolverConfig(), x0=np.zeros(3))
    with pytest.raises(P.DimensionError, match="compliance: vector length 5"):
        P.compliance(ops, np.zeros(5))
    with pytest.raises(P.DimensionError, match="element_energies: vector length 5"):
        P.element_energies(ops, np.zeros(5))
    mat = P.MaterialModel()
    with pytest.raises(P.DimensionError, match="sensitivities: density grid does not match level"):
        P.sensitivities(ops, np.zeros((15, 4)), mat)
    with pytest.raises(P.DimensionError, match="sensitivities: phase count mismatch"):
        P.sensitivities(ops, np.zeros((16, 3)), mat)
    with pytest.raises(P.DimensionError, match="element_energies: vector length 9"):
        P.sensitivities(ops, np.zeros((16, 4)), mat, u=np.zeros(9))
    with pytest.raises(P.DimensionError, match="filter: density grid does not match level"):
        P.filter_sensitivities(ops, np.zeros(16), np.zeros((15, 4)), 0, 1.5)
