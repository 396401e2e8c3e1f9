"""Shared problem builders for the parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

import paper_2301_07457_b200 as P
from oracle import pyoracle as po

MAT = P.MaterialModel(phase_moduli=[1.0, 0.5, 0.2, 1e-9], poisson_ratio=0.3, penalty=3.0)


def moduli(nx, ny, recipe="iid", seed=0):
    if recipe == "iid":
        a = P.density_iid(nx, ny, seed)
    elif recipe == "checker":
        a = P.density_checker(nx, ny, max(1, min(16, nx // 4)), seed)
    elif recipe == "uniform":
        a = np.tile(np.array([0.15, 0.15, 0.15, 0.55]), (nx * ny, 1))
    else:
        raise ValueError(recipe)
    return a, P.effective_moduli(a, MAT)


def checker(kind="orc"):
    if kind == "ref" and not po.available("ref"):
        return None
    return kind


def pair(nx, ny, nc, recipe="iid", seed=0, load="uniform", omega=0.6, kind="orc", bc=None, nu=0.3):
    """(GPU operators, CPU checker system, rhs, alpha, E) on identical inputs."""
    a, E = moduli(nx, ny, recipe, seed)
    g = P.GridLevel(nx, ny)
    if bc is None:
        bc = P.wall_boundary_conditions(g, load)
    ops = P.MultigridOperators(g, nc, nu, bc)
    ops.set_moduli(E, omega)
    sysc = po.System(kind, nx, ny, E, nu, bc.fixed_dofs, bc.point_loads).build_mg(nc, omega)
    b = sysc.rhs()
    return ops, sysc, b, a, E


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
