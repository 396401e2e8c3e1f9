"""B200-native pCGMG for topopt-mg (arXiv 2301.07457).

The hot path -- the SIMP multi-material Q4 elasticity solve K(alpha) u = f by
CG preconditioned with a geometric-multigrid gamma-cycle, plus the compliance,
sensitivity and filter kernels that consume u -- runs as hand-written sm_100a
CUDA in ``libtmg_gpu.so`` behind the C ABI of ``include/tmg_gpu.h``. This
package is the Python mirror of the reference interface over that ABI.
"""
from .topmg import (  # noqa: F401
    BoundaryConditions,
    ConfigError,
    CudaError,
    DefinitenessError,
    DimensionError,
    GridLevel,
    MaterialModel,
    MultigridOperators,
    MultiplierError,
    NumericError,
    PreconditionerError,
    SolveReport,
    SolverConfig,
    SplittingError,
    assemble_rhs,
    build_multigrid_operators,
    compliance,
    density_checker,
    density_iid,
    effective_moduli,
    emit_outputs,
    element_energies,
    element_stiffness,
    filter_sensitivities,
    mg_cycle,
    nccl_unique_id,
    OptimConfig,
    OptimReport,
    oc_timings,
    optimize,
    oc_update_pair,
    pcgmg_solve,
    sensitivities,
    slab_partition,
    wall_boundary_conditions,
    write_composite_ppm,
    write_history_csv,
    write_phase_pgm,
    write_residual_csv,
)
