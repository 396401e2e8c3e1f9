/*
 * tmg_gpu.h -- C ABI of the B200-native pCGMG solve (libtmg_gpu.so).
 *
 * Drop-in boundary for the hot path of topopt-mg (arXiv 2301.07457): the
 * per-outer-iteration block of optimize() at proj/src/mto.cpp:267-310,
 *
 *     sys   = assemble_elasticity(grid, density, material, bc)   fem.cpp:221
 *     ops   = build_multigrid_operators(hier, sys.matrix, omega)  solvers.cpp:460
 *     solve = pcgmg_solve(ops, sys.rhs, cfg, x0)                  solvers.cpp:516
 *     C     = compliance(sys.matrix, u)                           fem.cpp:284
 *     raw   = sensitivities(u, density, material, grid)           mto.cpp:61
 *     filt  = filter_sensitivities(raw[i], density, i, r, grid)   mto.cpp:87
 *
 * The reference's solver boundary takes an assembled CSR matrix
 * (solvers.hpp:100-114). The GPU path is matrix-free, so the boundary sits one
 * level up: it takes what assemble_from_moduli takes (GridLevel, per-element
 * moduli, Poisson ratio, BoundaryConditions -- fem.hpp:14-19, 43-46) and
 * returns what pcgmg_solve returns (SolveReport -- solvers.hpp:29-36).
 *
 * Conventions
 *  - Every function returns a status (TMG_OK or one of the error codes below,
 *    which map 1:1 onto include/topmg/errors.hpp:9-47 of the reference).
 *    tmg_gpu_last_error() returns the message and, for TMG_ERR_DEFINITENESS,
 *    the failing row (DefinitenessError::row).
 *  - Host vectors use the reference layout: node (x, y) -> x*(ny+1) + y
 *    (column-major, grid.hpp:10-24), dof = 2*node + component; elements
 *    (ex, ey) -> ex*ny + ey. All arithmetic is IEEE fp64.
 *  - Level indices follow the reference: 0 = coarsest, num_coarsenings =
 *    finest (GridHierarchy::levels is coarsest-first, grid.hpp:47-56).
 *  - One handle = one GPU + one CUDA stream; a handle is not shareable
 *    between host threads mid-call. Results are
 *    deterministic run to run (fixed-order reductions, no fp atomics).
 *  - There is no CPU fallback: without a usable sm_100 device every call that
 *    needs the GPU returns TMG_ERR_CUDA.
 */
#ifndef TMG_GPU_H
#define TMG_GPU_H

#ifdef __cplusplus
extern "C" {
#endif

enum {
  TMG_OK = 0,
  TMG_ERR_CONFIG = 1,         /* topmg::ConfigError          errors.hpp:9   */
  TMG_ERR_DIMENSION = 2,      /* topmg::DimensionError       errors.hpp:14  */
  TMG_ERR_DEFINITENESS = 3,   /* topmg::DefinitenessError    errors.hpp:24  */
  TMG_ERR_PRECONDITIONER = 4, /* topmg::PreconditionerError  errors.hpp:36  */
  TMG_ERR_SPLITTING = 5,      /* topmg::SplittingError       errors.hpp:31  */
  TMG_ERR_CUDA = 6,           /* device / driver failure (no reference twin) */
  TMG_ERR_NCCL = 7,           /* multi-GPU transport failure               */
  TMG_ERR_MULTIPLIER = 8      /* topmg::MultiplierError      errors.hpp:41  */
};

typedef struct tmg_gpu_handle tmg_gpu_handle;

/* ---- lifecycle ------------------------------------------------------- */

/* Replaces build_hierarchy(nx, ny, num_coarsenings, 2) (grid.cpp:53-96) and
 * the device allocation for all levels. Same ConfigError cases: nx, ny >= 1,
 * num_coarsenings >= 0, divisibility by 2^num_coarsenings. dofs_per_node must
 * be 2 (plane elasticity). device = CUDA ordinal. Limit (no reference twin):
 * the coarsest level, solved through a dense explicit inverse, may have at
 * most 16900 dofs, i.e. 2 (nx/2^nc + 1)(ny/2^nc + 1) <= 16900 (ConfigError
 * otherwise). Every BASELINE configuration coarsens to 8x8 = 162 dofs; the
 * reference default num_coarsenings = 2 (solvers.hpp:25) stays inside the
 * limit up to 256x256 or 512x256 elements. Above 2048 dofs the band is
 * factored in L2 by one CTA and the handle holds three dense n x n arrays;
 * such a level may have columns of at most 148 nodes (ny/2^nc + 1 <= 148,
 * ConfigError otherwise), which keeps the factor around a second. */
int tmg_gpu_create(int nx, int ny, int num_coarsenings, int dofs_per_node,
                   int device, tmg_gpu_handle** out);
void tmg_gpu_destroy(tmg_gpu_handle* h);

/* ---- x-slab decomposition (multi-GPU) ---------------------------------- */
/* The mesh is split into x-slabs: contiguous node-column ranges of the
 * reference's column-major numbering (grid.hpp:19). Every level finer than
 * `replicated_level` is distributed (one ghost column exchanged per pass, two
 * before the fused restriction); levels 0..replicated_level are assembled on
 * every rank and solved redundantly. replicated_level = -1 picks the finest
 * level at which a slab would hold fewer than 16 node columns. Slab
 * boundaries are multiples of 2^(num_coarsenings - replicated_level) fine
 * columns and of the fine-level reduction tile width (8..64 columns, from
 * nx and ny). Reductions sum per-tile partials of a global tile layout in one
 * fixed order, so every partition (1..N ranks) gives bitwise the same PCG
 * scalars, iterates and solution as the single-rank solve. */

/* x0s[r] = first fine node column of rank r (nranks + 1 entries, the last is
 * nx + 1); *rep_out = the replicated level used. Host-only. */
int tmg_partition(int nx, int ny, int num_coarsenings, int nranks, int replicated_level, int* x0s, int* rep_out);
/* One process, `nslabs` ranks on one device: the decomposition run end to end
 * on a single GPU (halo exchange by device copies). */
int tmg_gpu_create_local_slabs(int nx, int ny, int num_coarsenings, int dofs_per_node, int device, int nslabs,
                               int replicated_level, tmg_gpu_handle** out);
/* One rank per process (torchrun): exchanges by NCCL send/recv/broadcast and
 * all-reduce over NVLink / NVSwitch. nccl_unique_id: the 128-byte
 * ncclUniqueId created by rank 0 with tmg_nccl_unique_id and shared by the
 * caller. Host vectors passed to this handle are global; each rank reads and
 * writes only its own columns. nranks = 1 is allowed: the slab machinery
 * (all-reduced partials, halo calls, replicated coarse levels) then runs
 * through a one-rank communicator and solves bitwise like tmg_gpu_create. */
int tmg_gpu_create_nccl(int nx, int ny, int num_coarsenings, int dofs_per_node, int device, int nranks, int rank,
                        const void* nccl_unique_id, int replicated_level, tmg_gpu_handle** out);
int tmg_nccl_unique_id(void* out128);
/* Message of the last failing call; *row = DefinitenessError::row or -1. */
int tmg_gpu_last_error(tmg_gpu_handle* h, char* buf, int len, int* row);

/* ---- problem data (what assemble_from_moduli consumes, fem.cpp:181) --- */

/* Poisson ratio (-> unit-modulus Ke of element_stiffness, fem.cpp:131-169)
 * and the homogeneous Dirichlet dofs (BoundaryConditions::fixed_dofs,
 * validated like BoundaryConditions::validate, fem.cpp:110-129; a dof listed
 * k times gets diagonal k exactly like finish_assembly, fem.cpp:89-106). */
int tmg_gpu_set_problem(tmg_gpu_handle* h, double nu, const int* fixed_dofs,
                        int n_fixed);

/* Per-element moduli (host, nx*ny, the output of effective_moduli,
 * density.cpp:78-85) -> device; then tmg_gpu_setup(). Together these replace
 * assemble_from_moduli + build_multigrid_operators (mto.cpp:267-281):
 * the fine operator is never assembled; the Galerkin hierarchy (1/4)P^T A P
 * (solvers.cpp:397-458) and the coarsest factor (solvers.cpp:89-152) are built
 * on the device. omega is fixed here, like MultigridOperators::omega
 * (solvers.hpp:98, solvers.cpp:471). */
int tmg_gpu_set_moduli(tmg_gpu_handle* h, const double* moduli, long n_elem,
                       double omega);
int tmg_gpu_upload_moduli(tmg_gpu_handle* h, const double* moduli, long n_elem);
int tmg_gpu_setup(tmg_gpu_handle* h, double omega);

/* SIMP on the device (density.cpp:68-85): alpha element-major
 * [nx*ny][nphases] (DensityField layout, density.hpp:49-54), then setup. */
int tmg_gpu_set_density(tmg_gpu_handle* h, const double* alpha, int nphases,
                        const double* phase_moduli, double penalty, double omega);

/* ---- solve (pcgmg_solve, solvers.cpp:516-530 / pcg_solve 332-395) ------ */

/* b: host rhs (2N). x0: host warm start or NULL (mto.cpp:270-271).
 * x_out: host solution (2N). history: residual_history (entry 0 = initial
 * relative residual), capacity history_cap (>= max_iter + 1 recommended);
 * *history_len = entries written. seconds = PCG time (SolveReport::seconds,
 * setup excluded as in solvers.cpp:335, 393). Non-convergence is
 * *converged = 0, not an error. pre != post -> TMG_ERR_CONFIG
 * (solvers.cpp:518-521). zr <= 0 -> TMG_ERR_PRECONDITIONER, pAp <= 0 ->
 * TMG_ERR_DEFINITENESS (solvers.cpp:362-380). */
int tmg_gpu_solve(tmg_gpu_handle* h, const double* b, const double* x0,
                  double tol, int max_iter, int gamma, int pre_sweeps,
                  int post_sweeps, double* x_out, int* iterations,
                  double* final_residual, int* converged, double* seconds,
                  double* history, int history_cap, int* history_len);

/* Device-resident variant: rhs / warm start already uploaded with
 * tmg_gpu_upload_rhs / tmg_gpu_upload_x0; the solution stays on the device
 * (tmg_gpu_download_solution fetches it). use_x0 != 0 uses the uploaded x0. */
int tmg_gpu_upload_rhs(tmg_gpu_handle* h, const double* b);
int tmg_gpu_upload_x0(tmg_gpu_handle* h, const double* x0);
int tmg_gpu_solve_resident(tmg_gpu_handle* h, int use_x0, double tol,
                           int max_iter, int gamma, int pre_sweeps,
                           int post_sweeps, int* iterations,
                           double* final_residual, int* converged,
                           double* seconds, double* history, int history_cap,
                           int* history_len);
int tmg_gpu_download_solution(tmg_gpu_handle* h, double* x_out);
/* Promote the resident solution to the warm start of the next solve. */
int tmg_gpu_solution_to_x0(tmg_gpu_handle* h);

/* ---- pipelined solves (serving a stream of independent problems) ------- */

/* The blocking tmg_gpu_set_moduli + tmg_gpu_solve pair moves 24 B of inputs
 * per element+node over PCIe before each solve and 16 B per node after it,
 * with the device idle. These three calls overlap those copies with the
 * previous / next solve on a second (copy) stream, for callers that solve
 * many independent problems on one mesh (the same outer loop as
 * mto.cpp:264-310 with the inputs supplied per call):
 *
 *   stage(0, E_0, b_0)
 *   for k: stage((k+1)&1, E_{k+1}, b_{k+1});   (returns at once)
 *          solve_staged(k&1, ..., u_k)         (blocks until the iteration
 *                                               count is known; u_k arrives
 *                                               during the next solve)
 *   sync_outputs()                             (every u_k is on the host)
 *
 * tmg_gpu_stage_inputs copies moduli (nx*ny, element order of
 * tmg_gpu_upload_moduli) and b (2N) into staging slot 0 or 1 on the copy
 * stream, after the slot's previous contents were installed. Host buffers
 * must be PINNED (tmg_host_alloc) for the copies to overlap; pageable
 * memory still works, synchronously. The host arrays are read while the
 * copies run: keep them unchanged until the slot's tmg_gpu_solve_staged
 * returns.
 *
 * tmg_gpu_solve_staged installs the slot's inputs, builds the hierarchy with
 * omega (tmg_gpu_setup) and solves from x0 = 0 exactly like tmg_gpu_solve
 * (same outputs and errors); x_out (2N, pinned) is written asynchronously
 * and is complete after tmg_gpu_sync_outputs (call it before reading).
 * Results are bitwise those of tmg_gpu_set_moduli + tmg_gpu_solve. */
int tmg_gpu_stage_inputs(tmg_gpu_handle* h, int slot, const double* moduli,
                         long n_elem, const double* b);
int tmg_gpu_solve_staged(tmg_gpu_handle* h, int slot, double omega, double tol,
                         int max_iter, int gamma, int pre_sweeps,
                         int post_sweeps, double* x_out, int* iterations,
                         double* final_residual, int* converged,
                         double* seconds, double* history, int history_cap,
                         int* history_len);
int tmg_gpu_sync_outputs(tmg_gpu_handle* h);

/* ---- consumers of u (mto.cpp:300-310) ---------------------------------- */

/* u^T K u with the eliminated operator (fem.cpp:284-290). u = NULL uses the
 * resident solution. */
int tmg_gpu_compliance(tmg_gpu_handle* h, const double* u, double* out);
/* u_e^T khat u_e per element, khat = unit-modulus Ke (fem.cpp:292-318). */
int tmg_gpu_element_energies(tmg_gpu_handle* h, const double* u, double* out);
/* dC/dalpha = -p alpha^(p-1) E0 u_e^T khat u_e for every phase (mto.cpp:61-85);
 * out is phase-major [nphases][nx*ny] like the reference's vector of vectors. */
int tmg_gpu_sensitivities(tmg_gpu_handle* h, const double* u, int nphases,
                          const double* alpha, const double* phase_moduli,
                          double penalty, double* out);
/* Density-weighted cone sensitivity filter of one phase (mto.cpp:87-117);
 * radius <= 1 returns raw unchanged. */
int tmg_gpu_filter(tmg_gpu_handle* h, int nphases, const double* alpha, int phase,
                   double radius, const double* raw, double* out);

/* One OC exchange between phases a and b of the element-major density
 * alpha[e * nphases + phase] (host, updated in place), replacing
 * oc_update_pair (mto.cpp:142-227, mto.hpp:73-77): move[e] is the element's
 * move limit, floor_eps the density floor (DensityField::floor_eps). The
 * bisection for the volume multiplier runs on the device with deterministic
 * reductions. TMG_ERR_MULTIPLIER (alpha unchanged) when the target is missed
 * after 101 steps, TMG_ERR_CONFIG for phase_a == phase_b. Single-rank
 * handles. */
int tmg_gpu_oc_update_pair(tmg_gpu_handle* h, double* alpha, int nphases, double floor_eps,
                           int phase_a, int phase_b, const double* sens_a, const double* sens_b,
                           double target, const double* move, double damping);
/* OptimConfig (mto.hpp:12-27) with Method::pcgmg, flattened; Poisson's ratio
 * is the handle's (tmg_gpu_set_problem). */
typedef struct {
  int nphases;
  const double* phase_moduli;     /* MaterialModel::phase_moduli [nphases] */
  double penalty;                 /* MaterialModel::penalty */
  const double* volume_fractions; /* [nphases] */
  double filter_radius, filter_tol, tol;
  int inner_sweeps;
  double move_limit, oc_damping;
  int warm_start, max_outer;
  double density_floor;
  double solver_tol;              /* SolverConfig */
  int solver_max_iter, gamma, pre_sweeps, post_sweeps;
  double omega;
} tmg_optim_config;

/* The whole optimizer, optimize() with Method::pcgmg (mto.cpp:229-354), with
 * every per-iteration step on the device: effective moduli + Galerkin
 * setup, the warm-startable solve, compliance, sensitivities, the filter,
 * the OC pair sweeps, the move-limit adaptation and the max-change test.
 * rhs: the load vector (fixed dofs zero). Outputs mirror OptimReport: the
 * final element-major density [ne * nphases] and per outer iteration the
 * compliance, max density change, solver iterations and seconds (arrays of
 * max_outer entries). Single-rank handles. */
int tmg_gpu_optimize(tmg_gpu_handle* h, const tmg_optim_config* cfg, const double* rhs,
                     double* density_out, double* compliance_hist, double* change_hist,
                     int* iters_hist, double* seconds_hist, int* outer_iterations,
                     long* total_solver_iterations, int* converged, double* seconds);
/* Device time (ms) and bisection steps of the last tmg_gpu_oc_update_pair. */
int tmg_gpu_oc_timings(tmg_gpu_handle* h, double* device_ms, int* steps);

/* ---- kernel-level entry points (parity tests, profiling) --------------- */

/* y = A_level x (SparseSymMatrix::multiply on ops.matrices[level],
 * sparse.cpp:70-86). Host vectors of the level's dof count. */
int tmg_gpu_apply(tmg_gpu_handle* h, int level, const double* x, double* y);
/* Fills vals[] for a CSR pattern (offsets/cols of level `level`, reference
 * dof numbering) from the device operator -- compares the Galerkin hierarchy
 * entry by entry with galerkin_coarse_matrix (solvers.cpp:397-458). */
int tmg_gpu_level_values(tmg_gpu_handle* h, int level, const int* offsets,
                         const int* cols, double* vals);
/* One gamma-cycle at the finest level, u in/out (mg_cycle, solvers.cpp:483). */
int tmg_gpu_vcycle(tmg_gpu_handle* h, const double* f, double* u, int gamma,
                   int pre_sweeps, int post_sweeps);
/* prolongate / restrict between level-1 and level (grid.cpp:98-142). */
int tmg_gpu_prolongate(tmg_gpu_handle* h, int level, const double* coarse, double* fine);
int tmg_gpu_restrict(tmg_gpu_handle* h, int level, const double* fine, double* coarse);
/* `sweeps` damped-Jacobi sweeps at `level` (jacobi_sweep, solvers.cpp:30-37). */
int tmg_gpu_smooth(tmg_gpu_handle* h, int level, const double* f, double* u, int sweeps);

/* ---- instrumentation -------------------------------------------------- */

/* cudaStream_t of the handle (as void*). */
void* tmg_gpu_stream(tmg_gpu_handle* h);
/* Number of kernels this library has launched through the handle (graph
 * nodes counted per replay). */
long tmg_gpu_launch_count(tmg_gpu_handle* h);
/* Times `reps` back-to-back launches of one fine-level kernel on resident
 * data with CUDA events on the handle's stream. which: 0 = K.u apply,
 * 1 = damped-Jacobi sweep, 2 = the fused PCG update + two pre-sweeps (the
 * solve's dominant pass; scratch outputs, needs a prior solve). *avg_ms =
 * mean launch duration, *bytes = the kernel's algorithmic bytes per launch
 * (DESIGN.md). */
int tmg_gpu_time_kernel(tmg_gpu_handle* h, int which, int reps, double* avg_ms,
                        double* bytes);
/* Breakdown of the last resident solve: setup ms, pcg ms (device events). */
int tmg_gpu_last_timings(tmg_gpu_handle* h, double* setup_ms, double* pcg_ms);
/* CUDA events on the handle's stream (slots 0..7) for callers that time a
 * region of library calls on the launching stream. */
int tmg_gpu_event_record(tmg_gpu_handle* h, int slot);
int tmg_gpu_event_elapsed(tmg_gpu_handle* h, int slot_a, int slot_b, double* ms);
/* Page-locked host buffers for host<->device copies at full PCIe/C2C rate. */
void* tmg_host_alloc(unsigned long bytes);
void tmg_host_free(void* p);

/* ---- host-side input producers (tmg_inputs.cpp) ------------------------ */

void tmg_element_stiffness(double modulus, double nu, double* ke64);
void tmg_inputs_effective_moduli(long n_elem, int nphases, const double* alpha,
                                 const double* phase_moduli, double penalty,
                                 double* out);
void tmg_inputs_density_iid(int nx, int ny, int nmat, unsigned long long seed,
                            double* alpha);
void tmg_inputs_density_checker(int nx, int ny, int block, int nphases,
                                unsigned long long seed, double* alpha);
void tmg_inputs_wall_bc(int nx, int ny, int load_mode, int* fixed, int* n_fixed,
                        int* load_dofs, double* load_vals, int* n_loads);
/* BoundaryConditions::validate (fem.cpp:110-129) + the rhs of
 * assemble_from_moduli (fem.cpp:214-218): TMG_ERR_CONFIG for a dof outside
 * [0, 2(nx+1)(ny+1)) or a dof both fixed and loaded (b untouched) */
int tmg_inputs_rhs(int nx, int ny, const int* fixed, int n_fixed,
                   const int* load_dofs, const double* load_vals, int n_loads,
                   double* b);
/* poisson_element_matrix / poisson_mass_matrix (fem.cpp:37-81), row-major 4x4 */
void tmg_poisson_element_matrices(double* k16, double* m16);
/* the right-hand side of assemble_poisson (fem.cpp:243-276) for a per-node
 * source: -M f assembled, boundary entries 0 */
void tmg_inputs_poisson_rhs(int nx, int ny, const double* node_source, double* b);

/* ---- Poisson pCGMG (tmg_poisson.cuh) -------------
 * -lap(u) = -f on an nx x ny Q4 grid, 1 dof per node, every boundary node
 * fixed (assemble_poisson, fem.cpp:232-276), solved by pcgmg_solve
 * (solvers.cpp:516-530) with the Galerkin hierarchy of
 * build_multigrid_operators (solvers.cpp:460-481) over
 * build_hierarchy(nx, ny, num_coarsenings, 1). Single GPU. */
typedef struct tmg_poisson_handle tmg_poisson_handle;
int tmg_poisson_create(int nx, int ny, int num_coarsenings, int device,
                       tmg_poisson_handle** out);
void tmg_poisson_destroy(tmg_poisson_handle* h);
int tmg_poisson_last_error(tmg_poisson_handle* h, char* buf, int len);
/* assembles the fine operator on the device, the Galerkin levels and the
 * coarsest inverse; omega is the Jacobi damping of the cycle */
int tmg_poisson_setup(tmg_poisson_handle* h, double omega);
/* level operator as 5 node-major planes (centre, N, SE, E, NE), each
 * (nx_l+1)(ny_l+1) doubles in the reference node order */
int tmg_poisson_level_values(tmg_poisson_handle* h, int level, double* planes);
/* mg_cycle (solvers.cpp:483-514) at the finest level, u updated in place */
int tmg_poisson_vcycle(tmg_poisson_handle* h, const double* f, double* u, int gamma,
                       int pre_sweeps, int post_sweeps);
/* pcgmg_solve with x0 (nullable); hist gets up to hist_cap entries */
int tmg_poisson_solve(tmg_poisson_handle* h, const double* b, const double* x0, double tol,
                      int max_iter, int gamma, int pre_sweeps, int post_sweeps, double* x,
                      int* iterations, double* final_relres, int* converged, double* seconds,
                      double* hist, int hist_cap, int* hist_len);

#ifdef __cplusplus
}
#endif
#endif /* TMG_GPU_H */
