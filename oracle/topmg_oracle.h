/*
 * TEST INFRASTRUCTURE ONLY -- the CPU checker for the GPU pCGMG path.
 *
 * Plain-C restatement of the reference topopt-mg solve path (all file:line
 * citations are relative to /root/reference/proj). Only tests/, the smoke()
 * check in __graft_entry__.py and bench.py's cpu_baseline / --impl reference
 * legs may load liboracle.so. The product library (paper_2301_07457_b200/)
 * never links it and has no CPU fallback.
 *
 * Parity pin: every routine is checked against the unmodified reference
 * (oracle/_ref/libtopmg_ref.so, built from the reference's own sources) and
 * against the golden fixtures in tests/golden/ that were generated from it
 * (tests/golden/make_golden.py). Because the restatement performs the same
 * floating-point operations in the same order (same loop nesting, sequential
 * dots, stable assembly summation order, envelope Cholesky, -ffp-contract=off)
 * the pinned results are bit-identical, not merely close.
 *
 * Function set and signatures mirror oracle/ref_shim.cpp (prefix ref_).
 * Status codes follow include/tmg_gpu.h (0 ok, 1 config, 2 dimension,
 * 3 definiteness, 4 preconditioner, 5 splitting, 8 multiplier).
 */
#ifndef TOPMG_ORACLE_H
#define TOPMG_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

/* fem.cpp:131-169 */
void orc_element_stiffness(double modulus, double nu, double* out64);

/* fem.cpp:181-219 (+ finish_assembly fem.cpp:89-106, from_triplets
 * sparse.cpp:12-52). Returns an opaque system; *status != 0 on error. */
void* orc_system_create(int nx, int ny, const double* moduli, double nu,
                        const int* fixed, int n_fixed, const int* load_dofs,
                        const double* load_vals, int n_loads, char* err,
                        int errlen, int* status);
/* grid.cpp:53-96 + solvers.cpp:460-481 */
int orc_system_build_mg(void* h, int num_coarsenings, double omega, char* err,
                        int errlen, int* row);
int orc_system_num_levels(void* h);
void orc_system_rhs(void* h, double* out);
long orc_system_level_nnz(void* h, int level);
int orc_system_level_size(void* h, int level);
int orc_system_level_csr(void* h, int level, int* offsets, int* cols, double* vals);
/* sparse.cpp:70-86 on the level's matrix (level 0 = coarsest) */
int orc_system_matvec(void* h, int level, const double* x, double* y);
/* solvers.cpp:483-514 at the finest level, u updated in place */
int orc_system_vcycle(void* h, const double* f, double* u, int gamma, int pre, int post);
/* solvers.cpp:516-530 -> pcg_solve solvers.cpp:332-395 */
int orc_system_solve(void* h, const double* b, const double* x0, double tol,
                     int max_iter, int gamma, int pre, int post, double* x,
                     int* iters, double* final_relres, int* converged,
                     double* hist, int* hist_len, char* err, int errlen);
void orc_system_times(void* h, double* out3);
/* fem.cpp:284-290 */
double orc_system_compliance(void* h, const double* u);
void orc_system_destroy(void* h);

/* fem.cpp:292-318 */
int orc_element_energies(int nx, int ny, const double* u, double nu, double* out);
/* BASELINE densities with the reference's oracle::Rng recipe
 * (tests/oracles.hpp:15-36): iid fractions and the c2
 * checkerboard, element-major [nx*ny][nphases] */
void orc_density_iid(int nx, int ny, int nmat, unsigned long long seed, double* alpha);
void orc_density_checker(int nx, int ny, int block, int nphases, unsigned long long seed, double* alpha);
/* density.cpp:68-85 */
void orc_effective_moduli(int nx, int ny, int nphases, const double* alpha,
                          const double* phase_moduli, double penalty, double* out);
/* mto.cpp:61-85; out is phase-major [nphases][nx*ny] */
int orc_sensitivities(int nx, int ny, int nphases, const double* alpha,
                      const double* phase_moduli, double penalty, double nu,
                      const double* u, double* out);
/* mto.cpp:87-117 */
int orc_filter(int nx, int ny, int nphases, const double* alpha, int phase,
               double radius, const double* raw, double* out);
/* mto.cpp:142-227: in place on alpha[e * nphases + phase]; 8 = MultiplierError */
int orc_oc_update_pair(long ne, int nphases, double floor_eps, double* alpha, int phase_a,
                       int phase_b, const double* sens_a, const double* sens_b, double target,
                       const double* move, double damping);
/* fem.cpp:37-81: the Q4 Laplacian and mass element matrices (4x4 each) */
void orc_poisson_matrices(double* k16, double* m16);
/* assemble_poisson (fem.cpp:232-276), 1 dof per node, every boundary node
 * fixed; the returned system works with every orc_system_* call */
void* orc_poisson_create(int nx, int ny, const double* node_source, char* err, int errlen,
                         int* status);
/* optimize() with Method::pcgmg (mto.cpp:229-354); density [ne * np] out,
 * histories of up to max_outer entries */
int orc_optimize(int nx, int ny, int np, const double* phase_moduli, double penalty, double nu,
                 const int* fixed, int n_fixed, const int* load_dofs, const double* load_vals,
                 int n_loads, const double* fractions, double filter_radius, double filter_tol,
                 double tol, int inner_sweeps, double move_limit, double oc_damping, int warm_start,
                 int max_outer, double density_floor, int num_coarsenings, double omega,
                 double solver_tol, int solver_max_iter, int gamma, int pre, int post,
                 double* density, double* compliance_hist, double* change_hist, int* iters_hist,
                 int* outer_iterations, long* total_iters, int* converged, char* err, int errlen);

#ifdef __cplusplus
}
#endif
#endif
