// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// C-ABI shim over the UNMODIFIED reference library (topopt-mg, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It lets the
// pytest suite, tests/golden/make_golden.py and bench.py's cpu_baseline /
// --impl reference leg drive the reference's own code path:
//   assemble_from_moduli      (proj/src/fem.cpp:181-219)
//   build_hierarchy           (proj/src/grid.cpp:53-96)
//   build_multigrid_operators (proj/src/solvers.cpp:460-481)
//   mg_cycle / pcgmg_solve    (proj/src/solvers.cpp:483-530)
//   compliance / element_energies (proj/src/fem.cpp:284-318)
//   sensitivities / filter_sensitivities (proj/src/mto.cpp:61-117)
// The function set and signatures are identical to oracle/topmg_oracle.h with
// the prefix ref_ instead of orc_, so tests can swap one checker for the other.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "topmg/density.hpp"
#include "topmg/errors.hpp"
#include "topmg/fem.hpp"
#include "topmg/grid.hpp"
#include "topmg/mto.hpp"
#include "topmg/report.hpp"
#include "topmg/solvers.hpp"
#include "topmg/sparse.hpp"
// the reference test suite's deterministic generator (tests/oracles.hpp:15-36):
// its bit recipe defines the BASELINE densities
#include "oracles.hpp"

namespace {

using Clock = std::chrono::steady_clock;

struct RefSystem {
  topmg::GridLevel grid;
  topmg::LinearSystem sys;
  topmg::GridHierarchy hier;
  std::unique_ptr<topmg::MultigridOperators> ops;
  double nu = 0.3;
  double t_assemble = 0.0, t_setup = 0.0, t_pcg = 0.0;
};

void put_err(char* err, int len, const char* msg) {
  if (err && len > 0) {
    std::snprintf(err, static_cast<std::size_t>(len), "%s", msg);
  }
}

// Maps the reference exception hierarchy (include/topmg/errors.hpp:9-47) onto
// the status codes of include/tmg_gpu.h.
int map_exception(char* err, int len, int* row) {
  try {
    throw;
  } catch (const topmg::ConfigError& e) {
    put_err(err, len, e.what());
    return 1;
  } catch (const topmg::DimensionError& e) {
    put_err(err, len, e.what());
    return 2;
  } catch (const topmg::DefinitenessError& e) {
    put_err(err, len, e.what());
    if (row) *row = e.row;
    return 3;
  } catch (const topmg::PreconditionerError& e) {
    put_err(err, len, e.what());
    return 4;
  } catch (const topmg::SplittingError& e) {
    put_err(err, len, e.what());
    return 5;
  } catch (const topmg::MultiplierError& e) {
    put_err(err, len, e.what());
    return 8;
  } catch (const std::exception& e) {
    put_err(err, len, e.what());
    return 9;
  }
}

const topmg::SparseSymMatrix& level_matrix(const RefSystem* s, int level) {
  if (s->ops) return s->ops->matrices.at(static_cast<std::size_t>(level));
  if (level != 0) throw topmg::DimensionError("no multigrid operators built");
  return s->sys.matrix;
}

}  // namespace

extern "C" {

void ref_element_stiffness(double modulus, double nu, double* out64) {
  const topmg::ElementMatrix k = topmg::element_stiffness(modulus, nu);
  std::memcpy(out64, k.data(), 64 * sizeof(double));
}

void* ref_system_create(int nx, int ny, const double* moduli, double nu,
                        const int* fixed, int n_fixed, const int* load_dofs,
                        const double* load_vals, int n_loads, char* err,
                        int errlen, int* status) {
  try {
    auto s = std::make_unique<RefSystem>();
    s->grid = topmg::GridLevel{nx, ny, 2, 0};
    s->nu = nu;
    topmg::BoundaryConditions bc;
    bc.fixed_dofs.assign(fixed, fixed + n_fixed);
    for (int i = 0; i < n_loads; ++i) bc.point_loads.emplace_back(load_dofs[i], load_vals[i]);
    std::vector<double> e(moduli, moduli + static_cast<std::size_t>(nx) * ny);
    const auto t0 = Clock::now();
    s->sys = topmg::assemble_from_moduli(s->grid, e, nu, bc);
    s->t_assemble = std::chrono::duration<double>(Clock::now() - t0).count();
    *status = 0;
    return s.release();
  } catch (...) {
    *status = map_exception(err, errlen, nullptr);
    return nullptr;
  }
}

// assemble_poisson (fem.cpp:232-276): the Poisson system on a 1-dof grid
void* ref_poisson_create(int nx, int ny, const double* source, char* err, int errlen, int* status) {
  try {
    auto s = std::make_unique<RefSystem>();
    s->grid = topmg::GridLevel{nx, ny, 1, 0};
    std::vector<double> f(source, source + static_cast<std::size_t>(nx + 1) * (ny + 1));
    const auto t0 = Clock::now();
    s->sys = topmg::assemble_poisson(s->grid, f);
    s->t_assemble = std::chrono::duration<double>(Clock::now() - t0).count();
    *status = 0;
    return s.release();
  } catch (...) {
    *status = map_exception(err, errlen, nullptr);
    return nullptr;
  }
}

int ref_system_build_mg(void* h, int num_coarsenings, double omega, char* err,
                        int errlen, int* row) {
  auto* s = static_cast<RefSystem*>(h);
  try {
    s->hier = topmg::build_hierarchy(s->grid.nx, s->grid.ny, num_coarsenings, s->grid.dofs_per_node);
    const auto t0 = Clock::now();
    s->ops = std::make_unique<topmg::MultigridOperators>(
        topmg::build_multigrid_operators(s->hier, s->sys.matrix, omega));
    s->t_setup = std::chrono::duration<double>(Clock::now() - t0).count();
    return 0;
  } catch (...) {
    s->ops.reset();
    return map_exception(err, errlen, row);
  }
}

int ref_system_num_levels(void* h) {
  auto* s = static_cast<RefSystem*>(h);
  return s->ops ? static_cast<int>(s->ops->matrices.size()) : 1;
}

void ref_system_rhs(void* h, double* out) {
  auto* s = static_cast<RefSystem*>(h);
  std::memcpy(out, s->sys.rhs.data(), s->sys.rhs.size() * sizeof(double));
}

long ref_system_level_nnz(void* h, int level) {
  try {
    return static_cast<long>(level_matrix(static_cast<RefSystem*>(h), level).nnz());
  } catch (...) {
    return -1;
  }
}

int ref_system_level_size(void* h, int level) {
  try {
    return level_matrix(static_cast<RefSystem*>(h), level).size();
  } catch (...) {
    return -1;
  }
}

int ref_system_level_csr(void* h, int level, int* offsets, int* cols, double* vals) {
  try {
    const topmg::SparseSymMatrix& m = level_matrix(static_cast<RefSystem*>(h), level);
    std::memcpy(offsets, m.row_offsets().data(), m.row_offsets().size() * sizeof(int));
    std::memcpy(cols, m.col_indices().data(), m.col_indices().size() * sizeof(int));
    std::memcpy(vals, m.values().data(), m.values().size() * sizeof(double));
    return 0;
  } catch (...) {
    return 2;
  }
}

int ref_system_matvec(void* h, int level, const double* x, double* y) {
  try {
    const topmg::SparseSymMatrix& m = level_matrix(static_cast<RefSystem*>(h), level);
    std::vector<double> xv(x, x + m.size()), yv;
    m.multiply(xv, yv);
    std::memcpy(y, yv.data(), yv.size() * sizeof(double));
    return 0;
  } catch (...) {
    return 2;
  }
}

int ref_system_vcycle(void* h, const double* f, double* u, int gamma, int pre,
                      int post) {
  auto* s = static_cast<RefSystem*>(h);
  if (!s->ops) return 2;
  const int n = s->grid.dof_count();
  std::vector<double> fv(f, f + n), uv(u, u + n);
  topmg::mg_cycle(*s->ops, s->hier.finest(), uv, fv, gamma, pre, post);
  std::memcpy(u, uv.data(), static_cast<std::size_t>(n) * sizeof(double));
  return 0;
}

int ref_system_solve(void* h, const double* b, const double* x0, double tol,
                     int max_iter, int gamma, int pre, int post, double* x,
                     int* iters, double* final_relres, int* converged,
                     double* hist, int* hist_len, char* err, int errlen) {
  auto* s = static_cast<RefSystem*>(h);
  if (!s->ops) {
    put_err(err, errlen, "multigrid operators not built");
    return 2;
  }
  try {
    const int n = s->grid.dof_count();
    std::vector<double> bv(b, b + n), x0v;
    if (x0) x0v.assign(x0, x0 + n);
    topmg::SolverConfig cfg;
    cfg.method = topmg::Method::pcgmg;
    cfg.tol = tol;
    cfg.max_iter = max_iter;
    cfg.omega = s->ops->omega;
    cfg.gamma = gamma;
    cfg.pre_sweeps = pre;
    cfg.post_sweeps = post;
    cfg.num_coarsenings = s->hier.finest();
    const topmg::SolveReport rep = topmg::pcgmg_solve(*s->ops, bv, cfg, x0 ? &x0v : nullptr);
    std::memcpy(x, rep.solution.data(), rep.solution.size() * sizeof(double));
    *iters = rep.iterations;
    *final_relres = rep.final_residual;
    *converged = rep.converged ? 1 : 0;
    std::memcpy(hist, rep.residual_history.data(),
                rep.residual_history.size() * sizeof(double));
    *hist_len = static_cast<int>(rep.residual_history.size());
    s->t_pcg = rep.seconds;
    return 0;
  } catch (...) {
    return map_exception(err, errlen, nullptr);
  }
}

// seconds of the last assemble / build_multigrid_operators / pcgmg_solve
void ref_system_times(void* h, double* out3) {
  auto* s = static_cast<RefSystem*>(h);
  out3[0] = s->t_assemble;
  out3[1] = s->t_setup;
  out3[2] = s->t_pcg;
}

double ref_system_compliance(void* h, const double* u) {
  auto* s = static_cast<RefSystem*>(h);
  std::vector<double> uv(u, u + s->grid.dof_count());
  return topmg::compliance(s->sys.matrix, uv);
}

void ref_system_destroy(void* h) { delete static_cast<RefSystem*>(h); }

int ref_element_energies(int nx, int ny, const double* u, double nu, double* out) {
  try {
    const topmg::GridLevel g{nx, ny, 2, 0};
    std::vector<double> uv(u, u + g.dof_count());
    const std::vector<double> e = topmg::element_energies(g, uv, nu);
    std::memcpy(out, e.data(), e.size() * sizeof(double));
    return 0;
  } catch (...) {
    return 2;
  }
}

namespace {
topmg::DensityField make_density(int nx, int ny, int nphases, const double* alpha) {
  topmg::DensityField d(nx, ny, nphases);
  for (int e = 0; e < nx * ny; ++e) {
    for (int i = 0; i < nphases; ++i) d.at(e, i) = alpha[static_cast<std::size_t>(e) * nphases + i];
  }
  return d;
}
}  // namespace

// BASELINE c1/c4 densities drawn with the reference's own
// oracle::Rng (oracles.hpp:21-23): element-major, nmat fractions U(0,1) per
// element, divided by their sum when it exceeds 1, void = remainder.
void ref_density_iid(int nx, int ny, int nmat, unsigned long long seed, double* alpha) {
  oracle::Rng rng(seed);
  const long ne = static_cast<long>(nx) * ny;
  for (long e = 0; e < ne; ++e) {
    double* a = alpha + e * (nmat + 1);
    double s = 0.0;
    for (int m = 0; m < nmat; ++m) {
      a[m] = rng.uniform();
      s += a[m];
    }
    if (s > 1.0) {
      for (int m = 0; m < nmat; ++m) a[m] /= s;
      s = 0.0;
      for (int m = 0; m < nmat; ++m) s += a[m];
    }
    const double v = 1.0 - s;
    a[nmat] = v > 0.0 ? v : 0.0;
  }
}

// BASELINE c2 checkerboard: block x block element tiles visited x-major, one
// phase per tile from oracle::Rng::index (oracles.hpp:24), one-hot alpha.
void ref_density_checker(int nx, int ny, int block, int nphases, unsigned long long seed, double* alpha) {
  oracle::Rng rng(seed);
  std::memset(alpha, 0, sizeof(double) * static_cast<std::size_t>(nx) * ny * nphases);
  for (int i = 0; i < (nx + block - 1) / block; ++i)
    for (int j = 0; j < (ny + block - 1) / block; ++j) {
      const int ph = rng.index(nphases);
      for (int ex = i * block; ex < nx && ex < (i + 1) * block; ++ex)
        for (int ey = j * block; ey < ny && ey < (j + 1) * block; ++ey)
          alpha[(static_cast<long>(ex) * ny + ey) * nphases + ph] = 1.0;
    }
}

void ref_effective_moduli(int nx, int ny, int nphases, const double* alpha,
                          const double* phase_moduli, double penalty, double* out) {
  const topmg::DensityField d = make_density(nx, ny, nphases, alpha);
  topmg::MaterialModel mat;
  mat.phase_moduli.assign(phase_moduli, phase_moduli + nphases);
  mat.penalty = penalty;
  const std::vector<double> e = topmg::effective_moduli(d, mat);
  std::memcpy(out, e.data(), e.size() * sizeof(double));
}

int ref_sensitivities(int nx, int ny, int nphases, const double* alpha,
                      const double* phase_moduli, double penalty, double nu,
                      const double* u, double* out) {
  try {
    const topmg::GridLevel g{nx, ny, 2, 0};
    const topmg::DensityField d = make_density(nx, ny, nphases, alpha);
    topmg::MaterialModel mat;
    mat.phase_moduli.assign(phase_moduli, phase_moduli + nphases);
    mat.penalty = penalty;
    mat.poisson_ratio = nu;
    std::vector<double> uv(u, u + g.dof_count());
    const auto s = topmg::sensitivities(uv, d, mat, g);
    for (int i = 0; i < nphases; ++i) {
      std::memcpy(out + static_cast<std::size_t>(i) * nx * ny, s[static_cast<std::size_t>(i)].data(),
                  s[static_cast<std::size_t>(i)].size() * sizeof(double));
    }
    return 0;
  } catch (...) {
    return 2;
  }
}

int ref_filter(int nx, int ny, int nphases, const double* alpha, int phase,
               double radius, const double* raw, double* out) {
  try {
    const topmg::GridLevel g{nx, ny, 2, 0};
    const topmg::DensityField d = make_density(nx, ny, nphases, alpha);
    std::vector<double> rv(raw, raw + static_cast<std::size_t>(nx) * ny);
    const std::vector<double> f = topmg::filter_sensitivities(rv, d, phase, radius, g);
    std::memcpy(out, f.data(), f.size() * sizeof(double));
    return 0;
  } catch (...) {
    return 2;
  }
}

int ref_oc_update_pair(long ne, int nphases, double floor_eps, double* alpha, int phase_a, int phase_b,
                       const double* sens_a, const double* sens_b, double target, const double* move,
                       double damping) {
  try {
    topmg::DensityField d(static_cast<int>(ne), 1, nphases, floor_eps);
    for (long e = 0; e < ne; ++e)
      for (int i = 0; i < nphases; ++i) d.at(static_cast<int>(e), i) = alpha[e * nphases + i];
    const std::vector<double> a(sens_a, sens_a + ne), b(sens_b, sens_b + ne), mv(move, move + ne);
    topmg::oc_update_pair(d, phase_a, phase_b, a, b, target, mv, damping);
    std::memcpy(alpha, d.values().data(), sizeof(double) * static_cast<std::size_t>(ne) * nphases);
    return 0;
  } catch (...) {
    return map_exception(nullptr, 0, nullptr);
  }
}

int ref_optimize(int nx, int ny, int np, const double* pm, double penalty, double nu, const int* fixed, int n_fixed,
                 const int* load_dofs, const double* load_vals, int n_loads, const double* fractions,
                 double filter_radius, double filter_tol, double tol, int inner_sweeps, double move_limit,
                 double oc_damping, int warm_start, int max_outer, double density_floor, int num_coarsenings,
                 double omega, double solver_tol, int solver_max_iter, int gamma, int pre, int post,
                 double* density, double* compliance_hist, double* change_hist, int* iters_hist,
                 int* outer_iterations, long* total_iters, int* converged, char* err, int errlen) {
  try {
    topmg::Problem prob;
    prob.grid = topmg::GridLevel{nx, ny, 2, 0};
    prob.bc.fixed_dofs.assign(fixed, fixed + n_fixed);
    for (int k = 0; k < n_loads; ++k) prob.bc.point_loads.emplace_back(load_dofs[k], load_vals[k]);
    prob.material.phase_moduli.assign(pm, pm + np);
    prob.material.poisson_ratio = nu;
    prob.material.penalty = penalty;
    topmg::OptimConfig cfg;
    cfg.volume_fractions.assign(fractions, fractions + np);
    cfg.filter_radius = filter_radius;
    cfg.filter_tol = filter_tol;
    cfg.tol = tol;
    cfg.inner_sweeps = inner_sweeps;
    cfg.move_limit = move_limit;
    cfg.oc_damping = oc_damping;
    cfg.warm_start = warm_start != 0;
    cfg.max_outer = max_outer;
    cfg.density_floor = density_floor;
    cfg.solver.method = topmg::Method::pcgmg;
    cfg.solver.num_coarsenings = num_coarsenings;
    cfg.solver.omega = omega;
    cfg.solver.tol = solver_tol;
    cfg.solver.max_iter = solver_max_iter;
    cfg.solver.gamma = gamma;
    cfg.solver.pre_sweeps = pre;
    cfg.solver.post_sweeps = post;
    const topmg::OptimReport r = topmg::optimize(prob, cfg);
    std::memcpy(density, r.density.values().data(), sizeof(double) * r.density.values().size());
    for (size_t k = 0; k < r.compliance_history.size(); ++k) {
      compliance_hist[k] = r.compliance_history[k];
      change_hist[k] = r.change_history[k];
      iters_hist[k] = r.solver_iteration_history[k];
    }
    *outer_iterations = r.outer_iterations;
    *total_iters = r.total_solver_iterations;
    *converged = r.converged ? 1 : 0;
    return 0;
  } catch (...) {
    return map_exception(err, errlen, nullptr);
  }
}

// report.cpp:34-97: the reference's own output writers, for byte-compatibility
// tests of the Python mirror's writers
int ref_write_history_csv(int n, const double* compliance, const double* change, const int* iters,
                          const double* seconds, const char* path) {
  try {
    topmg::OptimReport r;
    r.compliance_history.assign(compliance, compliance + n);
    r.change_history.assign(change, change + n);
    r.solver_iteration_history.assign(iters, iters + n);
    r.seconds_history.assign(seconds, seconds + n);
    topmg::write_history_csv(r, path);
    return 0;
  } catch (...) {
    return map_exception(nullptr, 0, nullptr);
  }
}

int ref_write_residual_csv(int n, const double* hist, const char* path) {
  try {
    topmg::SolveReport r;
    r.residual_history.assign(hist, hist + n);
    topmg::write_residual_csv(r, path);
    return 0;
  } catch (...) {
    return map_exception(nullptr, 0, nullptr);
  }
}

int ref_write_density_images(int nx, int ny, int nphases, const double* alpha, const char* dir) {
  try {
    topmg::DensityField d = make_density(nx, ny, nphases, alpha);
    for (int i = 0; i < nphases; ++i)
      topmg::write_phase_pgm(d, i, std::string(dir) + "/phase_" + std::to_string(i + 1) + ".pgm");
    topmg::write_composite_ppm(d, std::string(dir) + "/composite.ppm");
    return 0;
  } catch (...) {
    return map_exception(nullptr, 0, nullptr);
  }
}

}  // extern "C"
