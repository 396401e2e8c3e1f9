// topmg_gpu.hpp -- header-only C++ drop-in over the C ABI (tmg_gpu.h) for the
// reference optimizer (topopt-mg, proj/src/mto.cpp).
//
// Include AFTER the reference headers (topmg/fem.hpp, topmg/solvers.hpp,
// topmg/density.hpp, topmg/errors.hpp); it reuses their types unchanged:
// GridLevel, BoundaryConditions, DensityField, MaterialModel, SolverConfig,
// SolveReport and the exception hierarchy of errors.hpp.
//
// One PcgmgGpu replaces, per outer iteration of optimize() (mto.cpp:267-310),
//   assemble_elasticity + build_multigrid_operators   -> set_density / set_moduli
//   pcgmg_solve(ops, sys.rhs, cfg, x0)                 -> solve(rhs, cfg, x0)
//   compliance(sys.matrix, u)                          -> compliance()
//   sensitivities(u, density, material, grid)          -> sensitivities(...)
//   filter_sensitivities(raw, density, i, r, grid)     -> filter_sensitivities(...)
//   oc_update_pair(density, a, b, fa, fb, V, move, d)  -> oc_update_pair(...)
// The mesh, supports and hierarchy stay resident on the GPU across outer
// iterations; only the moduli (or the density) change. See INTEGRATION.md.
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "tmg_gpu.h"

namespace topmg {
namespace gpu {

[[noreturn]] inline void throw_status(int status, tmg_gpu_handle* h) {
  char buf[512] = {0};
  int row = -1;
  if (h) tmg_gpu_last_error(h, buf, sizeof buf, &row);
  const std::string msg(buf);
  switch (status) {
    case TMG_ERR_CONFIG: throw ConfigError(msg);
    case TMG_ERR_DIMENSION: throw DimensionError(msg);
    case TMG_ERR_DEFINITENESS: throw DefinitenessError(msg, row);
    case TMG_ERR_PRECONDITIONER: throw PreconditionerError(msg);
    case TMG_ERR_SPLITTING: throw SplittingError(msg);
    case TMG_ERR_MULTIPLIER: throw MultiplierError(msg);
    default: throw NumericError("tmg_gpu: " + msg);
  }
}

class PcgmgGpu {
 public:
  // build_hierarchy(grid.nx, grid.ny, num_coarsenings, 2) + device residency
  PcgmgGpu(const GridLevel& grid, int num_coarsenings, double poisson_ratio,
           const BoundaryConditions& bc, int device = 0)
      : grid_(grid) {
    int st = tmg_gpu_create(grid.nx, grid.ny, num_coarsenings, grid.dofs_per_node, device, &h_);
    if (st != TMG_OK) fail(st);
    st = tmg_gpu_set_problem(h_, poisson_ratio, bc.fixed_dofs.data(),
                             static_cast<int>(bc.fixed_dofs.size()));
    if (st != TMG_OK) fail(st);
  }
  ~PcgmgGpu() { tmg_gpu_destroy(h_); }
  PcgmgGpu(const PcgmgGpu&) = delete;
  PcgmgGpu& operator=(const PcgmgGpu&) = delete;

  // assemble_from_moduli + build_multigrid_operators (fem.cpp:181, solvers.cpp:460)
  void set_moduli(const std::vector<double>& element_moduli, double omega) {
    check(tmg_gpu_set_moduli(h_, element_moduli.data(), static_cast<long>(element_moduli.size()), omega));
  }
  // effective_moduli on the device (density.cpp:68-85), then set_moduli
  void set_density(const DensityField& d, const MaterialModel& mat, double omega) {
    check_density(d, mat, "set_density");
    check(tmg_gpu_set_density(h_, d.values().data(), d.num_phases(), mat.phase_moduli.data(), mat.penalty,
                              omega));
  }

  // pcgmg_solve (solvers.cpp:516-530): same SolveReport, same exceptions
  SolveReport solve(const std::vector<double>& b, const SolverConfig& cfg,
                    const std::vector<double>* x0 = nullptr) {
    if (static_cast<int>(b.size()) != grid_.dof_count())
      throw DimensionError("pcgmg_solve: rhs length does not match the grid");
    // r = b - A x0 (solvers.cpp:346-350) checks x0 through the matvec (sparse.cpp:72-75)
    if (x0 && x0->size() != b.size())
      throw DimensionError("matvec: vector length " + std::to_string(x0->size()) + " does not match matrix size " +
                           std::to_string(b.size()));
    SolveReport rep;
    rep.solution.resize(b.size());
    rep.residual_history.resize(static_cast<size_t>(cfg.max_iter) + 1);
    int iters = 0, conv = 0, hl = 0;
    check(tmg_gpu_solve(h_, b.data(), x0 ? x0->data() : nullptr, cfg.tol, cfg.max_iter, cfg.gamma,
                        cfg.pre_sweeps, cfg.post_sweeps, rep.solution.data(), &iters,
                        &rep.final_residual, &conv, &rep.seconds, rep.residual_history.data(),
                        static_cast<int>(rep.residual_history.size()), &hl));
    rep.iterations = iters;
    rep.converged = conv != 0;
    rep.residual_history.resize(static_cast<size_t>(hl));
    return rep;
  }

  // A stream of independent problems {(element moduli, rhs)} on this mesh:
  // per problem set_moduli(moduli, omega) + solve(rhs, cfg) semantics and
  // results (bitwise), with each problem's host<->device copies overlapping
  // the neighbouring solves (tmg_gpu_stage_inputs / tmg_gpu_solve_staged,
  // include/tmg_gpu.h). The inputs are read while their copies run; they stay
  // untouched in the caller's vectors. Pinned memory overlaps best; std::vector
  // storage works (serialised copies).
  std::vector<SolveReport> solve_many(const std::vector<std::pair<std::vector<double>, std::vector<double>>>& probs,
                                      const SolverConfig& cfg, double omega) {
    for (const auto& p : probs) {
      if (static_cast<int>(p.first.size()) != grid_.element_count())
        throw DimensionError("solve_many: element modulus count does not match the grid");
      if (static_cast<int>(p.second.size()) != grid_.dof_count())
        throw DimensionError("pcgmg_solve: rhs length does not match the grid");
    }
    std::vector<SolveReport> out(probs.size());
    auto stage = [&](size_t k) {
      check(tmg_gpu_stage_inputs(h_, static_cast<int>(k & 1), probs[k].first.data(),
                                 static_cast<long>(probs[k].first.size()), probs[k].second.data()));
    };
    if (!probs.empty()) stage(0);
    for (size_t k = 0; k < probs.size(); ++k) {
      if (k + 1 < probs.size()) stage(k + 1);
      SolveReport& rep = out[k];
      rep.solution.resize(probs[k].second.size());
      rep.residual_history.resize(static_cast<size_t>(cfg.max_iter) + 1);
      int iters = 0, conv = 0, hl = 0;
      check(tmg_gpu_solve_staged(h_, static_cast<int>(k & 1), omega, cfg.tol, cfg.max_iter, cfg.gamma,
                                 cfg.pre_sweeps, cfg.post_sweeps, rep.solution.data(), &iters, &rep.final_residual,
                                 &conv, &rep.seconds, rep.residual_history.data(),
                                 static_cast<int>(rep.residual_history.size()), &hl));
      rep.iterations = iters;
      rep.converged = conv != 0;
      rep.residual_history.resize(static_cast<size_t>(hl));
    }
    check(tmg_gpu_sync_outputs(h_));
    return out;
  }

  // compliance of the resident solution (fem.cpp:284-290)
  double compliance() const {
    double c = 0.0;
    check(tmg_gpu_compliance(h_, nullptr, &c));
    return c;
  }
  std::vector<double> element_energies() const {
    std::vector<double> e(static_cast<size_t>(grid_.element_count()));
    check(tmg_gpu_element_energies(h_, nullptr, e.data()));
    return e;
  }
  // sensitivities (mto.cpp:61-85) of the resident solution
  std::vector<std::vector<double>> sensitivities(const DensityField& d, const MaterialModel& mat) const {
    check_density(d, mat, "sensitivities");  // mto.cpp:65-70
    const size_t ne = static_cast<size_t>(grid_.element_count());
    std::vector<double> flat(ne * static_cast<size_t>(d.num_phases()));
    check(tmg_gpu_sensitivities(h_, nullptr, d.num_phases(), d.values().data(), mat.phase_moduli.data(),
                                mat.penalty, flat.data()));
    std::vector<std::vector<double>> out(static_cast<size_t>(d.num_phases()));
    for (size_t i = 0; i < out.size(); ++i) out[i].assign(flat.begin() + i * ne, flat.begin() + (i + 1) * ne);
    return out;
  }
  // filter_sensitivities (mto.cpp:87-117)
  std::vector<double> filter_sensitivities(const std::vector<double>& raw, const DensityField& d, int phase,
                                           double radius) const {
    if (static_cast<int>(raw.size()) != grid_.element_count())  // mto.cpp:90-92
      throw DimensionError("filter: field length does not match element count");
    if (radius > 1.0 && (d.nx() != grid_.nx || d.ny() != grid_.ny))
      throw DimensionError("filter: density grid does not match level");
    std::vector<double> out(raw.size());
    check(tmg_gpu_filter(h_, d.num_phases(), d.values().data(), phase, radius, raw.data(), out.data()));
    return out;
  }

  // oc_update_pair (mto.cpp:142-227), per-element move limits (mto.hpp:73-77)
  void oc_update_pair(DensityField& d, int phase_a, int phase_b, const std::vector<double>& filtered_sens_a,
                      const std::vector<double>& filtered_sens_b, double target_fraction,
                      const std::vector<double>& move, double damping) const {
    const size_t ne = static_cast<size_t>(d.element_count());
    if (d.nx() != grid_.nx || d.ny() != grid_.ny)
      throw DimensionError("oc_update_pair: density grid does not match the handle's grid");
    if (phase_a == phase_b) throw ConfigError("oc_update_pair: phases must differ");
    if (filtered_sens_a.size() != ne || filtered_sens_b.size() != ne || move.size() != ne)
      throw DimensionError("oc_update_pair: field length does not match grid");
    std::vector<double> v = d.values();
    check(tmg_gpu_oc_update_pair(h_, v.data(), d.num_phases(), d.floor_eps(), phase_a, phase_b,
                                 filtered_sens_a.data(), filtered_sens_b.data(), target_fraction, move.data(),
                                 damping));
    for (size_t e = 0; e < ne; ++e)
      for (int i = 0; i < d.num_phases(); ++i)
        d.at(static_cast<int>(e), i) = v[e * static_cast<size_t>(d.num_phases()) + static_cast<size_t>(i)];
  }
  // the scalar move-limit overload (mto.hpp:66-69)
  void oc_update_pair(DensityField& d, int phase_a, int phase_b, const std::vector<double>& filtered_sens_a,
                      const std::vector<double>& filtered_sens_b, double target_fraction, double move,
                      double damping) const {
    oc_update_pair(d, phase_a, phase_b, filtered_sens_a, filtered_sens_b, target_fraction,
                   std::vector<double>(static_cast<size_t>(d.element_count()), move), damping);
  }

  tmg_gpu_handle* handle() const { return h_; }

 private:
  [[noreturn]] void fail(int st) {
    tmg_gpu_handle* h = h_;
    try {
      throw_status(st, h);
    } catch (...) {
      tmg_gpu_destroy(h_);
      h_ = nullptr;
      throw;
    }
  }
  // sensitivities' checks (mto.cpp:65-70), applied wherever a density
  // crosses the boundary
  void check_density(const DensityField& d, const MaterialModel& mat, const char* what) const {
    if (d.nx() != grid_.nx || d.ny() != grid_.ny)
      throw DimensionError(std::string(what) + ": density grid does not match level");
    if (d.num_phases() != mat.num_phases()) throw DimensionError(std::string(what) + ": phase count mismatch");
  }
  void check(int st) const {
    if (st != TMG_OK) throw_status(st, h_);
  }

  GridLevel grid_;
  tmg_gpu_handle* h_ = nullptr;
};

}  // namespace gpu
}  // namespace topmg
