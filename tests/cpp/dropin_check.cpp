// TEST DRIVER (built only where /root/reference exists; runs on the GPU box).
//
// Demonstrates the drop-in: the reference's own types and optimizer state,
// with the per-outer-iteration solve block of optimize() (mto.cpp:267-310)
// served once by the reference and once by topmg::gpu::PcgmgGpu, on the same
// designs. The designs are the reference optimizer's own iterates: design k
// is optimize(problem, cfg with max_outer = k).density (mto.cpp:229-354),
// i.e. an open-loop comparison, which is the protocol SURVEY.md 8(c)
// recommends because late optimization iterations are chaotic.
//
// Prints one line per design:  k iters_ref iters_gpu relerr_u relerr_C
//                              max_relerr_sens max_relerr_filtered
//                              max_abs_density_diff_after_oc_sweep
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "topmg/density.hpp"
#include "topmg/errors.hpp"
#include "topmg/fem.hpp"
#include "topmg/grid.hpp"
#include "topmg/mto.hpp"
#include "topmg/solvers.hpp"
#include "topmg_gpu.hpp"

using namespace topmg;

namespace {

double rel(const std::vector<double>& a, const std::vector<double>& b) {
  double n = 0.0, d = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    n += (a[i] - b[i]) * (a[i] - b[i]);
    d += b[i] * b[i];
  }
  return std::sqrt(n) / std::max(std::sqrt(d), 1e-300);
}

double maxrel(const std::vector<double>& a, const std::vector<double>& b) {
  double m = 0.0, s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    m = std::max(m, std::abs(a[i] - b[i]));
    s = std::max(s, std::abs(b[i]));
  }
  return m / std::max(s, 1e-300);
}

}  // namespace

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 64;
  const int designs = argc > 2 ? std::atoi(argv[2]) : 8;
  // BASELINE config 0: E = {1, 0.5, 0.2, 1e-9}, nu 0.3, p 3, V = 0.15 x 3,
  // r_f 1.5, 4 levels, damped Jacobi 0.6 with 2+2 sweeps, tol 1e-8, and the
  // unit total load spread over the top edge
  MaterialModel mat;
  mat.phase_moduli = {1.0, 0.5, 0.2, 1e-9};
  mat.poisson_ratio = 0.3;
  mat.penalty = 3.0;
  Problem prob;
  prob.grid = GridLevel{n, n, 2, 0};
  prob.material = mat;
  for (int x = 0; x <= n; ++x) {
    const int bottom = prob.grid.node_index(x, 0), top = prob.grid.node_index(x, n);
    prob.bc.fixed_dofs.push_back(2 * bottom);
    prob.bc.fixed_dofs.push_back(2 * bottom + 1);
    prob.bc.point_loads.emplace_back(2 * top + 1, -1.0 / (n + 1));
  }
  OptimConfig cfg;
  cfg.volume_fractions = {0.15, 0.15, 0.15, 0.55};
  cfg.filter_radius = 1.5;
  cfg.tol = 1e-12;
  cfg.solver.method = Method::pcgmg;
  cfg.solver.tol = 1e-8;
  cfg.solver.max_iter = 2000;
  cfg.solver.num_coarsenings = 3;
  cfg.solver.omega = 0.6;

  const GridHierarchy hier = build_hierarchy(n, n, cfg.solver.num_coarsenings, 2);
  gpu::PcgmgGpu dev(prob.grid, cfg.solver.num_coarsenings, mat.poisson_ratio, prob.bc);
  int bad = 0;
  // every design's (moduli, rhs) and blocking solution, for the pipelined pass below
  std::vector<std::pair<std::vector<double>, std::vector<double>>> served;
  std::vector<SolveReport> blocking;
  for (int k = 0; k < designs; ++k) {
    DensityField d = DensityField::uniform(n, n, cfg.volume_fractions, cfg.density_floor);
    if (k > 0) {
      OptimConfig ck = cfg;
      ck.max_outer = k;
      d = optimize(prob, ck).density;
    }
    // reference block (mto.cpp:267-310)
    const LinearSystem sys = assemble_elasticity(prob.grid, d, mat, prob.bc);
    const MultigridOperators ops = build_multigrid_operators(hier, sys.matrix, cfg.solver.omega);
    const SolveReport ref = pcgmg_solve(ops, sys.rhs, cfg.solver);
    const double c_ref = compliance(sys.matrix, ref.solution);
    const auto s_ref = sensitivities(ref.solution, d, mat, prob.grid);
    // the same block through the GPU drop-in
    dev.set_moduli(effective_moduli(d, mat), cfg.solver.omega);
    const SolveReport got = dev.solve(sys.rhs, cfg.solver);
    served.emplace_back(effective_moduli(d, mat), sys.rhs);
    blocking.push_back(got);
    const double c_gpu = dev.compliance();
    const auto s_gpu = dev.sensitivities(d, mat);
    double es = 0.0, ef = 0.0;
    std::vector<std::vector<double>> filt(static_cast<size_t>(mat.num_phases()));
    for (int i = 0; i < mat.num_phases(); ++i) {
      es = std::max(es, maxrel(s_gpu[i], s_ref[i]));
      const auto f_ref = filter_sensitivities(s_ref[i], d, i, cfg.filter_radius, prob.grid);
      const auto f_gpu = dev.filter_sensitivities(s_gpu[i], d, i, cfg.filter_radius);
      ef = std::max(ef, maxrel(f_gpu, f_ref));
      filt[static_cast<size_t>(i)] = f_ref;
    }
    // the OC pair sweep of mto.cpp:312-323 (one sweep per pair, the default
    // inner_sweeps) from the same filtered sensitivities: reference vs GPU
    DensityField d_ref = d, d_gpu = d;
    const std::vector<double> move(static_cast<size_t>(d.element_count()), cfg.move_limit);
    for (int a = 0; a < mat.num_phases() - 1; ++a)
      for (int b = a + 1; b < mat.num_phases(); ++b) {
        oc_update_pair(d_ref, a, b, filt[static_cast<size_t>(a)], filt[static_cast<size_t>(b)],
                       cfg.volume_fractions[static_cast<size_t>(a)], move, cfg.oc_damping);
        dev.oc_update_pair(d_gpu, a, b, filt[static_cast<size_t>(a)], filt[static_cast<size_t>(b)],
                           cfg.volume_fractions[static_cast<size_t>(a)], move, cfg.oc_damping);
      }
    const double eoc = DensityField::max_change(d_gpu, d_ref);
    const double eu = rel(got.solution, ref.solution), ec = std::abs(c_gpu - c_ref) / std::abs(c_ref);
    std::printf("%d %d %d %.3e %.3e %.3e %.3e %.3e\n", k, ref.iterations, got.iterations, eu, ec, es, ef, eoc);
    if (!(eu <= 1e-8 && ec <= 1e-9 && std::abs(ref.iterations - got.iterations) <= 2 && es <= 1e-8 &&
          ef <= 1e-8 && eoc <= 1e-12))
      ++bad;
  }
  // the same designs as one pipelined stream (PcgmgGpu::solve_many): bitwise
  // the blocking solves
  const std::vector<SolveReport> many = dev.solve_many(served, cfg.solver, cfg.solver.omega);
  int diff = 0;
  for (size_t k = 0; k < many.size(); ++k)
    if (many[k].solution != blocking[k].solution || many[k].iterations != blocking[k].iterations ||
        many[k].residual_history != blocking[k].residual_history)
      ++diff;
  std::printf("many %zu %d\n", many.size(), diff);
  return bad + diff;
}
