// Host-side input preparation for the pCGMG path (part of libtmg_gpu.so).
//
// These are the producers that sit in front of the solve in the reference:
//   * element_stiffness          proj/src/fem.cpp:131-169  (unit-modulus Ke)
//   * effective_moduli           proj/src/density.cpp:68-85 (E_e = sum a^p E_i)
//   * wall supports / loads      proj/src/fem.cpp:320-336 and the BASELINE
//                                variant (unit load spread over the top edge)
//   * rhs of assemble_from_moduli proj/src/fem.cpp:214-218 + 98-101
// plus the seeded synthetic density recipes of SURVEY.md section 8(d), drawn
// with std::mt19937_64 and the bit recipe of proj/tests/oracles.hpp:21-23 so
// the same arrays feed the GPU path and the CPU checkers.
//
// They run once per problem on the host (O(elements), no solve work) and are
// computed with the same IEEE operation order as the reference, so the moduli
// the GPU consumes are bit-identical to the ones the reference assembles.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#include <random>

#include "../../include/tmg_gpu.h"

namespace {

double uniform01(std::mt19937_64& g) {
  return static_cast<double>(g() >> 11) * 0x1.0p-53;
}

}  // namespace

extern "C" {

void tmg_element_stiffness(double modulus, double nu, double* ke) {
  // 2x2 Gauss on the unit square; d/dx = 2 d/dxi; corners CCW from lower left
  const double g = 0.57735026918962576451;
  const double c = modulus / (1.0 - nu * nu);
  const double d00 = c, d01 = c * nu, d22 = c * (1.0 - nu) / 2.0;
  const double gp[2] = {-g, g};
  const int sgx[4] = {-1, 1, 1, -1}, sgy[4] = {-1, -1, 1, 1};
  std::memset(ke, 0, 64 * sizeof(double));
  for (double xi : gp) {
    for (double eta : gp) {
      double dx[4], dy[4];
      for (int a = 0; a < 4; ++a) {
        const double fe = sgy[a] < 0 ? 1.0 - eta : 1.0 + eta;
        const double fx = sgx[a] < 0 ? 1.0 - xi : 1.0 + xi;
        dx[a] = 2.0 * ((sgx[a] < 0 ? -fe : fe) / 4.0);
        dy[a] = 2.0 * ((sgy[a] < 0 ? -fx : fx) / 4.0);
      }
      for (int i = 0; i < 8; ++i) {
        const bool iu = (i & 1) == 0;
        const double p0 = iu ? dx[i / 2] : 0.0, p1 = iu ? 0.0 : dy[i / 2];
        const double p2 = iu ? dy[i / 2] : dx[i / 2];
        for (int j = i; j < 8; ++j) {
          const bool ju = (j & 1) == 0;
          const double q0 = ju ? dx[j / 2] : 0.0, q1 = ju ? 0.0 : dy[j / 2];
          const double q2 = ju ? dy[j / 2] : dx[j / 2];
          const double v = p0 * (d00 * q0 + d01 * q1) + p1 * (d01 * q0 + d00 * q1) +
                           p2 * d22 * q2;
          ke[i * 8 + j] += 0.25 * v;
        }
      }
    }
  }
  for (int i = 1; i < 8; ++i)
    for (int j = 0; j < i; ++j) ke[i * 8 + j] = ke[j * 8 + i];
}

void tmg_inputs_effective_moduli(long n_elem, int nphases, const double* alpha,
                                 const double* phase_moduli, double penalty,
                                 double* out) {
  for (long e = 0; e < n_elem; ++e) {
    double v = 0.0;
    for (int i = 0; i < nphases; ++i) {
      v += std::pow(alpha[e * nphases + i], penalty) * phase_moduli[i];
    }
    out[e] = v;
  }
}

// SURVEY.md 8(d) c1/c4 recipe: element-major (e = ex*ny + ey), per element the
// material fractions rho_0..rho_{m-1} ~ U(0,1); if their sum exceeds 1 they are
// divided by it; the void phase takes the remainder (clamped at 0).
void tmg_inputs_density_iid(int nx, int ny, int nmat, unsigned long long seed,
                            double* alpha) {
  std::mt19937_64 g(seed);
  const long ne = static_cast<long>(nx) * ny;
  const int np = nmat + 1;
  for (long e = 0; e < ne; ++e) {
    double* a = alpha + e * np;
    double s = 0.0;
    for (int m = 0; m < nmat; ++m) {
      a[m] = uniform01(g);
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

// SURVEY.md 8(d) c2 recipe: block x block element tiles, tiles visited
// x-major, each tile assigned one phase uniformly (rng.index of
// oracles.hpp:24: gen() % nphases); alpha is one-hot.
void tmg_inputs_density_checker(int nx, int ny, int block, int nphases,
                                unsigned long long seed, double* alpha) {
  std::mt19937_64 g(seed);
  const int bx = (nx + block - 1) / block, by = (ny + block - 1) / block;
  std::memset(alpha, 0, sizeof(double) * static_cast<size_t>(nx) * ny * nphases);
  for (int i = 0; i < bx; ++i) {
    for (int j = 0; j < by; ++j) {
      const int ph = static_cast<int>(g() % static_cast<std::uint64_t>(nphases));
      for (int ex = i * block; ex < nx && ex < (i + 1) * block; ++ex)
        for (int ey = j * block; ey < ny && ey < (j + 1) * block; ++ey)
          alpha[(static_cast<long>(ex) * ny + ey) * nphases + ph] = 1.0;
    }
  }
}

// Square-wall supports: both dofs of every bottom node fixed (fem.cpp:328-332).
// load_mode 0: the reference's single unit point load at the top-mid node
// (fem.cpp:333-334); load_mode 1: BASELINE's unit total load spread as
// -1/(nx+1) on the v-dof of every top node. Returns the counts through
// n_fixed / n_loads (arrays sized 2*(nx+1) and nx+1).
void tmg_inputs_wall_bc(int nx, int ny, int load_mode, int* fixed, int* n_fixed,
                        int* load_dofs, double* load_vals, int* n_loads) {
  int k = 0;
  for (int x = 0; x <= nx; ++x) {
    const int node = x * (ny + 1);
    fixed[k++] = 2 * node;
    fixed[k++] = 2 * node + 1;
  }
  *n_fixed = k;
  if (load_mode == 0) {
    load_dofs[0] = 2 * ((nx / 2) * (ny + 1) + ny) + 1;
    load_vals[0] = -1.0;
    *n_loads = 1;
  } else {
    for (int x = 0; x <= nx; ++x) {
      load_dofs[x] = 2 * (x * (ny + 1) + ny) + 1;
      load_vals[x] = -1.0 / (nx + 1);
    }
    *n_loads = nx + 1;
  }
}

// rhs of the eliminated system: loads summed in order, fixed entries zeroed.
// BoundaryConditions::validate first (fem.cpp:110-129): a fixed or loaded dof
// outside [0, n) or a dof both fixed and loaded returns TMG_ERR_CONFIG and
// leaves b untouched.
int tmg_inputs_rhs(int nx, int ny, const int* fixed, int n_fixed, const int* load_dofs,
                   const double* load_vals, int n_loads, double* b) {
  const long n = 2L * (nx + 1) * (ny + 1);
  std::vector<char> is_fixed(static_cast<size_t>(n), 0);
  for (int i = 0; i < n_fixed; ++i) {
    if (fixed[i] < 0 || fixed[i] >= n) return 1;
    is_fixed[static_cast<size_t>(fixed[i])] = 1;
  }
  for (int i = 0; i < n_loads; ++i)
    if (load_dofs[i] < 0 || load_dofs[i] >= n || is_fixed[static_cast<size_t>(load_dofs[i])]) return 1;
  std::memset(b, 0, sizeof(double) * static_cast<size_t>(n));
  for (int i = 0; i < n_loads; ++i) b[load_dofs[i]] += load_vals[i];
  for (int i = 0; i < n_fixed; ++i) b[fixed[i]] = 0.0;
  return 0;
}

// poisson_element_matrix / poisson_mass_matrix (fem.cpp:37-81): 2x2 Gauss
// on the unit square, upper triangle accumulated then mirrored.
void tmg_poisson_element_matrices(double* k16, double* m16) {
  const double g = 0.57735026918962576451;
  const double pts[2] = {-g, g};
  std::memset(k16, 0, 16 * sizeof(double));
  std::memset(m16, 0, 16 * sizeof(double));
  for (double xi : pts)
    for (double eta : pts) {
      const double dx[4] = {2.0 * (-(1.0 - eta) / 4.0), 2.0 * ((1.0 - eta) / 4.0), 2.0 * ((1.0 + eta) / 4.0),
                            2.0 * (-(1.0 + eta) / 4.0)};
      const double dy[4] = {2.0 * (-(1.0 - xi) / 4.0), 2.0 * (-(1.0 + xi) / 4.0), 2.0 * ((1.0 + xi) / 4.0),
                            2.0 * ((1.0 - xi) / 4.0)};
      const double nv[4] = {(1.0 - xi) * (1.0 - eta) / 4.0, (1.0 + xi) * (1.0 - eta) / 4.0,
                            (1.0 + xi) * (1.0 + eta) / 4.0, (1.0 - xi) * (1.0 + eta) / 4.0};
      for (int i = 0; i < 4; ++i)
        for (int j = i; j < 4; ++j) {
          k16[i * 4 + j] += 0.25 * (dx[i] * dx[j] + dy[i] * dy[j]);
          m16[i * 4 + j] += 0.25 * nv[i] * nv[j];
        }
    }
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < i; ++j) {
      k16[i * 4 + j] = k16[j * 4 + i];
      m16[i * 4 + j] = m16[j * 4 + i];
    }
}

// The right-hand side of assemble_poisson (fem.cpp:243-276): the consistent
// load -M f summed element by element (ex outer, ey inner), boundary entries
// zeroed. node_source has (nx+1)(ny+1) entries in the reference node order.
void tmg_inputs_poisson_rhs(int nx, int ny, const double* node_source, double* b) {
  double k16[16], m16[16];
  tmg_poisson_element_matrices(k16, m16);
  const long n = static_cast<long>(nx + 1) * (ny + 1);
  std::memset(b, 0, sizeof(double) * static_cast<size_t>(n));
  for (int ex = 0; ex < nx; ++ex)
    for (int ey = 0; ey < ny; ++ey) {
      const long nd[4] = {static_cast<long>(ex) * (ny + 1) + ey, static_cast<long>(ex + 1) * (ny + 1) + ey,
                          static_cast<long>(ex + 1) * (ny + 1) + ey + 1, static_cast<long>(ex) * (ny + 1) + ey + 1};
      for (int a = 0; a < 4; ++a) {
        double load = 0.0;
        for (int c = 0; c < 4; ++c) load += m16[a * 4 + c] * node_source[nd[c]];
        b[nd[a]] -= load;
      }
    }
  for (int x = 0; x <= nx; ++x)
    for (int y = 0; y <= ny; ++y)
      if (x == 0 || y == 0 || x == nx || y == ny) b[static_cast<long>(x) * (ny + 1) + y] = 0.0;
}

}  // extern "C"
