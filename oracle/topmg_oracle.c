/*
 * TEST INFRASTRUCTURE ONLY -- CPU checker for the GPU pCGMG path.
 * See topmg_oracle.h for the contract. Citations are /root/reference/proj
 * file:line. This file is a restatement in plain C: CSR matrices on the host,
 * sequential loops, the same operation order as the reference so that the
 * results are bit-identical (pinned by tests/test_oracle_pin.py).
 */
#define _POSIX_C_SOURCE 200809L
#include "topmg_oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

enum { ST_OK = 0, ST_CONFIG = 1, ST_DIM = 2, ST_DEF = 3, ST_PRECOND = 4, ST_MULTIPLIER = 8 };

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static void set_err(char* err, int len, const char* msg) {
  if (err && len > 0) snprintf(err, (size_t)len, "%s", msg);
}

/* ------------------------------------------------------------------ CSR -- */

typedef struct {
  int n;
  int* off; /* n+1 */
  int* col;
  double* val;
} Csr;

static void csr_free(Csr* m) {
  free(m->off);
  free(m->col);
  free(m->val);
  memset(m, 0, sizeof(*m));
}

/* y = A x, sequential per row in stored (ascending column) order:
 * sparse.cpp:70-86 */
static void csr_mul(const Csr* a, const double* x, double* y) {
  for (int i = 0; i < a->n; ++i) {
    double s = 0.0;
    for (int k = a->off[i]; k < a->off[i + 1]; ++k) s += a->val[k] * x[a->col[k]];
    y[i] = s;
  }
}

/* value_at by binary search, used for the diagonal: sparse.cpp:101-117 */
static double csr_at(const Csr* a, int i, int j) {
  int lo = a->off[i], hi = a->off[i + 1];
  while (lo < hi) {
    int mid = lo + (hi - lo) / 2;
    if (a->col[mid] < j) lo = mid + 1; else hi = mid;
  }
  return (lo < a->off[i + 1] && a->col[lo] == j) ? a->val[lo] : 0.0;
}

/* sparse.cpp:134-144 */
static double vdot(const double* a, const double* b, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* ------------------------------------------------------- element matrix -- */

/* Q4 plane stress on the unit square, 2x2 Gauss: fem.cpp:131-169 with the
 * shape derivatives of fem.cpp:18-27 (d/dx = 2 d/dxi). */
void orc_element_stiffness(double modulus, double nu, double* ke) {
  const double g = 0.57735026918962576451;
  const double c = modulus / (1.0 - nu * nu);
  const double d00 = c, d01 = c * nu, d22 = c * (1.0 - nu) / 2.0;
  const double pts[2] = {-g, g};
  /* sign pattern of dN/dxi and dN/deta per corner (CCW from lower left) */
  static const double sx[4] = {-1.0, 1.0, 1.0, -1.0};
  static const double sy[4] = {-1.0, -1.0, 1.0, 1.0};
  memset(ke, 0, 64 * sizeof(double));
  for (int q = 0; q < 4; ++q) {
    const double xi = pts[q / 2], eta = pts[q % 2];
    double gx[4], gy[4];
    for (int a = 0; a < 4; ++a) {
      /* dN_a/dx = 2 * (sx * (1 + sy*eta) / 4) ; dN_a/dy = 2 * (sy * (1 + sx*xi) / 4) */
      const double fe = (sy[a] < 0.0) ? (1.0 - eta) : (1.0 + eta);
      const double fx = (sx[a] < 0.0) ? (1.0 - xi) : (1.0 + xi);
      gx[a] = 2.0 * ((sx[a] < 0.0 ? -fe : fe) / 4.0);
      gy[a] = 2.0 * ((sy[a] < 0.0 ? -fx : fx) / 4.0);
    }
    for (int i = 0; i < 8; ++i) {
      const int na = i / 2, iu = (i % 2 == 0);
      const double b0 = iu ? gx[na] : 0.0, b1 = iu ? 0.0 : gy[na];
      const double b2 = iu ? gy[na] : gx[na];
      for (int j = i; j < 8; ++j) {
        const int nb = j / 2, ju = (j % 2 == 0);
        const double c0 = ju ? gx[nb] : 0.0, c1 = ju ? 0.0 : gy[nb];
        const double c2 = ju ? gy[nb] : gx[nb];
        const double v = b0 * (d00 * c0 + d01 * c1) + b1 * (d01 * c0 + d00 * c1) +
                         b2 * d22 * c2;
        ke[i * 8 + j] += 0.25 * v;
      }
    }
  }
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < i; ++j) ke[i * 8 + j] = ke[j * 8 + i];
}

/* ------------------------------------------------------------ hierarchy -- */

typedef struct {
  int nx, ny;
} Lvl;

static int lvl_nodes(Lvl l) { return (l.nx + 1) * (l.ny + 1); }

/* Prolongation rows per fine dof, <= 4 parents, bilinear weights:
 * grid.cpp:13-46. Stored like the reference (offsets / parents / weights). */
typedef struct {
  int nf, nc;
  int* off;
  int* par;
  double* w;
} Prol;

static void prol_build(Prol* p, Lvl coarse, Lvl fine, int dpn) {
  const int nf = dpn * lvl_nodes(fine);
  p->nf = nf;
  p->nc = dpn * lvl_nodes(coarse);
  p->off = malloc(sizeof(int) * (size_t)(nf + 1));
  p->par = malloc(sizeof(int) * (size_t)nf * 4);
  p->w = malloc(sizeof(double) * (size_t)nf * 4);
  int k = 0, r = 0;
  p->off[0] = 0;
  for (int fx = 0; fx <= fine.nx; ++fx) {
    for (int fy = 0; fy <= fine.ny; ++fy) {
      int px[2], py[2], mx, my;
      double wx[2], wy[2];
      px[0] = fx / 2; px[1] = fx / 2 + 1;
      py[0] = fy / 2; py[1] = fy / 2 + 1;
      if (fx % 2) { mx = 2; wx[0] = wx[1] = 0.5; } else { mx = 1; wx[0] = 1.0; }
      if (fy % 2) { my = 2; wy[0] = wy[1] = 0.5; } else { my = 1; wy[0] = 1.0; }
      for (int c = 0; c < dpn; ++c) {
        for (int a = 0; a < mx; ++a)
          for (int b = 0; b < my; ++b) {
            p->par[k] = (px[a] * (coarse.ny + 1) + py[b]) * dpn + c;
            p->w[k] = wx[a] * wy[b];
            ++k;
          }
        p->off[++r] = k;
      }
    }
  }
}

static void prol_free(Prol* p) {
  free(p->off);
  free(p->par);
  free(p->w);
}

/* fine = P coarse: grid.cpp:98-120 */
static void prolongate(const Prol* p, const double* coarse, double* fine) {
  for (int i = 0; i < p->nf; ++i) {
    double s = 0.0;
    for (int k = p->off[i]; k < p->off[i + 1]; ++k) s += p->w[k] * coarse[p->par[k]];
    fine[i] = s;
  }
}

/* coarse = P^T fine / 4, scatter form: grid.cpp:122-142 */
static void restrict_(const Prol* p, const double* fine, double* coarse) {
  memset(coarse, 0, sizeof(double) * (size_t)p->nc);
  for (int i = 0; i < p->nf; ++i) {
    const double v = 0.25 * fine[i];
    for (int k = p->off[i]; k < p->off[i + 1]; ++k) coarse[p->par[k]] += p->w[k] * v;
  }
}

/* ------------------------------------------------------------- assembly -- */

/* local corner index of offset (dx, dy) in {0,1}^2, CCW from lower left:
 * fem.cpp:83-86 */
static int corner(int dx, int dy) { return dy ? (dx ? 2 : 3) : (dx ? 1 : 0); }

/* Assembled fine operator Z(sum_e E_e Ke)Z + I_fixed with the elimination
 * convention of fem.cpp:89-106. The reference pushes 64 triplets per element
 * (ex outer, ey inner) and stable-sorts them, so each (row, col) value is the
 * sum over the shared elements in element order starting from 0.0
 * (sparse.cpp:12-52); rows hold their columns in ascending dof order. The
 * same sums are formed here directly on the structured grid. */
static int assemble(int nx, int ny, const double* E, const double* ke,
                    const int* fixcount, Csr* out) {
  const int nn = (nx + 1) * (ny + 1), n = 2 * nn;
  out->n = n;
  out->off = malloc(sizeof(int) * (size_t)(n + 1));
  out->col = malloc(sizeof(int) * (size_t)n * 18);
  out->val = malloc(sizeof(double) * (size_t)n * 18);
  if (!out->off || !out->col || !out->val) return ST_DIM;
  int k = 0;
  out->off[0] = 0;
  for (int x = 0; x <= nx; ++x) {
    for (int y = 0; y <= ny; ++y) {
      for (int c = 0; c < 2; ++c) {
        const int row = 2 * (x * (ny + 1) + y) + c;
        if (fixcount[row]) {
          double d = 0.0;
          for (int t = 0; t < fixcount[row]; ++t) d += 1.0;
          out->col[k] = row;
          out->val[k++] = d;
          out->off[row + 1] = k;
          continue;
        }
        for (int x2 = x - 1; x2 <= x + 1; ++x2) {
          if (x2 < 0 || x2 > nx) continue;
          for (int y2 = y - 1; y2 <= y + 1; ++y2) {
            if (y2 < 0 || y2 > ny) continue;
            for (int d = 0; d < 2; ++d) {
              const int colid = 2 * (x2 * (ny + 1) + y2) + d;
              if (fixcount[colid]) continue;
              double s = 0.0;
              for (int ex = x - 1; ex <= x; ++ex) {
                if (ex < 0 || ex >= nx || x2 - ex < 0 || x2 - ex > 1) continue;
                for (int ey = y - 1; ey <= y; ++ey) {
                  if (ey < 0 || ey >= ny || y2 - ey < 0 || y2 - ey > 1) continue;
                  const int a = corner(x - ex, y - ey), b = corner(x2 - ex, y2 - ey);
                  s += E[ex * ny + ey] * ke[(2 * a + c) * 8 + 2 * b + d];
                }
              }
              out->col[k] = colid;
              out->val[k++] = s;
            }
          }
        }
        out->off[row + 1] = k;
      }
    }
  }
  return ST_OK;
}

/* Galerkin (1/4) P^T A P on the nine-point coarse pattern, accumulated in
 * the reference's loop order: solvers.cpp:397-458 */
static void galerkin(const Csr* a, const Prol* p, Lvl cl, Csr* out, int dpn) {
  const int nc = p->nc;
  out->n = nc;
  out->off = malloc(sizeof(int) * (size_t)(nc + 1));
  out->col = malloc(sizeof(int) * (size_t)nc * 18);
  int k = 0;
  out->off[0] = 0;
  for (int x = 0; x <= cl.nx; ++x)
    for (int y = 0; y <= cl.ny; ++y)
      for (int c = 0; c < dpn; ++c) {
        /* neighbor dofs ascending: node index grows with x then y */
        for (int x2 = x - 1; x2 <= x + 1; ++x2) {
          if (x2 < 0 || x2 > cl.nx) continue;
          for (int y2 = y - 1; y2 <= y + 1; ++y2) {
            if (y2 < 0 || y2 > cl.ny) continue;
            for (int d = 0; d < dpn; ++d) out->col[k++] = dpn * (x2 * (cl.ny + 1) + y2) + d;
          }
        }
        out->off[dpn * (x * (cl.ny + 1) + y) + c + 1] = k;
      }
  out->val = calloc((size_t)k, sizeof(double));
  for (int i = 0; i < p->nf; ++i) {
    for (int ki = p->off[i]; ki < p->off[i + 1]; ++ki) {
      const int ci = p->par[ki];
      const double wi = 0.25 * p->w[ki];
      const int rb = out->off[ci], re = out->off[ci + 1];
      for (int q = a->off[i]; q < a->off[i + 1]; ++q) {
        const int j = a->col[q];
        const double wiv = wi * a->val[q];
        for (int kj = p->off[j]; kj < p->off[j + 1]; ++kj) {
          const int cj = p->par[kj];
          int lo = rb, hi = re;
          while (lo < hi) {
            int mid = lo + (hi - lo) / 2;
            if (out->col[mid] < cj) lo = mid + 1; else hi = mid;
          }
          out->val[lo] += wiv * p->w[kj];
        }
      }
    }
  }
}

/* ------------------------------------------------------------- cholesky -- */

/* Envelope (profile) Cholesky: solvers.cpp:89-152, solve solvers.cpp:154-183 */
typedef struct {
  int n;
  int* first;
  size_t* off;
  double* v;
} Chol;

static int chol_factor(const Csr* a, Chol* f, int* bad_row, double* bad_pivot) {
  const int n = a->n;
  f->n = n;
  f->first = malloc(sizeof(int) * (size_t)n);
  f->off = malloc(sizeof(size_t) * (size_t)(n + 1));
  f->off[0] = 0;
  for (int i = 0; i < n; ++i) {
    int fi = i;
    if (a->off[i] < a->off[i + 1] && a->col[a->off[i]] < fi) fi = a->col[a->off[i]];
    f->first[i] = fi;
    f->off[i + 1] = f->off[i] + (size_t)(i - fi + 1);
  }
  f->v = calloc(f->off[n], sizeof(double));
  for (int i = 0; i < n; ++i)
    for (int q = a->off[i]; q < a->off[i + 1]; ++q)
      if (a->col[q] <= i) f->v[f->off[i] + (size_t)(a->col[q] - f->first[i])] = a->val[q];
  double* L = f->v;
  for (int i = 0; i < n; ++i) {
    const int fi = f->first[i];
    double* Li = L + f->off[i] - fi; /* Li[k] addresses column k of row i */
    for (int j = fi; j < i; ++j) {
      const int fj = f->first[j];
      const double* Lj = L + f->off[j] - fj;
      double s = Li[j];
      for (int q = (fi > fj ? fi : fj); q < j; ++q) s -= Li[q] * Lj[q];
      Li[j] = s / Lj[j];
    }
    double d = Li[i];
    for (int q = fi; q < i; ++q) d -= Li[q] * Li[q];
    if (!(d > 0.0)) {
      *bad_row = i;
      *bad_pivot = d;
      return ST_DEF;
    }
    Li[i] = sqrt(d);
  }
  return ST_OK;
}

static void chol_solve(const Chol* f, const double* b, double* x) {
  const int n = f->n;
  memcpy(x, b, sizeof(double) * (size_t)n);
  for (int i = 0; i < n; ++i) {
    const double* Li = f->v + f->off[i] - f->first[i];
    double s = x[i];
    for (int q = f->first[i]; q < i; ++q) s -= Li[q] * x[q];
    x[i] = s / Li[i];
  }
  for (int i = n - 1; i >= 0; --i) {
    const double* Li = f->v + f->off[i] - f->first[i];
    const double xi = x[i] / Li[i];
    x[i] = xi;
    for (int q = f->first[i]; q < i; ++q) x[q] -= Li[q] * xi;
  }
}

static void chol_free(Chol* f) {
  free(f->first);
  free(f->off);
  free(f->v);
}

/* --------------------------------------------------------------- system -- */

typedef struct {
  int nx, ny, n;
  int dpn; /* dofs per node: 2 elasticity, 1 Poisson */
  double nu, omega;
  Csr fine;
  double* rhs;
  int nlev; /* 0 until build_mg */
  Lvl* lv;  /* coarsest first, like GridHierarchy::levels (grid.hpp:47-56) */
  Csr* mat; /* mat[nlev-1] aliases fine */
  Prol* pr; /* pr[l-1]: level l-1 -> l */
  Chol coarse;
  double t_asm, t_setup, t_pcg;
} Sys;

void* orc_system_create(int nx, int ny, const double* moduli, double nu,
                        const int* fixed, int n_fixed, const int* load_dofs,
                        const double* load_vals, int n_loads, char* err,
                        int errlen, int* status) {
  const double t0 = now_s();
  const int n = 2 * (nx + 1) * (ny + 1);
  char msg[160];
  /* BoundaryConditions::validate, fem.cpp:110-129 */
  int* fc = calloc((size_t)n, sizeof(int));
  for (int i = 0; i < n_fixed; ++i) {
    if (fixed[i] < 0 || fixed[i] >= n) {
      snprintf(msg, sizeof msg, "fixed dof %d outside [0, %d)", fixed[i], n);
      set_err(err, errlen, msg);
      free(fc);
      *status = ST_CONFIG;
      return NULL;
    }
    fc[fixed[i]]++;
  }
  for (int i = 0; i < n_loads; ++i) {
    const int d = load_dofs[i];
    if (d < 0 || d >= n || fc[d]) {
      if (d < 0 || d >= n) snprintf(msg, sizeof msg, "loaded dof %d outside [0, %d)", d, n);
      else snprintf(msg, sizeof msg, "dof %d is both fixed and loaded", d);
      set_err(err, errlen, msg);
      free(fc);
      *status = ST_CONFIG;
      return NULL;
    }
  }
  Sys* s = calloc(1, sizeof(Sys));
  s->nx = nx;
  s->ny = ny;
  s->n = n;
  s->dpn = 2;
  s->nu = nu;
  double ke[64];
  orc_element_stiffness(1.0, nu, ke);
  assemble(nx, ny, moduli, ke, fc, &s->fine);
  /* rhs: loads summed, fixed entries zeroed: fem.cpp:214-218, 98-101 */
  s->rhs = calloc((size_t)n, sizeof(double));
  for (int i = 0; i < n_loads; ++i) s->rhs[load_dofs[i]] += load_vals[i];
  for (int i = 0; i < n_fixed; ++i) s->rhs[fixed[i]] = 0.0;
  free(fc);
  s->t_asm = now_s() - t0;
  *status = ST_OK;
  return s;
}

static void drop_mg(Sys* s) {
  if (!s->nlev) return;
  for (int l = 0; l + 1 < s->nlev; ++l) {
    csr_free(&s->mat[l]);
    prol_free(&s->pr[l]);
  }
  chol_free(&s->coarse);
  free(s->mat);
  free(s->pr);
  free(s->lv);
  s->nlev = 0;
}

int orc_system_build_mg(void* h, int nc, double omega, char* err, int errlen, int* row) {
  Sys* s = h;
  char msg[200];
  drop_mg(s);
  /* build_hierarchy validation: grid.cpp:55-80 */
  if (nc < 0) {
    set_err(err, errlen, "num_coarsenings must be non-negative");
    return ST_CONFIG;
  }
  const int f = 1 << nc;
  if (s->nx % f || s->ny % f) {
    snprintf(msg, sizeof msg, "%s = %d is not divisible by 2^%d = %d",
             s->nx % f ? "nx" : "ny", s->nx % f ? s->nx : s->ny, nc, f);
    set_err(err, errlen, msg);
    return ST_CONFIG;
  }
  const double t0 = now_s();
  s->nlev = nc + 1;
  s->omega = omega;
  s->lv = malloc(sizeof(Lvl) * (size_t)s->nlev);
  s->mat = calloc((size_t)s->nlev, sizeof(Csr));
  s->pr = calloc((size_t)s->nlev, sizeof(Prol));
  for (int l = 0; l <= nc; ++l) {
    s->lv[l].nx = s->nx >> (nc - l);
    s->lv[l].ny = s->ny >> (nc - l);
  }
  for (int l = 1; l <= nc; ++l) prol_build(&s->pr[l - 1], s->lv[l - 1], s->lv[l], s->dpn);
  s->mat[nc] = s->fine;
  for (int l = nc; l >= 1; --l) galerkin(&s->mat[l], &s->pr[l - 1], s->lv[l - 1], &s->mat[l - 1], s->dpn);
  int bad = -1;
  double piv = 0.0;
  const int st = chol_factor(&s->mat[0], &s->coarse, &bad, &piv);
  if (st != ST_OK) {
    snprintf(msg, sizeof msg, "matrix is not positive definite: pivot %f at row %d", piv, bad);
    set_err(err, errlen, msg);
    if (row) *row = bad;
    /* leave the hierarchy unbuilt, like the exception in the reference */
    s->coarse.n = 0;
    for (int l = 0; l < nc; ++l) {
      csr_free(&s->mat[l]);
      prol_free(&s->pr[l]);
    }
    free(s->mat);
    free(s->pr);
    free(s->lv);
    chol_free(&s->coarse);
    s->nlev = 0;
    return ST_DEF;
  }
  s->t_setup = now_s() - t0;
  return ST_OK;
}

int orc_system_num_levels(void* h) {
  Sys* s = h;
  return s->nlev ? s->nlev : 1;
}

void orc_system_rhs(void* h, double* out) {
  Sys* s = h;
  memcpy(out, s->rhs, sizeof(double) * (size_t)s->n);
}

static const Csr* level_mat(Sys* s, int level) {
  if (s->nlev) return (level >= 0 && level < s->nlev) ? &s->mat[level] : NULL;
  return level == 0 ? &s->fine : NULL;
}

long orc_system_level_nnz(void* h, int level) {
  const Csr* m = level_mat(h, level);
  return m ? (long)m->off[m->n] : -1;
}

int orc_system_level_size(void* h, int level) {
  const Csr* m = level_mat(h, level);
  return m ? m->n : -1;
}

int orc_system_level_csr(void* h, int level, int* offsets, int* cols, double* vals) {
  const Csr* m = level_mat(h, level);
  if (!m) return ST_DIM;
  memcpy(offsets, m->off, sizeof(int) * (size_t)(m->n + 1));
  memcpy(cols, m->col, sizeof(int) * (size_t)m->off[m->n]);
  memcpy(vals, m->val, sizeof(double) * (size_t)m->off[m->n]);
  return ST_OK;
}

int orc_system_matvec(void* h, int level, const double* x, double* y) {
  const Csr* m = level_mat(h, level);
  if (!m) return ST_DIM;
  csr_mul(m, x, y);
  return ST_OK;
}

/* x += omega D^-1 (b - A x) with the old x: solvers.cpp:30-37 */
static void jacobi(const Csr* a, double* x, const double* b, const double* dg,
                   double omega, double* scratch) {
  csr_mul(a, x, scratch);
  for (int i = 0; i < a->n; ++i) x[i] += omega * (b[i] - scratch[i]) / dg[i];
}

/* gamma-cycle, Alg. 1: solvers.cpp:483-514 */
static void cycle(Sys* s, int l, double* u, const double* f, int gamma, int pre, int post) {
  if (l == 0) {
    double* t = malloc(sizeof(double) * (size_t)s->mat[0].n);
    chol_solve(&s->coarse, f, t);
    memcpy(u, t, sizeof(double) * (size_t)s->mat[0].n);
    free(t);
    return;
  }
  const Csr* a = &s->mat[l];
  const int n = a->n, ncd = s->mat[l - 1].n;
  double* dg = malloc(sizeof(double) * (size_t)n);
  double* sc = calloc((size_t)n, sizeof(double));
  for (int i = 0; i < n; ++i) dg[i] = csr_at(a, i, i);
  for (int t = 0; t < pre; ++t) jacobi(a, u, f, dg, s->omega, sc);
  csr_mul(a, u, sc);
  for (int i = 0; i < n; ++i) sc[i] = f[i] - sc[i];
  double* fc = malloc(sizeof(double) * (size_t)ncd);
  double* uc = calloc((size_t)ncd, sizeof(double));
  restrict_(&s->pr[l - 1], sc, fc);
  const int visits = (l == s->nlev - 1) ? 1 : gamma;
  for (int t = 0; t < visits; ++t) cycle(s, l - 1, uc, fc, gamma, pre, post);
  prolongate(&s->pr[l - 1], uc, sc);
  for (int i = 0; i < n; ++i) u[i] += sc[i];
  for (int t = 0; t < post; ++t) jacobi(a, u, f, dg, s->omega, sc);
  free(dg);
  free(sc);
  free(fc);
  free(uc);
}

int orc_system_vcycle(void* h, const double* f, double* u, int gamma, int pre, int post) {
  Sys* s = h;
  if (!s->nlev) return ST_DIM;
  cycle(s, s->nlev - 1, u, f, gamma, pre, post);
  return ST_OK;
}

/* pcgmg_solve (solvers.cpp:516-530) around pcg_solve (solvers.cpp:332-395) */
int orc_system_solve(void* h, const double* b, const double* x0, double tol,
                     int max_iter, int gamma, int pre, int post, double* x,
                     int* iters, double* final_relres, int* converged,
                     double* hist, int* hist_len, char* err, int errlen) {
  Sys* s = h;
  char msg[200];
  if (!s->nlev) {
    set_err(err, errlen, "multigrid operators not built");
    return ST_DIM;
  }
  if (pre != post) {
    set_err(err, errlen, "pcgmg needs pre_sweeps == post_sweeps for a symmetric preconditioner");
    return ST_CONFIG;
  }
  const double t0 = now_s();
  const int n = s->n;
  const Csr* a = &s->fine;
  int nh = 0, st = ST_OK;
  *iters = 0;
  *converged = 0;
  const double bnorm = sqrt(vdot(b, b, n));
  if (bnorm == 0.0) {
    memset(x, 0, sizeof(double) * (size_t)n);
    *converged = 1;
    *final_relres = 0.0;
    hist[nh++] = 0.0;
    *hist_len = nh;
    s->t_pcg = now_s() - t0;
    return ST_OK;
  }
  double* r = malloc(sizeof(double) * (size_t)n);
  double* z = malloc(sizeof(double) * (size_t)n);
  double* p = malloc(sizeof(double) * (size_t)n);
  double* ap = malloc(sizeof(double) * (size_t)n);
  if (x0) {
    memcpy(x, x0, sizeof(double) * (size_t)n);
    csr_mul(a, x, r);
    for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
  } else {
    memset(x, 0, sizeof(double) * (size_t)n);
    memcpy(r, b, sizeof(double) * (size_t)n);
  }
  double rel = sqrt(vdot(r, r, n)) / bnorm, zr_prev = 0.0;
  hist[nh++] = rel;
  *final_relres = rel;
  if (rel <= tol) {
    *converged = 1;
  } else {
    for (int it = 1; it <= max_iter; ++it) {
      memset(z, 0, sizeof(double) * (size_t)n);
      cycle(s, s->nlev - 1, z, r, gamma, pre, post);
      const double zr = vdot(z, r, n);
      if (!(zr > 0.0)) {
        snprintf(msg, sizeof msg,
                 "preconditioner is not positive definite: z^T r = %f at iteration %d", zr, it);
        set_err(err, errlen, msg);
        st = ST_PRECOND;
        break;
      }
      if (it == 1) {
        memcpy(p, z, sizeof(double) * (size_t)n);
      } else {
        const double beta = zr / zr_prev;
        for (int i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
      }
      zr_prev = zr;
      csr_mul(a, p, ap);
      const double pap = vdot(p, ap, n);
      if (!(pap > 0.0)) {
        snprintf(msg, sizeof msg, "PCG breakdown: p^T A p = %f at iteration %d", pap, it);
        set_err(err, errlen, msg);
        st = ST_DEF;
        break;
      }
      const double alpha = zr / pap;
      for (int i = 0; i < n; ++i) x[i] += alpha * p[i];
      for (int i = 0; i < n; ++i) r[i] += -alpha * ap[i];
      rel = sqrt(vdot(r, r, n)) / bnorm;
      *iters = it;
      *final_relres = rel;
      hist[nh++] = rel;
      if (rel <= tol || rel == 0.0) {
        *converged = 1;
        break;
      }
    }
  }
  *hist_len = nh;
  free(r);
  free(z);
  free(p);
  free(ap);
  s->t_pcg = now_s() - t0;
  return st;
}

void orc_system_times(void* h, double* out3) {
  Sys* s = h;
  out3[0] = s->t_asm;
  out3[1] = s->t_setup;
  out3[2] = s->t_pcg;
}

/* u^T K u with the assembled (eliminated) matrix: fem.cpp:284-290 */
double orc_system_compliance(void* h, const double* u) {
  Sys* s = h;
  double* y = malloc(sizeof(double) * (size_t)s->n);
  csr_mul(&s->fine, u, y);
  const double c = vdot(u, y, s->n);
  free(y);
  return c;
}

void orc_system_destroy(void* h) {
  Sys* s = h;
  if (!s) return;
  if (s->nlev) {
    s->mat[s->nlev - 1].off = NULL; /* alias of fine; freed below */
    for (int l = 0; l + 1 < s->nlev; ++l) {
      csr_free(&s->mat[l]);
      prol_free(&s->pr[l]);
    }
    chol_free(&s->coarse);
    free(s->mat);
    free(s->pr);
    free(s->lv);
  }
  csr_free(&s->fine);
  free(s->rhs);
  free(s);
}

/* ------------------------------------------------------------ consumers -- */

/* u_e^T khat u_e per element: fem.cpp:292-318 */
int orc_element_energies(int nx, int ny, const double* u, double nu, double* out) {
  double k[64];
  orc_element_stiffness(1.0, nu, k);
  for (int ex = 0; ex < nx; ++ex)
    for (int ey = 0; ey < ny; ++ey) {
      const int nd[4] = {ex * (ny + 1) + ey, (ex + 1) * (ny + 1) + ey,
                         (ex + 1) * (ny + 1) + ey + 1, ex * (ny + 1) + ey + 1};
      double ue[8];
      for (int a = 0; a < 4; ++a) {
        ue[2 * a] = u[2 * nd[a]];
        ue[2 * a + 1] = u[2 * nd[a] + 1];
      }
      double s = 0.0;
      for (int a = 0; a < 8; ++a) {
        double row = 0.0;
        for (int b = 0; b < 8; ++b) row += k[a * 8 + b] * ue[b];
        s += ue[a] * row;
      }
      out[ex * ny + ey] = s;
    }
  return ST_OK;
}

/* E_e = sum_i alpha_i^p E_i: density.cpp:68-85 */
/* std::mt19937_64 (the generator of the reference's oracle::Rng,
 * tests/oracles.hpp:15-36) restated in C: the standard's 64-bit Mersenne
 * twister parameters, seeded by the standard's recurrence. */
typedef struct {
  uint64_t mt[312];
  int idx;
} Mt64;

static void mt64_seed(Mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(Mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* oracle::Rng::uniform (oracles.hpp:21-23) */
static double mt64_uniform(Mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; }

/* BASELINE c1/c4 densities: element-major, nmat fractions
 * U(0,1), divided by their sum when it exceeds 1, void = remainder */
void orc_density_iid(int nx, int ny, int nmat, unsigned long long seed, double* alpha) {
  Mt64* g = (Mt64*)malloc(sizeof(Mt64));
  mt64_seed(g, seed);
  const long ne = (long)nx * ny;
  for (long e = 0; e < ne; ++e) {
    double* a = alpha + e * (nmat + 1);
    double s = 0.0;
    for (int m = 0; m < nmat; ++m) {
      a[m] = mt64_uniform(g);
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
  free(g);
}

/* BASELINE c2 checkerboard: one phase per block x block tile (x-major,
 * oracle::Rng::index, oracles.hpp:24), one-hot */
void orc_density_checker(int nx, int ny, int block, int nphases, unsigned long long seed, double* alpha) {
  Mt64* g = (Mt64*)malloc(sizeof(Mt64));
  mt64_seed(g, seed);
  memset(alpha, 0, sizeof(double) * (size_t)nx * ny * nphases);
  for (int i = 0; i < (nx + block - 1) / block; ++i)
    for (int j = 0; j < (ny + block - 1) / block; ++j) {
      const int ph = (int)(mt64_next(g) % (uint64_t)nphases);
      for (int ex = i * block; ex < nx && ex < (i + 1) * block; ++ex)
        for (int ey = j * block; ey < ny && ey < (j + 1) * block; ++ey)
          alpha[((long)ex * ny + ey) * nphases + ph] = 1.0;
    }
  free(g);
}

void orc_effective_moduli(int nx, int ny, int np, const double* alpha,
                          const double* pm, double pen, double* out) {
  const long ne = (long)nx * ny;
  for (long e = 0; e < ne; ++e) {
    double v = 0.0;
    for (int i = 0; i < np; ++i) v += pow(alpha[e * np + i], pen) * pm[i];
    out[e] = v;
  }
}

/* -p alpha^(p-1) E0 u_e^T khat u_e: mto.cpp:61-85 */
int orc_sensitivities(int nx, int ny, int np, const double* alpha, const double* pm,
                      double pen, double nu, const double* u, double* out) {
  const long ne = (long)nx * ny;
  double* en = malloc(sizeof(double) * (size_t)ne);
  orc_element_energies(nx, ny, u, nu, en);
  for (int i = 0; i < np; ++i)
    for (long e = 0; e < ne; ++e)
      out[i * ne + e] = -pen * pow(alpha[e * np + i], pen - 1.0) * pm[i] * en[e];
  free(en);
  return ST_OK;
}

/* density-weighted cone sensitivity filter: mto.cpp:87-117 */
int orc_filter(int nx, int ny, int np, const double* alpha, int phase, double radius,
               const double* raw, double* out) {
  const long ne = (long)nx * ny;
  if (radius <= 1.0) {
    memcpy(out, raw, sizeof(double) * (size_t)ne);
    return ST_OK;
  }
  const int reach = (int)ceil(radius) - 1;
  for (int ex = 0; ex < nx; ++ex)
    for (int ey = 0; ey < ny; ++ey) {
      double acc = 0.0, ws = 0.0;
      const int x0 = ex - reach < 0 ? 0 : ex - reach, x1 = ex + reach > nx - 1 ? nx - 1 : ex + reach;
      const int y0 = ey - reach < 0 ? 0 : ey - reach, y1 = ey + reach > ny - 1 ? ny - 1 : ey + reach;
      for (int jx = x0; jx <= x1; ++jx)
        for (int jy = y0; jy <= y1; ++jy) {
          const double w = radius - sqrt((double)((ex - jx) * (ex - jx) + (ey - jy) * (ey - jy)));
          if (w <= 0.0) continue;
          const long j = (long)jx * ny + jy;
          acc += w * alpha[j * np + phase] * raw[j];
          ws += w;
        }
      const long e = (long)ex * ny + ey;
      out[e] = acc / (alpha[e * np + phase] * ws);
    }
  return ST_OK;
}

/* std::max / std::min / clamp exactly as <algorithm> evaluates them (mto.cpp:16) */
static double smax(double a, double b) { return (a < b) ? b : a; }
static double smin(double a, double b) { return (b < a) ? b : a; }
static double sclamp(double v, double lo, double hi) { return smin(hi, smax(lo, v)); }

/* One OC exchange between phases a and b (oc_update_pair, mto.cpp:142-227),
 * in place on the element-major density alpha[e * np + phase]; move is the
 * per-element move limit. Returns ST_MULTIPLIER when the volume target is
 * missed after 101 bisection steps. */
int orc_oc_update_pair(long ne, int np, double floor_eps, double* alpha, int pa, int pb,
                       const double* sa, const double* sb, double target, const double* move,
                       double damping) {
  if (pa == pb) return ST_CONFIG;
  double* gain = malloc(sizeof(double) * (size_t)ne);
  double* pair = malloc(sizeof(double) * (size_t)ne);
  double* lo = malloc(sizeof(double) * (size_t)ne);
  double* hi = malloc(sizeof(double) * (size_t)ne);
  double* cand = malloc(sizeof(double) * (size_t)ne);
  double max_gain = -1e300, max_move = 0.0;
  for (long e = 0; e < ne; ++e) {
    gain[e] = sb[e] - sa[e];
    max_gain = smax(max_gain, gain[e]);
    max_move = smax(max_move, move[e]);
    const double a = alpha[e * np + pa];
    pair[e] = a + alpha[e * np + pb];
    lo[e] = smax(floor_eps, a - move[e]);
    hi[e] = smin(pair[e] - floor_eps, a + move[e]);
  }
  const double vol_tol = 1e-6;
  int met = 0;
  if (max_gain <= 0.0) {
    double t_lo = -max_move, t_hi = max_move;
    for (int it = 0; it <= 100; ++it) {
      const double t = 0.5 * (t_lo + t_hi);
      double mean = 0.0;
      for (long e = 0; e < ne; ++e) {
        cand[e] = sclamp(alpha[e * np + pa] + t, lo[e], hi[e]);
        mean += cand[e];
      }
      mean /= ne;
      if (fabs(mean - target) <= vol_tol) {
        met = 1;
        break;
      }
      if (mean > target) t_hi = t;
      else t_lo = t;
    }
  } else {
    const double floor_gain = 1e-4 * max_gain;
    double l_lo = 1e-10, l_hi = 1e10;
    for (int it = 0; it <= 100; ++it) {
      const double lambda = sqrt(l_lo * l_hi);
      double mean = 0.0;
      for (long e = 0; e < ne; ++e) {
        const double b = smax(floor_gain, gain[e]) / lambda;
        const double a = alpha[e * np + pa];
        cand[e] = sclamp(a * pow(b, damping), lo[e], hi[e]);
        mean += cand[e];
      }
      mean /= ne;
      if (fabs(mean - target) <= vol_tol) {
        met = 1;
        break;
      }
      if (mean > target) l_lo = lambda;
      else l_hi = lambda;
    }
  }
  if (met) {
    for (long e = 0; e < ne; ++e) {
      alpha[e * np + pa] = cand[e];
      alpha[e * np + pb] = pair[e] - cand[e];
    }
  }
  free(gain);
  free(pair);
  free(lo);
  free(hi);
  free(cand);
  return met ? ST_OK : ST_MULTIPLIER;
}

/* max |a - b| over all entries (DensityField::max_change, density.cpp:60-66) */
static double max_change(const double* a, const double* b, long n) {
  double w = 0.0;
  for (long i = 0; i < n; ++i) w = smax(w, fabs(a[i] - b[i]));
  return w;
}

/* optimize() with Method::pcgmg (mto.cpp:229-354): uniform start, per outer
 * iteration assemble (effective moduli + system), build_multigrid_operators,
 * pcgmg_solve (warm start optional), compliance, sensitivities, filtered
 * sensitivities, the OC pair sweeps, the per-element move-limit adaptation
 * and the max-change convergence test. Histories hold up to max_outer
 * entries. */
int orc_optimize(int nx, int ny, int np, const double* pm, double penalty, double nu, const int* fixed,
                 int n_fixed, const int* load_dofs, const double* load_vals, int n_loads, const double* fractions,
                 double filter_radius, double filter_tol, double tol, int inner_sweeps, double move_limit,
                 double oc_damping, int warm_start, int max_outer, double density_floor, int num_coarsenings,
                 double omega, double solver_tol, int solver_max_iter, int gamma, int pre, int post,
                 double* density, double* compliance_hist, double* change_hist, int* iters_hist,
                 int* outer_iterations, long* total_iters, int* converged, char* err, int errlen) {
  const long ne = (long)nx * ny, nv = ne * np, n = 2L * (nx + 1) * (ny + 1);
  int st = ST_OK;
  for (long e = 0; e < ne; ++e)
    for (int i = 0; i < np; ++i) density[e * np + i] = fractions[i];  /* DensityField::uniform */
  double* move = malloc(sizeof(double) * (size_t)ne);
  double* last = calloc((size_t)nv, sizeof(double));
  double* before = malloc(sizeof(double) * (size_t)nv);
  double* pre_sweep = malloc(sizeof(double) * (size_t)nv);
  double* E = malloc(sizeof(double) * (size_t)ne);
  double* u = malloc(sizeof(double) * (size_t)n);
  double* x = malloc(sizeof(double) * (size_t)n);
  double* rhs = malloc(sizeof(double) * (size_t)n);
  double* hist = malloc(sizeof(double) * (size_t)(solver_max_iter + 1));
  double* raw = malloc(sizeof(double) * (size_t)nv);
  double* filt = malloc(sizeof(double) * (size_t)nv);
  for (long e = 0; e < ne; ++e) move[e] = move_limit;
  int have_u = 0;
  *outer_iterations = 0;
  *total_iters = 0;
  *converged = 0;
  for (int outer = 1; outer <= max_outer; ++outer) {
    orc_effective_moduli(nx, ny, np, density, pm, penalty, E);
    void* s = orc_system_create(nx, ny, E, nu, fixed, n_fixed, load_dofs, load_vals, n_loads, err, errlen, &st);
    if (st) break;
    int row = -1;
    st = orc_system_build_mg(s, num_coarsenings, omega, err, errlen, &row);
    if (!st) {
      orc_system_rhs(s, rhs);
      int it = 0, cv = 0, hl = 0;
      double fr = 0.0;
      st = orc_system_solve(s, rhs, (warm_start && have_u) ? u : NULL, solver_tol, solver_max_iter, gamma, pre,
                            post, x, &it, &fr, &cv, hist, &hl, err, errlen);
      if (!st) {
        memcpy(u, x, sizeof(double) * (size_t)n);
        have_u = 1;
        compliance_hist[outer - 1] = orc_system_compliance(s, u);
        iters_hist[outer - 1] = it;
        *total_iters += it;
      }
    }
    orc_system_destroy(s);
    if (st) break;
    orc_sensitivities(nx, ny, np, density, pm, penalty, nu, u, raw);
    for (int i = 0; i < np; ++i) orc_filter(nx, ny, np, density, i, filter_radius, raw + i * ne, filt + i * ne);
    memcpy(before, density, sizeof(double) * (size_t)nv);
    for (int a = 0; a < np - 1 && !st; ++a)
      for (int b = a + 1; b < np && !st; ++b)
        for (int sweep = 0; sweep < inner_sweeps; ++sweep) {
          memcpy(pre_sweep, density, sizeof(double) * (size_t)nv);
          st = orc_oc_update_pair(ne, np, density_floor, density, a, b, filt + a * ne, filt + b * ne, fractions[a],
                                  move, oc_damping);
          if (st) {
            if (err && errlen > 0)
              snprintf(err, (size_t)errlen, "volume target %f for phase %d is unreachable under the current bounds",
                       fractions[a], a + 1);
            break;
          }
          if (max_change(density, pre_sweep, nv) <= filter_tol) break;
        }
    if (st) break;
    for (long e = 0; e < ne; ++e) {
      int flipped = 0, moved = 0;
      for (int i = 0; i < np; ++i) {
        const double delta = density[e * np + i] - before[e * np + i];
        double* l = &last[e * np + i];
        if (fabs(delta) > 1e-12) moved = 1;
        if (delta * *l < -1e-12) flipped = 1;
        *l = delta;
      }
      if (flipped) move[e] = smax(1e-4, 0.5 * move[e]);
      else if (moved) move[e] = smin(move_limit, 1.05 * move[e]);
    }
    const double change = max_change(density, before, nv);
    change_hist[outer - 1] = change;
    *outer_iterations = outer;
    if (change <= tol) {
      *converged = 1;
      break;
    }
  }
  free(move);
  free(last);
  free(before);
  free(pre_sweep);
  free(E);
  free(u);
  free(x);
  free(rhs);
  free(hist);
  free(raw);
  free(filt);
  return st;
}

/* ------------------------------------------------------------- poisson -- */

/* poisson_element_matrix / poisson_mass_matrix: 2x2 Gauss on the unit
 * square, upper triangle accumulated then mirrored (fem.cpp:37-81) */
void orc_poisson_matrices(double* k, double* m) {
  const double g = 0.57735026918962576451;
  const double pts[2] = {-g, g};
  memset(k, 0, 16 * sizeof(double));
  memset(m, 0, 16 * sizeof(double));
  for (int qa = 0; qa < 2; ++qa)
    for (int qb = 0; qb < 2; ++qb) {
      const double xi = pts[qa], eta = pts[qb];
      const double dx[4] = {2.0 * (-(1.0 - eta) / 4.0), 2.0 * ((1.0 - eta) / 4.0), 2.0 * ((1.0 + eta) / 4.0),
                            2.0 * (-(1.0 + eta) / 4.0)};
      const double dy[4] = {2.0 * (-(1.0 - xi) / 4.0), 2.0 * (-(1.0 + xi) / 4.0), 2.0 * ((1.0 + xi) / 4.0),
                            2.0 * ((1.0 - xi) / 4.0)};
      const double nv[4] = {(1.0 - xi) * (1.0 - eta) / 4.0, (1.0 + xi) * (1.0 - eta) / 4.0,
                            (1.0 + xi) * (1.0 + eta) / 4.0, (1.0 - xi) * (1.0 + eta) / 4.0};
      for (int i = 0; i < 4; ++i)
        for (int j = i; j < 4; ++j) {
          k[i * 4 + j] += 0.25 * (dx[i] * dx[j] + dy[i] * dy[j]);
          m[i * 4 + j] += 0.25 * nv[i] * nv[j];
        }
    }
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < i; ++j) {
      k[i * 4 + j] = k[j * 4 + i];
      m[i * 4 + j] = m[j * 4 + i];
    }
}

/* assemble_poisson (fem.cpp:232-276): the Q4 Laplacian with the consistent
 * load -M f, every boundary node fixed (identity row, rhs 0) */
void* orc_poisson_create(int nx, int ny, const double* source, char* err, int errlen, int* status) {
  (void)err;
  (void)errlen;
  const double t0 = now_s();
  const int n = (nx + 1) * (ny + 1);
  double k[16], m[16];
  orc_poisson_matrices(k, m);
  int* fc = calloc((size_t)n, sizeof(int));
  for (int x = 0; x <= nx; ++x)
    for (int y = 0; y <= ny; ++y)
      if (x == 0 || y == 0 || x == nx || y == ny) fc[x * (ny + 1) + y] = 1;
  Sys* s = calloc(1, sizeof(Sys));
  s->nx = nx;
  s->ny = ny;
  s->n = n;
  s->dpn = 1;
  Csr* out = &s->fine;
  out->n = n;
  out->off = malloc(sizeof(int) * (size_t)(n + 1));
  out->col = malloc(sizeof(int) * (size_t)n * 9);
  out->val = malloc(sizeof(double) * (size_t)n * 9);
  int q = 0;
  out->off[0] = 0;
  for (int x = 0; x <= nx; ++x)
    for (int y = 0; y <= ny; ++y) {
      const int row = x * (ny + 1) + y;
      if (fc[row]) {
        out->col[q] = row;
        out->val[q++] = 1.0;
        out->off[row + 1] = q;
        continue;
      }
      for (int x2 = x - 1; x2 <= x + 1; ++x2) {
        if (x2 < 0 || x2 > nx) continue;
        for (int y2 = y - 1; y2 <= y + 1; ++y2) {
          if (y2 < 0 || y2 > ny) continue;
          const int colid = x2 * (ny + 1) + y2;
          if (fc[colid]) continue;
          double v = 0.0;
          for (int ex = x - 1; ex <= x; ++ex) {
            if (ex < 0 || ex >= nx || x2 - ex < 0 || x2 - ex > 1) continue;
            for (int ey = y - 1; ey <= y; ++ey) {
              if (ey < 0 || ey >= ny || y2 - ey < 0 || y2 - ey > 1) continue;
              v += k[corner(x - ex, y - ey) * 4 + corner(x2 - ex, y2 - ey)];
            }
          }
          out->col[q] = colid;
          out->val[q++] = v;
        }
      }
      out->off[row + 1] = q;
    }
  s->rhs = calloc((size_t)n, sizeof(double));
  for (int ex = 0; ex < nx; ++ex)
    for (int ey = 0; ey < ny; ++ey) {
      const int nd[4] = {ex * (ny + 1) + ey, (ex + 1) * (ny + 1) + ey, (ex + 1) * (ny + 1) + ey + 1,
                         ex * (ny + 1) + ey + 1};
      for (int a = 0; a < 4; ++a) {
        double load = 0.0;
        for (int b = 0; b < 4; ++b) load += m[a * 4 + b] * source[nd[b]];
        s->rhs[nd[a]] -= load;
      }
    }
  for (int i = 0; i < n; ++i)
    if (fc[i]) s->rhs[i] = 0.0;
  free(fc);
  s->t_asm = now_s() - t0;
  *status = ST_OK;
  return s;
}
