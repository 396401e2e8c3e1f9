// Poisson pCGMG on the device (the paper's Table 1
// path): -lap(u) = -f on a Q4 grid with 1 dof per node and every boundary
// node fixed (assemble_poisson, fem.cpp:232-276), solved by the same PCG with
// a Galerkin geometric-multigrid preconditioner as the elasticity system
// (pcgmg_solve, solvers.cpp:516-530).
//
// Layout: scalar fields (one double per node) in the padded column-major
// layout of tmg_device.cuh. Every level stores its operator as a symmetric
// nine-point stencil, 5 doubles per node in SoA planes (centre, N, SE, E,
// NE; the other four read from the neighbour): the fine level is assembled
// on the device from the 4x4 Laplacian element matrix with the identity rows
// of the boundary, the coarse ones by the Galerkin product (1/4) P^T A P, the
// coarsest by a dense Cholesky factor and explicit inverse. Kernels are one
// thread per node (the paper's meshes are small; every pass is L2-resident),
// and one PCG iteration is one CUDA graph.
//
// Included at the end of tmg_gpu.cu (one translation unit: the shared
// kernels of tmg_kernels.cuh are defined once).
#pragma once

namespace tmgp {

using namespace tmg;

constexpr int kPPlanes = 5;
constexpr int kPT = 128;  // threads per block (y-contiguous)

struct PLevel {
  Grid g{};
  double* S = nullptr;  // kPPlanes planes of g.size
  double* u[2] = {nullptr, nullptr};
  double* f = nullptr;
  double* r = nullptr;
  int cur = 0;
};

__device__ __forceinline__ bool on_mesh(const Grid& g, int x, int y) {
  return x >= 0 && x <= g.nx && y >= 0 && y <= g.ny;
}

// corner of offset (dx, dy) in {0,1}^2 of an element, CCW from lower left
// (fem.cpp:83-86)
__device__ __forceinline__ int p_corner(int dx, int dy) { return dy ? (dx ? 2 : 3) : (dx ? 1 : 0); }

// Fine operator: Z K Z + I_boundary (fem.cpp:89-106, 232-276); a value is
// the sum over the shared elements in element order (ex outer, ey inner),
// as the reference's stable-sorted triplets sum it.
__global__ void k_p_fine_stencil(Grid g, const double* __restrict__ k16, double* __restrict__ S) {
  const int y = blockIdx.x * kPT + threadIdx.x, x = blockIdx.y;
  if (x > g.nx || y > g.ny) return;
  const long i = g.idx(x, y);
  auto fixed = [&](int xx, int yy) { return xx == 0 || yy == 0 || xx == g.nx || yy == g.ny; };
  const int off[kPPlanes][2] = {{0, 0}, {0, 1}, {1, -1}, {1, 0}, {1, 1}};
  for (int p = 0; p < kPPlanes; ++p) {
    const int x2 = x + off[p][0], y2 = y + off[p][1];
    double v = 0.0;
    if (fixed(x, y)) {
      v = (p == 0) ? 1.0 : 0.0;
    } else if (on_mesh(g, x2, y2) && !fixed(x2, y2)) {
      for (int ex = x - 1; ex <= x; ++ex) {
        if (ex < 0 || ex >= g.nx || x2 - ex < 0 || x2 - ex > 1) continue;
        for (int ey = y - 1; ey <= y; ++ey) {
          if (ey < 0 || ey >= g.ny || y2 - ey < 0 || y2 - ey > 1) continue;
          v += k16[p_corner(x - ex, y - ey) * 4 + p_corner(x2 - ex, y2 - ey)];
        }
      }
    }
    S[p * g.size + i] = v;
  }
}

// A(i, j) for j = i + (dx, dy), from the half stencil (backward entries are
// the neighbour's forward ones)
__device__ __forceinline__ double p_entry(const double* S, const Grid& g, long i, int dx, int dy) {
  const long LS = g.size;
  if (dx == 0 && dy == 0) return S[i];
  if (dx == 0 && dy == 1) return S[LS + i];
  if (dx == 1 && dy == -1) return S[2 * LS + i];
  if (dx == 1 && dy == 0) return S[3 * LS + i];
  if (dx == 1 && dy == 1) return S[4 * LS + i];
  const long j = i + static_cast<long>(dx) * g.P + dy;
  return p_entry(S, g, j, -dx, -dy);
}

// Galerkin (1/4) P^T A P (galerkin_coarse_matrix, solvers.cpp:397-458) as a
// gather over the 3x3 fine children i of coarse node I and their 3x3 fine
// neighbours j, for the five forward coarse neighbours J of I.
__global__ void k_p_galerkin(const double* __restrict__ Sf, Grid fg, Grid cg, double* __restrict__ Sc) {
  const int Y = blockIdx.x * kPT + threadIdx.x, X = blockIdx.y;
  if (X > cg.nx || Y > cg.ny) return;
  const int off[kPPlanes][2] = {{0, 0}, {0, 1}, {1, -1}, {1, 0}, {1, 1}};
  double acc[kPPlanes] = {0.0, 0.0, 0.0, 0.0, 0.0};
  auto pw = [](int o) { return o == 0 ? 1.0 : (o == 1 || o == -1 ? 0.5 : 0.0); };
  for (int ix = -1; ix <= 1; ++ix)
    for (int iy = -1; iy <= 1; ++iy) {
      const int fx = 2 * X + ix, fy = 2 * Y + iy;
      if (!on_mesh(fg, fx, fy)) continue;
      const double wi = 0.25 * pw(ix) * pw(iy);
      const long i = fg.idx(fx, fy);
      for (int jx = -1; jx <= 1; ++jx)
        for (int jy = -1; jy <= 1; ++jy) {
          const int gx = fx + jx, gy = fy + jy;
          if (!on_mesh(fg, gx, gy)) continue;
          const double a = wi * p_entry(Sf, fg, i, jx, jy);
          // coarse parents of j: weight of J = I + off[p]
          for (int p = 0; p < kPPlanes; ++p) {
            const int dx = gx - 2 * (X + off[p][0]), dy = gy - 2 * (Y + off[p][1]);
            if (dx < -1 || dx > 1 || dy < -1 || dy > 1) continue;
            if (!on_mesh(cg, X + off[p][0], Y + off[p][1])) continue;
            acc[p] += a * pw(dx) * pw(dy);
          }
        }
    }
  const long ic = cg.idx(X, Y);
  for (int p = 0; p < kPPlanes; ++p) Sc[p * cg.size + ic] = acc[p];
}

// dense coarsest matrix in the reference dof order (node x*(ny+1)+y)
__global__ void k_p_dense(const double* __restrict__ S, Grid g, double* __restrict__ A, int n) {
  const int y = blockIdx.x * kPT + threadIdx.x, x = blockIdx.y;
  if (x > g.nx || y > g.ny) return;
  const long i = g.idx(x, y);
  const int ri = x * (g.ny + 1) + y;
  for (int dx = -1; dx <= 1; ++dx)
    for (int dy = -1; dy <= 1; ++dy) {
      if (!on_mesh(g, x + dx, y + dy)) continue;
      A[static_cast<long>(ri) * n + (x + dx) * (g.ny + 1) + y + dy] = p_entry(S, g, i, dx, dy);
    }
}

__device__ __forceinline__ double p_apply(const double* S, const Grid& g, long i, const double* x, double& d) {
  const long LS = g.size;
  const int P = g.P;
  d = S[i];
  double a = d * x[i];
  a = fma(S[LS + i], x[i + 1], a);                       // N
  a = fma(S[2 * LS + i], x[i + P - 1], a);               // SE
  double b = S[3 * LS + i] * x[i + P];                   // E
  b = fma(S[4 * LS + i], x[i + P + 1], b);               // NE
  double c = S[LS + i - 1] * x[i - 1];                   // S  = N of (x, y-1)
  c = fma(S[2 * LS + i - P + 1], x[i - P + 1], c);       // NW = SE of (x-1, y+1)
  b = fma(S[3 * LS + i - P], x[i - P], b);               // W  = E of (x-1, y)
  c = fma(S[4 * LS + i - P - 1], x[i - P - 1], c);       // SW = NE of (x-1, y-1)
  return (a + b) + c;
}

// x_out = x + omega (f - A x) / d (jacobi_sweep, solvers.cpp:30-37); ZERO: x = 0
template <bool ZERO>
__global__ void k_p_sweep(const double* __restrict__ S, Grid g, const double* __restrict__ xin,
                          double* __restrict__ xout, const double* __restrict__ f, double omega) {
  const int y = blockIdx.x * kPT + threadIdx.x, x = blockIdx.y;
  if (x > g.nx || y > g.ny) return;
  const long i = g.idx(x, y);
  if (ZERO) {
    xout[i] = omega * f[i] / S[i];
  } else {
    double d;
    const double ax = p_apply(S, g, i, xin, d);
    xout[i] = xin[i] + omega * (f[i] - ax) / d;
  }
}

__global__ void k_p_residual(const double* __restrict__ S, Grid g, const double* __restrict__ x,
                             const double* __restrict__ f, double* __restrict__ r) {
  const int y = blockIdx.x * kPT + threadIdx.x, xx = blockIdx.y;
  if (xx > g.nx || y > g.ny) return;
  const long i = g.idx(xx, y);
  double d;
  r[i] = f[i] - p_apply(S, g, i, x, d);
}

// f_c = (1/4) P^T r (restrict, grid.cpp:122-142)
__global__ void k_p_restrict(Grid cg, Grid fg, const double* __restrict__ r, double* __restrict__ fc) {
  const int Y = blockIdx.x * kPT + threadIdx.x, X = blockIdx.y;
  if (X > cg.nx || Y > cg.ny) return;
  const long c = fg.idx(2 * X, 2 * Y);
  const double w[3] = {0.5, 1.0, 0.5};
  double s = 0.0;
  for (int dx = -1; dx <= 1; ++dx)
    for (int dy = -1; dy <= 1; ++dy) s = fma(0.25 * w[dx + 1] * w[dy + 1], r[c + dx * fg.P + dy], s);
  fc[cg.idx(X, Y)] = s;
}

// x (+)= P u_c (prolongate, grid.cpp:98-120)
template <bool ADD>
__global__ void k_p_prolong(Grid fg, Grid cg, const double* __restrict__ uc, double* __restrict__ x) {
  const int y = blockIdx.x * kPT + threadIdx.x, xx = blockIdx.y;
  if (xx > fg.nx || y > fg.ny) return;
  const int X0 = xx >> 1, Y0 = y >> 1;
  const bool ox = xx & 1, oy = y & 1;
  const long c = cg.idx(X0, Y0);
  double s;
  if (!ox && !oy) s = uc[c];
  else if (ox && !oy) s = 0.5 * uc[c] + 0.5 * uc[c + cg.P];
  else if (!ox && oy) s = 0.5 * uc[c] + 0.5 * uc[c + 1];
  else s = 0.25 * uc[c] + 0.25 * uc[c + 1] + 0.25 * uc[c + cg.P] + 0.25 * uc[c + cg.P + 1];
  const long i = fg.idx(xx, y);
  x[i] = ADD ? x[i] + s : s;
}

__global__ void k_p_coarse_solve(const double* __restrict__ Ainv, int n, Grid g, const double* __restrict__ f,
                                 double* __restrict__ u) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int rows = g.ny + 1;
  double s = 0.0;
  for (int m = 0; m < n; ++m) s = fma(Ainv[static_cast<long>(m) * n + k], f[g.idx(m / rows, m % rows)], s);
  u[g.idx(k / rows, k % rows)] = s;
}

// ---- PCG vector kernels (flat over the padded arrays; padding holds 0)
__global__ void __launch_bounds__(kRedThreads) k_p_dot(const double* __restrict__ a, const double* __restrict__ b,
                                                     long n, double* partials, unsigned* ticket, RedOp op,
                                                     PcgState* st, HostMirror* hm, double* out) {
  double s = 0.0;
  for (long k = blockIdx.x * static_cast<long>(kRedThreads) + threadIdx.x; k < n;
       k += static_cast<long>(gridDim.x) * kRedThreads)
    s = fma(a[k], b[k], s);
  finish_reduction<kRedThreads>(s, partials, ticket, gridDim.x, op, st, hm, out);
}

// p = z + beta p (beta = 0 on the first iteration), Ap = A p, p.Ap
__global__ void __launch_bounds__(kPT) k_p_pupd(const double* __restrict__ S, Grid g, const double* __restrict__ z,
                                                double* __restrict__ p, double* __restrict__ pn,
                                                double* __restrict__ ap, double* partials, unsigned* ticket,
                                                PcgState* st, HostMirror* hm) {
  const int y = blockIdx.x * kPT + threadIdx.x, x = blockIdx.y;
  double part = 0.0;
  if (x <= g.nx && y <= g.ny) {
    const long i = g.idx(x, y);
    double d;
    const double v = p_apply(S, g, i, pn, d);
    ap[i] = v;
    part = pn[i] * v;
  }
  (void)z;
  (void)p;
  finish_reduction<kPT>(part, partials, ticket, gridDim.x * gridDim.y, kRedPap, st, hm, nullptr);
}

__global__ void k_p_newp(const double* __restrict__ z, const double* __restrict__ p, double* __restrict__ pn, long n,
                         const PcgState* st) {
  const double beta = st->beta;
  for (long k = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<long>(gridDim.x) * blockDim.x)
    pn[k] = z[k] + beta * p[k];
}

__global__ void __launch_bounds__(kRedThreads) k_p_update_xr(double* __restrict__ x, double* __restrict__ r,
                                                           const double* __restrict__ p,
                                                           const double* __restrict__ ap, long n, double* partials,
                                                           unsigned* ticket, PcgState* st, HostMirror* hm) {
  const double alpha = st->alpha;
  double s = 0.0;
  for (long k = blockIdx.x * static_cast<long>(kRedThreads) + threadIdx.x; k < n;
       k += static_cast<long>(gridDim.x) * kRedThreads) {
    x[k] += alpha * p[k];
    r[k] += -alpha * ap[k];
    s = fma(r[k], r[k], s);
  }
  finish_reduction<kRedThreads>(s, partials, ticket, gridDim.x, kRedRr, st, hm, nullptr);
}

}  // namespace tmgp

struct tmg_poisson_handle {
  int device = 0;
  int nx = 0, ny = 0, nc = 0;
  cudaStream_t stream = nullptr;
  std::vector<tmgp::PLevel> lev;
  double omega = 0.6;
  bool have_setup = false;
  int n0 = 0;
  double *A0 = nullptr, *LiT = nullptr, *Ainv = nullptr, *k16 = nullptr;
  int* bad_row = nullptr;
  double *x = nullptr, *rv = nullptr, *b = nullptr, *p[2] = {nullptr, nullptr}, *ap = nullptr;
  double* partials = nullptr;
  unsigned* ticket = nullptr;
  PcgState* st = nullptr;
  HostMirror* hm = nullptr;
  HostMirror* hm_dev = nullptr;
  double* scal = nullptr;
  double* scal_host = nullptr;
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  int g_gamma = -1, g_pre = -1, g_post = -1;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  double last_ms = 0.0;
  std::string err;
};

namespace {

using PH = tmg_poisson_handle;

dim3 p_grid(const Grid& g) { return dim3((g.ny + 1 + tmgp::kPT - 1) / tmgp::kPT, g.nx + 1); }

template <class F>
int p_guarded(PH* h, F&& fn) {
  if (!h) return TMG_ERR_DIMENSION;
  try {
    CK(cudaSetDevice(h->device));
    fn();
    h->err.clear();
    return TMG_OK;
  } catch (const TmgError& e) {
    h->err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    h->err = e.what();
    return TMG_ERR_CUDA;
  }
}

void p_upload(cudaStream_t s, double* d, const double* host, const Grid& g) {
  CK(cudaMemcpy2DAsync(d + g.idx(0, 0), sizeof(double) * g.P, host, sizeof(double) * (g.ny + 1),
                       sizeof(double) * (g.ny + 1), g.nx + 1, cudaMemcpyHostToDevice, s));
}
void p_download(cudaStream_t s, double* host, const double* d, const Grid& g) {
  CK(cudaMemcpy2DAsync(host, sizeof(double) * (g.ny + 1), d + g.idx(0, 0), sizeof(double) * g.P,
                       sizeof(double) * (g.ny + 1), g.nx + 1, cudaMemcpyDeviceToHost, s));
}

void p_free(PH* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (auto& gx : h->graph)
    if (gx) cudaGraphExecDestroy(gx);
  for (size_t l = 0; l < h->lev.size(); ++l) {
    auto& L = h->lev[l];
    for (void* q : {static_cast<void*>(L.S), static_cast<void*>(L.u[0]), static_cast<void*>(L.u[1]),
                    static_cast<void*>(L.r)})
      cudaFree(q);
    if (l + 1 < h->lev.size()) cudaFree(L.f);  // the finest f aliases the residual
  }
  for (void* q : {static_cast<void*>(h->A0), static_cast<void*>(h->LiT), static_cast<void*>(h->Ainv),
                  static_cast<void*>(h->k16), static_cast<void*>(h->bad_row), static_cast<void*>(h->x),
                  static_cast<void*>(h->rv), static_cast<void*>(h->b), static_cast<void*>(h->p[0]),
                  static_cast<void*>(h->p[1]), static_cast<void*>(h->ap), static_cast<void*>(h->partials),
                  static_cast<void*>(h->ticket), static_cast<void*>(h->st), static_cast<void*>(h->scal)})
    cudaFree(q);
  if (h->hm) cudaFreeHost(h->hm);
  if (h->scal_host) cudaFreeHost(h->scal_host);
  for (auto e : h->ev)
    if (e) cudaEventDestroy(e);
  if (h->stream) cudaStreamDestroy(h->stream);
}

// one gamma-cycle at level l (mg_cycle, solvers.cpp:483-514); zero: u = 0 on entry
void p_cycle(PH* h, int l, bool zero, int gamma, int pre, int post) {
  using namespace tmgp;
  PLevel& L = h->lev[l];
  if (l == 0) {
    k_p_coarse_solve<<<(h->n0 + 127) / 128, 128, 0, h->stream>>>(h->Ainv, h->n0, L.g, L.f, L.u[L.cur]);
    CKL();
    return;
  }
  auto cur = [&] { return L.u[L.cur]; };
  auto nxt = [&] { return L.u[L.cur ^ 1]; };
  for (int s = 0; s < pre; ++s) {
    if (zero) k_p_sweep<true><<<p_grid(L.g), kPT, 0, h->stream>>>(L.S, L.g, nullptr, nxt(), L.f, h->omega);
    else k_p_sweep<false><<<p_grid(L.g), kPT, 0, h->stream>>>(L.S, L.g, cur(), nxt(), L.f, h->omega);
    CKL();
    L.cur ^= 1;
    zero = false;
  }
  PLevel& C = h->lev[l - 1];
  if (zero) {
    k_p_restrict<<<p_grid(C.g), kPT, 0, h->stream>>>(C.g, L.g, L.f, C.f);
  } else {
    k_p_residual<<<p_grid(L.g), kPT, 0, h->stream>>>(L.S, L.g, cur(), L.f, L.r);
    CKL();
    k_p_restrict<<<p_grid(C.g), kPT, 0, h->stream>>>(C.g, L.g, L.r, C.f);
  }
  CKL();
  const int visits = (l == h->nc) ? 1 : gamma;  // gamma forced to 1 at the finest level
  for (int t = 0; t < visits; ++t) p_cycle(h, l - 1, t == 0, gamma, pre, post);
  if (zero) k_p_prolong<false><<<p_grid(L.g), kPT, 0, h->stream>>>(L.g, C.g, C.u[C.cur], cur());
  else k_p_prolong<true><<<p_grid(L.g), kPT, 0, h->stream>>>(L.g, C.g, C.u[C.cur], cur());
  CKL();
  for (int s = 0; s < post; ++s) {
    k_p_sweep<false><<<p_grid(L.g), kPT, 0, h->stream>>>(L.S, L.g, cur(), nxt(), L.f, h->omega);
    CKL();
    L.cur ^= 1;
  }
}

// one PCG iteration (solvers.cpp:360-393) as a graph; k selects the p buffers
void p_capture(PH* h, int gamma, int pre, int post) {
  using namespace tmgp;
  if (h->graph[0] && h->g_gamma == gamma && h->g_pre == pre && h->g_post == post) return;
  for (auto& gx : h->graph) {
    if (gx) cudaGraphExecDestroy(gx);
    gx = nullptr;
  }
  PLevel& F = h->lev[h->nc];
  const long n = F.g.size;
  for (int k = 0; k < 2; ++k) {
    for (auto& L : h->lev) L.cur = 0;
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    try {
      p_cycle(h, h->nc, true, gamma, pre, post);
      const double* z = F.u[F.cur];
      k_p_dot<<<kRedBlocks, kRedThreads, 0, h->stream>>>(z, h->rv, n, h->partials, h->ticket, kRedZr, h->st,
                                                        h->hm_dev, nullptr);
      CKL();
      k_p_newp<<<kRedBlocks, kRedThreads, 0, h->stream>>>(z, h->p[k], h->p[k ^ 1], n, h->st);
      CKL();
      k_p_pupd<<<p_grid(F.g), kPT, 0, h->stream>>>(F.S, F.g, z, h->p[k], h->p[k ^ 1], h->ap, h->partials,
                                                   h->ticket, h->st, h->hm_dev);
      CKL();
      k_p_update_xr<<<kRedBlocks, kRedThreads, 0, h->stream>>>(h->x, h->rv, h->p[k ^ 1], h->ap, n, h->partials,
                                                              h->ticket, h->st, h->hm_dev);
      CKL();
    } catch (...) {
      cudaStreamEndCapture(h->stream, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    CK(cudaStreamEndCapture(h->stream, &g));
    CK(cudaGraphInstantiate(&h->graph[k], g, 0));
    cudaGraphDestroy(g);
  }
  h->g_gamma = gamma;
  h->g_pre = pre;
  h->g_post = post;
}

void p_setup(PH* h, double omega) {
  using namespace tmgp;
  h->omega = omega;
  const int nc = h->nc;
  PLevel& F = h->lev[nc];
  k_p_fine_stencil<<<p_grid(F.g), kPT, 0, h->stream>>>(F.g, h->k16, F.S);
  CKL();
  for (int l = nc; l >= 1; --l) {
    k_p_galerkin<<<p_grid(h->lev[l - 1].g), kPT, 0, h->stream>>>(h->lev[l].S, h->lev[l].g, h->lev[l - 1].g,
                                                               h->lev[l - 1].S);
    CKL();
  }
  const int n = h->n0;
  PLevel& C = h->lev[0];
  CK(cudaMemsetAsync(h->A0, 0, sizeof(double) * n * n, h->stream));
  k_p_dense<<<p_grid(C.g), kPT, 0, h->stream>>>(C.S, C.g, h->A0, n);
  CKL();
  // 1 dof per node: the farthest lower neighbour (x-1, y-1) is ny + 2 back
  const int band = std::min(n - 1, C.g.ny + 2);
  const bool large = n > kDenseFactorMaxDofs;  // as on the elasticity handle (tmg_kernels.cuh)
  if (large)
    k_cholesky_band_g<<<1, kCholBandGThreads, sizeof(double) * band, h->stream>>>(h->A0, n, band, h->LiT, h->bad_row);
  else
    launch_cholesky(h->stream, h->A0, n, h->bad_row);
  CKL();
  int bad = -1;
  CK(cudaMemcpyAsync(&bad, h->bad_row, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  if (bad >= 0)
    fail(TMG_ERR_DEFINITENESS, "matrix is not positive definite: non-positive pivot at row " + std::to_string(bad),
         bad);
  if (large) {
    int RW = 32;
    while (RW < band + 1) RW *= 2;
    const int wpb = 8;
    k_lower_inverse_band<<<(n + wpb - 1) / wpb, 32 * wpb, sizeof(double) * RW * wpb, h->stream>>>(h->A0, h->LiT, n,
                                                                                                   band, RW);
    CKL();
    const int nt = (n + kGramTile - 1) / kGramTile;
    k_gram_tiled<<<dim3(nt, nt), 256, 0, h->stream>>>(h->LiT, h->Ainv, n);
    CKL();
  } else {
    const int wpb = 4;
    const size_t sm = sizeof(double) * n * wpb;
    CK(cudaFuncSetAttribute(k_lower_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
    k_lower_inverse<<<(n + wpb - 1) / wpb, 32 * wpb, sm, h->stream>>>(h->A0, h->LiT, n, n);
    CKL();
    k_gram<<<dim3((n + 127) / 128, n), 128, 0, h->stream>>>(h->LiT, h->Ainv, n);
    CKL();
  }
  CK(cudaStreamSynchronize(h->stream));
  h->have_setup = true;
}

}  // namespace

extern "C" {

int tmg_poisson_create(int nx, int ny, int num_coarsenings, int device, tmg_poisson_handle** out) {
  if (!out) return TMG_ERR_DIMENSION;
  *out = nullptr;
  // build_hierarchy validation (grid.cpp:55-80)
  if (num_coarsenings < 0) return TMG_ERR_CONFIG;
  if (nx < 1 || ny < 1) return TMG_ERR_CONFIG;
  const int f = 1 << num_coarsenings;
  if (nx % f || ny % f) return TMG_ERR_CONFIG;
  auto* h = new tmg_poisson_handle();
  h->device = device;
  h->nx = nx;
  h->ny = ny;
  h->nc = num_coarsenings;
  const int st = p_guarded(h, [&] {
    const int n0 = ((nx >> num_coarsenings) + 1) * ((ny >> num_coarsenings) + 1);
    if (n0 > kCoarsestMaxDofs)
      fail(TMG_ERR_CONFIG, "coarsest level has " + std::to_string(n0) + " dofs; at most " +
                               std::to_string(kCoarsestMaxDofs));
    if (n0 > kDenseFactorMaxDofs && (ny >> num_coarsenings) + 2 > kLargeCoarsestMaxBand)
      fail(TMG_ERR_CONFIG, "coarsest level has " + std::to_string(n0) + " dofs in columns of " +
                               std::to_string((ny >> num_coarsenings) + 1) + " nodes; at most " +
                               std::to_string(kLargeCoarsestMaxBand - 1) + " above " +
                               std::to_string(kDenseFactorMaxDofs) + " dofs");
    CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    h->lev.resize(num_coarsenings + 1);
    for (int l = 0; l <= num_coarsenings; ++l) {
      tmgp::PLevel& L = h->lev[l];
      L.g = make_grid(nx >> (num_coarsenings - l), ny >> (num_coarsenings - l), 0,
                      (nx >> (num_coarsenings - l)) + 1);
      const size_t vb = sizeof(double) * (L.g.size + kSlackNodes);
      for (double** v : {&L.u[0], &L.u[1], &L.f, &L.r}) {
        if (v == &L.f && l == num_coarsenings) continue;  // the finest f is the PCG residual
        CK(cudaMalloc(v, vb));
        CK(cudaMemsetAsync(*v, 0, vb, h->stream));
      }
      CK(cudaMalloc(&L.S, vb * tmgp::kPPlanes));
      CK(cudaMemsetAsync(L.S, 0, vb * tmgp::kPPlanes, h->stream));
    }
    tmgp::PLevel& F = h->lev[num_coarsenings];
    const size_t vb = sizeof(double) * (F.g.size + kSlackNodes);
    for (double** v : {&h->x, &h->rv, &h->b, &h->p[0], &h->p[1], &h->ap}) {
      CK(cudaMalloc(v, vb));
      CK(cudaMemsetAsync(*v, 0, vb, h->stream));
    }
    F.f = h->rv;  // the finest cycle smooths against the PCG residual
    h->n0 = n0;
    const size_t d0 = sizeof(double) * n0 * n0;
    CK(cudaMalloc(&h->A0, d0));
    CK(cudaMalloc(&h->LiT, d0));
    CK(cudaMalloc(&h->Ainv, d0));
    CK(cudaMalloc(&h->bad_row, sizeof(int)));
    const long nparts = std::max<long>(static_cast<long>(p_grid(F.g).x) * p_grid(F.g).y, kRedBlocks);
    CK(cudaMalloc(&h->partials, sizeof(double) * nparts));
    CK(cudaMalloc(&h->ticket, sizeof(unsigned)));
    CK(cudaMemsetAsync(h->ticket, 0, sizeof(unsigned), h->stream));
    CK(cudaMalloc(&h->st, sizeof(PcgState)));
    CK(cudaHostAlloc(&h->hm, sizeof(HostMirror), cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(&h->hm_dev, h->hm, 0));
    CK(cudaMalloc(&h->scal, 4 * sizeof(double)));
    CK(cudaHostAlloc(&h->scal_host, 4 * sizeof(double), cudaHostAllocDefault));
    // the 4x4 Laplacian element matrix, computed on the host like the
    // reference (fem.cpp:37-58)
    double k16[16], m16[16];
    tmg_poisson_element_matrices(k16, m16);
    CK(cudaMalloc(&h->k16, sizeof(k16)));
    CK(cudaMemcpyAsync(h->k16, k16, sizeof(k16), cudaMemcpyHostToDevice, h->stream));
    for (auto& e : h->ev) CK(cudaEventCreate(&e));
    CK(cudaStreamSynchronize(h->stream));
  });
  if (st != TMG_OK) {
    p_free(h);
    delete h;
    return st;
  }
  *out = h;
  return TMG_OK;
}

void tmg_poisson_destroy(tmg_poisson_handle* h) {
  p_free(h);
  delete h;
}

int tmg_poisson_last_error(tmg_poisson_handle* h, char* buf, int len) {
  if (!h || !buf || len <= 0) return TMG_ERR_DIMENSION;
  std::snprintf(buf, static_cast<size_t>(len), "%s", h->err.c_str());
  return TMG_OK;
}

int tmg_poisson_setup(tmg_poisson_handle* h, double omega) {
  return p_guarded(h, [&] { p_setup(h, omega); });
}

int tmg_poisson_level_values(tmg_poisson_handle* h, int level, double* planes) {
  return p_guarded(h, [&] {
    if (!h->have_setup) fail(TMG_ERR_DIMENSION, "tmg_poisson_setup first");
    if (level < 0 || level > h->nc) fail(TMG_ERR_DIMENSION, "level out of range");
    const tmgp::PLevel& L = h->lev[level];
    const long nn = static_cast<long>(L.g.nx + 1) * (L.g.ny + 1);
    for (int p = 0; p < tmgp::kPPlanes; ++p) p_download(h->stream, planes + p * nn, L.S + p * L.g.size, L.g);
    CK(cudaStreamSynchronize(h->stream));
  });
}

int tmg_poisson_vcycle(tmg_poisson_handle* h, const double* f, double* u, int gamma, int pre, int post) {
  return p_guarded(h, [&] {
    if (!h->have_setup) fail(TMG_ERR_DIMENSION, "tmg_poisson_setup first");
    tmgp::PLevel& F = h->lev[h->nc];
    for (auto& L : h->lev) L.cur = 0;
    p_upload(h->stream, F.f, f, F.g);
    p_upload(h->stream, F.u[0], u, F.g);
    const long n = static_cast<long>(h->nx + 1) * (h->ny + 1);
    const bool zero = std::all_of(u, u + n, [](double v) { return v == 0.0; });
    p_cycle(h, h->nc, zero, gamma, pre, post);
    p_download(h->stream, u, F.u[F.cur], F.g);
    CK(cudaStreamSynchronize(h->stream));
  });
}

int tmg_poisson_solve(tmg_poisson_handle* h, const double* b, const double* x0, double tol, int max_iter, int gamma,
                      int pre_sweeps, int post_sweeps, double* x, int* iterations, double* final_relres,
                      int* converged, double* seconds, double* hist, int hist_cap, int* hist_len) {
  return p_guarded(h, [&] {
    using namespace tmgp;
    if (!h->have_setup) fail(TMG_ERR_DIMENSION, "tmg_poisson_setup first");
    if (pre_sweeps != post_sweeps)
      fail(TMG_ERR_CONFIG, "pcgmg needs pre_sweeps == post_sweeps for a symmetric preconditioner");
    if (gamma != 1 && gamma != 2) fail(TMG_ERR_CONFIG, "gamma must be 1 (V-cycle) or 2 (W-cycle)");
    if (pre_sweeps < 0) fail(TMG_ERR_CONFIG, "smoothing sweep counts must be non-negative");
    p_capture(h, gamma, pre_sweeps, post_sweeps);
    PLevel& F = h->lev[h->nc];
    const long n = F.g.size;
    CK(cudaEventRecord(h->ev[0], h->stream));
    p_upload(h->stream, h->b, b, F.g);
    CK(cudaMemsetAsync(h->p[0], 0, sizeof(double) * n, h->stream));
    k_pcg_begin<<<1, 1, 0, h->stream>>>(h->st, tol, max_iter, nullptr);
    CKL();
    k_p_dot<<<kRedBlocks, kRedThreads, 0, h->stream>>>(h->b, h->b, n, h->partials, h->ticket, kRedB, h->st,
                                                      h->hm_dev, nullptr);
    CKL();
    // r = b - A x0 (x0 = 0: r = b)
    if (x0) {
      p_upload(h->stream, h->x, x0, F.g);
      k_p_residual<<<p_grid(F.g), kPT, 0, h->stream>>>(F.S, F.g, h->x, h->b, h->rv);
      CKL();
    } else {
      CK(cudaMemsetAsync(h->x, 0, sizeof(double) * n, h->stream));
      CK(cudaMemcpyAsync(h->rv, h->b, sizeof(double) * n, cudaMemcpyDeviceToDevice, h->stream));
    }
    k_p_dot<<<kRedBlocks, kRedThreads, 0, h->stream>>>(h->rv, h->rv, n, h->partials, h->ticket, kRedPlain,
                                                      nullptr, nullptr, h->scal);
    CKL();
    PcgState st0;
    CK(cudaMemcpyAsync(&st0, h->st, sizeof(PcgState), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(h->scal_host, h->scal, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    std::vector<double> hv;
    int its = 0, conv = 0;
    double rel = 0.0;
    // pcg_solve, solvers.cpp:336-395
    if (st0.bnorm == 0.0) {
      CK(cudaMemsetAsync(h->x, 0, sizeof(double) * n, h->stream));
      conv = 1;
      hv.push_back(0.0);
    } else {
      rel = std::sqrt(*h->scal_host) / st0.bnorm;
      hv.push_back(rel);
      if (rel <= tol) {
        conv = 1;
      } else {
        const volatile HostMirror* m = h->hm;
        for (int it = 1; it <= max_iter; ++it) {
          CK(cudaGraphLaunch(h->graph[(it - 1) & 1], h->stream));
          CK(cudaStreamSynchronize(h->stream));
          if (m->status == 4) {
            char buf[200];
            std::snprintf(buf, sizeof buf, "preconditioner is not positive definite: z^T r = %f at iteration %d",
                          static_cast<double>(m->zr), it);
            fail(TMG_ERR_PRECONDITIONER, buf);
          }
          if (m->status == 3) {
            char buf[200];
            std::snprintf(buf, sizeof buf, "PCG breakdown: p^T A p = %f at iteration %d",
                          static_cast<double>(m->pap), it);
            fail(TMG_ERR_DEFINITENESS, buf);
          }
          rel = m->relres;
          its = it;
          hv.push_back(rel);
          if (rel <= tol || rel == 0.0) {
            conv = 1;
            break;
          }
        }
      }
    }
    CK(cudaEventRecord(h->ev[1], h->stream));
    p_download(h->stream, x, h->x, F.g);
    CK(cudaStreamSynchronize(h->stream));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]));
    h->last_ms = ms;
    if (iterations) *iterations = its;
    if (final_relres) *final_relres = hv.back();
    if (converged) *converged = conv;
    if (seconds) *seconds = ms * 1e-3;
    const int nh = std::min<int>(static_cast<int>(hv.size()), hist_cap);
    if (hist)
      for (int i = 0; i < nh; ++i) hist[i] = hv[static_cast<size_t>(i)];
    if (hist_len) *hist_len = nh;
  });
}

}  // extern "C"
