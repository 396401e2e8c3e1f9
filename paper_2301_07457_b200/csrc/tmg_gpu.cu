// libtmg_gpu.so -- host orchestration of the B200 pCGMG solve behind the C ABI
// of include/tmg_gpu.h. One handle = one GPU, one stream, all levels resident.
//
// Per outer iteration of the reference optimizer (mto.cpp:267-283) the work is
//   setup : Galerkin hierarchy (K6) + coarsest factor/inverse (K7) on device
//   solve : PCG (K8) preconditioned by one gamma-cycle (K1-K5, K7) per
//           iteration; one PCG iteration is a captured CUDA graph, the host
//           only reads a 40-byte mirror of the PCG scalars to run the
//           reference's stopping test (solvers.cpp:388) and error checks.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/tmg_gpu.h"
#include "tmg_kernels.cuh"
#include "tmg_march.cuh"

using namespace tmg;

namespace {

struct TmgError {
  int code;
  std::string msg;
  int row;
};

[[noreturn]] void fail(int code, const std::string& msg, int row = -1) {
  throw TmgError{code, msg, row};
}

#define CK(call)                                                                     \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) fail(TMG_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define CKL()                                                                        \
  do {                                                                               \
    cudaError_t e_ = cudaGetLastError();                                             \
    if (e_ != cudaSuccess) fail(TMG_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

struct Level {
  Grid g{};
  long ndof = 0;
  double2* u[2] = {nullptr, nullptr};  // iterate (ping-pong for Jacobi)
  double2* f = nullptr;                // right-hand side of this level
  double2* res = nullptr;              // residual scratch
  double* S = nullptr;                 // stencil planes (coarse levels)
  int cur = 0;
};

dim3 node_block() { return dim3(kBX, kBY); }
dim3 node_grid(const Grid& g) {
  return dim3((g.ny + 1 + kBX - 1) / kBX, (g.nx + 1 + kBY - 1) / kBY);
}

Grid make_grid(int nx, int ny) {
  Grid g;
  g.nx = nx;
  g.ny = ny;
  // y in [-1, ny+1] at offset kOY; a multiple of 16 nodes keeps every column
  // start 16-byte aligned for the TMA bulk copies of the byte-wide mask
  g.P = ((ny + 2 + kOY) + 15) / 16 * 16;
  g.x0 = 0;
  g.ncol = nx + 1;
  g.size = static_cast<long>(g.ncol + 2 * kGX) * g.P;
  return g;
}

}  // namespace

struct tmg_gpu_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  int nx = 0, ny = 0, nc = 0;
  std::vector<Level> lev;  // lev[0] coarsest ... lev[nc] finest (grid.hpp:47)
  double* E = nullptr;
  uint8_t* M = nullptr;
  double nu = 0.3;
  double ke[64];
  bool have_problem = false, have_moduli = false, have_setup = false;
  double omega = 0.6;
  // coarsest level (K7)
  int n0 = 0;
  double *A0 = nullptr, *LiT = nullptr, *Ainv = nullptr;
  int* bad_row = nullptr;
  // PCG (K8)
  double2 *x = nullptr, *r = nullptr, *ap = nullptr, *b = nullptr, *x0 = nullptr;
  double2* pbuf[2] = {nullptr, nullptr};  // PCG directions (old / new alternate)
  double* partials = nullptr;
  unsigned* ticket = nullptr;
  PcgState* st = nullptr;
  HostMirror* hm = nullptr;      // pinned, mapped
  HostMirror* hm_dev = nullptr;  // device alias of hm
  double* scal = nullptr;        // device scalar for plain dots
  double* scal_host = nullptr;   // pinned
  bool have_solution = false;
  // captured PCG iteration
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  int g_gamma = -1, g_pre = -1, g_post = -1;
  long graph_kernels = 0;
  double2* z_final = nullptr;
  // scratch for consumers
  double* dense = nullptr;
  long dense_cap = 0;
  double* aux = nullptr;
  long aux_cap = 0;
  double* aux2 = nullptr;
  long aux2_cap = 0;
  int* iaux = nullptr;
  long iaux_cap = 0;
  // instrumentation
  long launches = 0;
  bool capturing = false;
  long capture_kernels = 0;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t uev[8] = {};
  double last_setup_ms = 0.0, last_pcg_ms = 0.0;
  std::string err;
  int err_row = -1;

  Level& fine() { return lev[nc]; }
  void count(long k = 1) {
    if (capturing) capture_kernels += k;
    else launches += k;
  }
  FineOp fine_op() const { return FineOp{E, M, lev[nc].g.P}; }
  StencilOp stencil_op(int l) const { return StencilOp{lev[l].S, lev[l].g.size, lev[l].g.P}; }
};

namespace {

using H = tmg_gpu_handle;

template <class F>
void with_op(H* h, int l, F&& fn) {
  if (l == h->nc) fn(h->fine_op());
  else fn(h->stencil_op(l));
}

double* grow(double*& p, long& cap, long need) {
  if (need > cap) {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    CK(cudaMalloc(&p, sizeof(double) * need));
    cap = need;
  }
  return p;
}

void upload_nodes(H* h, double2* d, const double* host, const Grid& g) {
  CK(cudaMemcpy2DAsync(d + g.idx(0, 0), sizeof(double2) * g.P, host, sizeof(double2) * (g.ny + 1),
                       sizeof(double2) * (g.ny + 1), g.nx + 1, cudaMemcpyHostToDevice, h->stream));
}

void download_nodes(H* h, double* host, const double2* d, const Grid& g) {
  CK(cudaMemcpy2DAsync(host, sizeof(double2) * (g.ny + 1), d + g.idx(0, 0), sizeof(double2) * g.P,
                       sizeof(double2) * (g.ny + 1), g.nx + 1, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
}

void check_level(H* h, int level) {
  if (level < 0 || level > h->nc) {
    fail(TMG_ERR_DIMENSION, "level " + std::to_string(level) + " outside [0, " +
                                std::to_string(h->nc) + "]");
  }
}

void need_setup(H* h) {
  if (!h->have_setup) fail(TMG_ERR_DIMENSION, "multigrid operators not built (call tmg_gpu_set_moduli)");
}

void free_handle(H* h) {
  cudaSetDevice(h->device);
  for (cudaGraphExec_t gx : h->graph)
    if (gx) cudaGraphExecDestroy(gx);
  for (Level& L : h->lev) {
    cudaFree(L.u[0]);
    cudaFree(L.u[1]);
    cudaFree(L.res);
    cudaFree(L.S);
    if (&L != &h->lev.back()) cudaFree(L.f);
  }
  cudaFree(h->E);
  cudaFree(h->M);
  cudaFree(h->A0);
  cudaFree(h->LiT);
  cudaFree(h->Ainv);
  cudaFree(h->bad_row);
  cudaFree(h->x);
  cudaFree(h->r);
  cudaFree(h->pbuf[0]);
  cudaFree(h->pbuf[1]);
  cudaFree(h->ap);
  cudaFree(h->b);
  cudaFree(h->x0);
  cudaFree(h->partials);
  cudaFree(h->ticket);
  cudaFree(h->st);
  cudaFree(h->scal);
  cudaFree(h->dense);
  cudaFree(h->aux);
  cudaFree(h->aux2);
  cudaFree(h->iaux);
  if (h->hm) cudaFreeHost(h->hm);
  if (h->scal_host) cudaFreeHost(h->scal_host);
  for (cudaEvent_t e : h->ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : h->uev)
    if (e) cudaEventDestroy(e);
  if (h->stream) cudaStreamDestroy(h->stream);
}

// ------------------------------------------------------------ launches --

// output columns per marching CTA: long strips amortise the prologue; short
// ones keep small grids spread over all 148 SMs
int march_tx(long rows_tiles, long cols) {
  const long want = (cols * rows_tiles + 148 * 8 - 1) / (148 * 8);
  return static_cast<int>(std::min<long>(64, std::max<long>(6, want)));
}

MarchArgs march_args(H* h, const double2* u) {
  MarchArgs a{};
  a.g = h->fine().g;
  if (h->nc > 0) a.gc = h->lev[h->nc - 1].g;
  a.u = u;
  a.E = h->E;
  a.M = h->M;
  a.omega = h->omega;
  a.partials = h->partials;
  a.ticket = h->ticket;
  a.rop = kRedNone;
  a.st = h->st;
  a.hm = h->hm_dev;
  return a;
}

template <class Stage, bool RED>
void launch_march(H* h, MarchArgs a) {
  dim3 grid;
  if constexpr (Stage::kRow0 == -1) {  // restriction: tiles of coarse rows / columns
    const long ty = (a.gc.ny + 1 + Stage::kOwned / 2 - 1) / (Stage::kOwned / 2);
    a.tx = march_tx(ty, a.gc.nx + 1);
    grid = dim3(ty, (a.gc.nx + 1 + a.tx - 1) / a.tx);
  } else {
    const long ty = (a.g.ny + 1 + Stage::kOwned - 1) / Stage::kOwned;
    a.tx = march_tx(ty, a.g.nx + 1);
    grid = dim3(ty, (a.g.nx + 1 + a.tx - 1) / a.tx);
  }
  const size_t sm = static_cast<size_t>(Stage::kSlot) * kStages;
  k_march<Stage, RED><<<grid, kMarchThreads, sm, h->stream>>>(a);
  CKL();
  h->count();
}

void apply_level(H* h, int l, const double2* x, double2* y) {
  const Level& L = h->lev[l];
  if (l == h->nc) {
    MarchArgs a = march_args(h, x);
    a.out0 = y;
    launch_march<StApply<false>, false>(h, a);
    return;
  }
  with_op(h, l, [&](auto op) {
    k_apply<decltype(op), false><<<node_grid(L.g), node_block(), 0, h->stream>>>(
        op, L.g, x, y, nullptr, nullptr, kRedNone, nullptr, nullptr, nullptr);
  });
  CKL();
  h->count();
}

// y = A x and out = x.y (reduction op `rop` updates the PCG scalars)
void apply_dot_fine(H* h, const double2* x, double2* y, RedOp rop, double* out) {
  MarchArgs a = march_args(h, x);
  a.out0 = y;
  a.rop = rop;
  a.red_out = out;
  launch_march<StApply<true>, true>(h, a);
}

// one damped-Jacobi sweep; at the finest level optionally fused with z.r
void sweep_level(H* h, int l, bool zero, const double2* xin, double2* xout, const double2* f,
                 RedOp rop = kRedNone) {
  const Level& L = h->lev[l];
  if (l == h->nc && !zero) {
    MarchArgs a = march_args(h, xin);
    a.f = f;
    a.out0 = xout;
    if (rop != kRedNone) {
      a.rop = rop;
      launch_march<StSweep<true>, true>(h, a);
    } else {
      launch_march<StSweep<false>, false>(h, a);
    }
    return;
  }
  with_op(h, l, [&](auto op) {
    if (zero)
      k_sweep<decltype(op), true><<<node_grid(L.g), node_block(), 0, h->stream>>>(op, L.g, xin, xout, f, h->omega);
    else
      k_sweep<decltype(op), false><<<node_grid(L.g), node_block(), 0, h->stream>>>(op, L.g, xin, xout, f, h->omega);
  });
  CKL();
  h->count();
}

void residual_level(H* h, int l, const double2* x, const double2* f, double2* r) {
  const Level& L = h->lev[l];
  if (l == h->nc) {
    MarchArgs a = march_args(h, x);
    a.f = f;
    a.out0 = r;
    launch_march<StResidual, false>(h, a);
    return;
  }
  with_op(h, l, [&](auto op) {
    k_residual<decltype(op)><<<node_grid(L.g), node_block(), 0, h->stream>>>(op, L.g, x, f, r);
  });
  CKL();
  h->count();
}

void restrict_level(H* h, int l, const double2* r, double2* fc) {
  k_restrict<<<node_grid(h->lev[l - 1].g), node_block(), 0, h->stream>>>(h->lev[l - 1].g, h->lev[l].g, r, fc);
  CKL();
  h->count();
}

void prolong_level(H* h, int l, const double2* uc, double2* x, bool add) {
  const Grid& fg = h->lev[l].g;
  if (add) k_prolong<true><<<node_grid(fg), node_block(), 0, h->stream>>>(fg, h->lev[l - 1].g, uc, x);
  else k_prolong<false><<<node_grid(fg), node_block(), 0, h->stream>>>(fg, h->lev[l - 1].g, uc, x);
  CKL();
  h->count();
}

void coarse_solve(H* h, const double2* f, double2* u) {
  const int nodes = h->n0 / 2;
  const int nt = 256;
  k_coarse_solve<<<(nodes + nt - 1) / nt, nt, sizeof(double) * h->n0, h->stream>>>(h->Ainv, h->n0, h->lev[0].g, f, u);
  CKL();
  h->count();
}

// One gamma-cycle at level l (mg_cycle, solvers.cpp:483-514). `zero` means
// the iterate is logically zero on entry (the reference zeroes u_coarse
// before the first visit, solvers.cpp:501, and pcgmg starts from z = 0,
// solvers.cpp:524); the buffer content is then never read. At the finest
// level the passes are the fused marching stages (tmg_march.cuh); when
// `zr_op` is set the last post-sweep also reduces z.r for PCG. Returns
// whether that reduction was fused.
bool enqueue_cycle(H* h, int l, bool zero, int gamma, int pre, int post, RedOp zr_op = kRedNone) {
  Level& L = h->lev[l];
  if (l == 0) {
    coarse_solve(h, L.f, L.u[L.cur]);
    return false;
  }
  Level& C = h->lev[l - 1];
  const bool fine = (l == h->nc);
  int s = 0;
  if (fine && zero && pre >= 2) {
    MarchArgs a = march_args(h, nullptr);
    a.f = L.f;
    a.out0 = L.u[L.cur ^ 1];
    launch_march<StSweep01, false>(h, a);
    L.cur ^= 1;
    s = 2;
    zero = false;
  }
  for (; s < pre; ++s) {
    sweep_level(h, l, zero, L.u[L.cur], L.u[L.cur ^ 1], L.f);
    L.cur ^= 1;
    zero = false;
  }
  if (zero) {
    restrict_level(h, l, L.f, C.f);  // residual of u = 0 is f
  } else if (fine) {
    MarchArgs a = march_args(h, L.u[L.cur]);
    a.f = L.f;
    a.out0 = C.f;
    launch_march<StResidRestrict, false>(h, a);
  } else {
    residual_level(h, l, L.u[L.cur], L.f, L.res);
    restrict_level(h, l, L.res, C.f);
  }
  const int visits = fine ? 1 : gamma;
  for (int t = 0; t < visits; ++t) enqueue_cycle(h, l - 1, t == 0, gamma, pre, post);
  int p = 0;
  if (fine && !zero && post >= 1) {
    MarchArgs a = march_args(h, L.u[L.cur]);
    a.uc = C.u[C.cur];
    a.f = L.f;
    a.out0 = L.u[L.cur ^ 1];
    launch_march<StProlongSweep, false>(h, a);
    L.cur ^= 1;
    p = 1;
  } else {
    prolong_level(h, l, C.u[C.cur], L.u[L.cur], !zero);
  }
  bool fused = false;
  for (; p < post; ++p) {
    const bool last = (p == post - 1);
    sweep_level(h, l, false, L.u[L.cur], L.u[L.cur ^ 1], L.f, (fine && last) ? zr_op : kRedNone);
    fused = fine && last && zr_op != kRedNone;
    L.cur ^= 1;
  }
  return fused;
}

long flat2(const Level& L) { return L.g.size; }  // double2 count of a padded field

int red_grid(long n2) {
  long b = (n2 + kRedThreads - 1) / kRedThreads;
  return static_cast<int>(b < kRedBlocks ? (b < 1 ? 1 : b) : kRedBlocks);
}

void dot(H* h, const double2* a, const double2* b, RedOp op, double* out) {
  // owned columns only: ghost columns may hold a neighbour's halo
  const Grid& g = h->fine().g;
  const long o = g.own_begin(), n2 = g.own_count();
  k_dot<<<red_grid(n2), kRedThreads, 0, h->stream>>>(a + o, b + o, n2, h->partials, h->ticket, op, h->st,
                                                     h->hm_dev, out);
  CKL();
  h->count();
}

// One PCG iteration (pcg_solve loop body, solvers.cpp:359-391) as a graph.
// Two graphs alternate the roles of the two direction buffers, because the
// fused p-update reads the old p around each node while writing the new one.
void capture_iteration(H* h, int gamma, int pre, int post) {
  if (h->graph[0] && h->g_gamma == gamma && h->g_pre == pre && h->g_post == post) return;
  for (auto& gx : h->graph) {
    if (gx) cudaGraphExecDestroy(gx);
    gx = nullptr;
  }
  const long n2 = flat2(h->fine());
  for (int k = 0; k < 2; ++k) {
    for (Level& L : h->lev) L.cur = 0;
    double2* p_old = h->pbuf[k];
    double2* p_new = h->pbuf[k ^ 1];
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    h->capturing = true;
    h->capture_kernels = 0;
    try {
      // z = M^-1 r: one cycle from z = 0 (solvers.cpp:523-527), fused with z.r
      const bool fused = enqueue_cycle(h, h->nc, true, gamma, pre, post, kRedZr);
      double2* z = h->fine().u[h->fine().cur];
      if (!fused) dot(h, z, h->r, kRedZr, nullptr);
      // p = z + beta p; Ap; pAp; alpha (solvers.cpp:367-382)
      MarchArgs a = march_args(h, z);
      a.u2 = p_old;
      a.out0 = p_new;
      a.out1 = h->ap;
      a.rop = kRedPap;
      launch_march<StPupd, true>(h, a);
      // x += alpha p; r -= alpha Ap; rr (solvers.cpp:383-386)
      const long o = h->fine().g.own_begin(), no = h->fine().g.own_count();
      k_update_xr<<<red_grid(no), kRedThreads, 0, h->stream>>>(h->x + o, h->r + o, p_new + o, h->ap + o, no,
                                                                 h->partials,
                                                                 h->ticket, h->st, h->hm_dev);
      CKL();
      h->count();
    } catch (...) {
      h->capturing = false;
      cudaStreamEndCapture(h->stream, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    h->capturing = false;
    CK(cudaStreamEndCapture(h->stream, &g));
    CK(cudaGraphInstantiate(&h->graph[k], g, 0));
    cudaGraphDestroy(g);
    h->graph_kernels = h->capture_kernels;
  }
  h->g_gamma = gamma;
  h->g_pre = pre;
  h->g_post = post;
}

// ----------------------------------------------------------------- setup --

void setup(H* h, double omega) {
  if (!h->have_problem) fail(TMG_ERR_DIMENSION, "tmg_gpu_set_problem must precede setup");
  if (!h->have_moduli) fail(TMG_ERR_DIMENSION, "no element moduli uploaded");
  h->omega = omega;
  h->have_setup = false;
  // Galerkin hierarchy, finest to coarsest (solvers.cpp:474-478)
  for (int l = h->nc; l >= 1; --l) {
    const Grid& cg = h->lev[l - 1].g;
    dim3 blk(32, 4), grd((cg.ny + 1 + 31) / 32, (cg.nx + 1 + 3) / 4);
    with_op(h, l, [&](auto op) {
      k_galerkin<decltype(op)><<<grd, blk, 0, h->stream>>>(op, h->lev[l].g, cg, h->lev[l - 1].S, cg.size);
    });
    CKL();
    h->count();
  }
  // coarsest: dense matrix -> Cholesky -> explicit symmetric inverse
  const int n = h->n0;
  const Grid& g0 = h->lev[0].g;
  CK(cudaMemsetAsync(h->A0, 0, sizeof(double) * n * n, h->stream));
  with_op(h, 0, [&](auto op) {
    k_dense_assemble<decltype(op)><<<dim3((g0.ny + 1 + 63) / 64, g0.nx + 1), 64, 0, h->stream>>>(op, g0, h->A0, n);
  });
  CKL();
  k_cholesky<<<1, 1024, 0, h->stream>>>(h->A0, n, h->bad_row);
  CKL();
  int bad = -1;
  CK(cudaMemcpyAsync(&bad, h->bad_row, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  h->count(3);
  if (bad >= 0) {
    fail(TMG_ERR_DEFINITENESS,
         "matrix is not positive definite: non-positive pivot at row " + std::to_string(bad), bad);
  }
  const int wpb = 4;
  const size_t sm = sizeof(double) * n * wpb;
  CK(cudaFuncSetAttribute(k_lower_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
  k_lower_inverse<<<(n + wpb - 1) / wpb, 32 * wpb, sm, h->stream>>>(h->A0, h->LiT, n);
  CKL();
  k_gram<<<dim3((n + 127) / 128, n), 128, 0, h->stream>>>(h->LiT, h->Ainv, n);
  CKL();
  h->count(2);
  h->have_setup = true;
}

// ----------------------------------------------------------------- solve --

struct SolveOut {
  int iterations = 0;
  double final_residual = 0.0;
  int converged = 0;
  double seconds = 0.0;
  std::vector<double> hist;
};

void solve_resident(H* h, bool use_x0, double tol, int max_iter, int gamma, int pre, int post,
                    SolveOut& o) {
  need_setup(h);
  // SolverConfig::validate subset enforced by pcgmg_solve (solvers.cpp:518-521)
  if (pre != post) {
    fail(TMG_ERR_CONFIG, "pcgmg needs pre_sweeps == post_sweeps for a symmetric preconditioner");
  }
  if (gamma != 1 && gamma != 2) fail(TMG_ERR_CONFIG, "gamma must be 1 (V-cycle) or 2 (W-cycle)");
  if (pre < 0) fail(TMG_ERR_CONFIG, "smoothing sweep counts must be non-negative");
  const Level& F = h->fine();
  const long n2 = flat2(F);
  capture_iteration(h, gamma, pre, post);
  CK(cudaEventRecord(h->ev[0], h->stream));
  dot(h, h->b, h->b, kRedB, nullptr);
  k_pcg_begin<<<1, 1, 0, h->stream>>>(h->st);
  CKL();
  h->count();
  CK(cudaMemsetAsync(h->pbuf[0], 0, sizeof(double2) * n2, h->stream));
  if (use_x0) {
    CK(cudaMemcpyAsync(h->x, h->x0, sizeof(double2) * n2, cudaMemcpyDeviceToDevice, h->stream));
    apply_level(h, h->nc, h->x, F.res);
    k_sub<<<red_grid(F.g.own_count()), kRedThreads, 0, h->stream>>>(h->b + F.g.own_begin(), F.res + F.g.own_begin(),
                                                                   h->r + F.g.own_begin(), F.g.own_count());
  } else {
    CK(cudaMemsetAsync(h->x, 0, sizeof(double2) * n2, h->stream));
    k_sub<<<red_grid(F.g.own_count()), kRedThreads, 0, h->stream>>>(h->b + F.g.own_begin(), nullptr,
                                                                   h->r + F.g.own_begin(), F.g.own_count());
  }
  CKL();
  h->count();
  dot(h, h->r, h->r, kRedPlain, h->scal);
  PcgState st0;
  CK(cudaMemcpyAsync(&st0, h->st, sizeof(PcgState), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaMemcpyAsync(h->scal_host, h->scal, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  o = SolveOut{};
  h->have_solution = true;
  // pcg_solve, solvers.cpp:336-357
  if (st0.bnorm == 0.0) {
    CK(cudaMemsetAsync(h->x, 0, sizeof(double2) * n2, h->stream));
    o.converged = 1;
    o.hist.push_back(0.0);
  } else {
    double rel = std::sqrt(*h->scal_host) / st0.bnorm;
    o.final_residual = rel;
    o.hist.push_back(rel);
    if (rel <= tol) {
      o.converged = 1;
    } else {
      for (int it = 1; it <= max_iter; ++it) {
        CK(cudaGraphLaunch(h->graph[(it - 1) & 1], h->stream));
        h->launches += h->graph_kernels;
        CK(cudaStreamSynchronize(h->stream));
        const volatile HostMirror* m = h->hm;
        const int status = m->status;
        if (status == 4) {
          char buf[200];
          std::snprintf(buf, sizeof buf,
                        "preconditioner is not positive definite: z^T r = %f at iteration %d",
                        static_cast<double>(m->zr), it);
          fail(TMG_ERR_PRECONDITIONER, buf);
        }
        if (status == 3) {
          char buf[200];
          std::snprintf(buf, sizeof buf, "PCG breakdown: p^T A p = %f at iteration %d",
                        static_cast<double>(m->pap), it);
          fail(TMG_ERR_DEFINITENESS, buf);
        }
        rel = m->relres;
        o.iterations = it;
        o.final_residual = rel;
        o.hist.push_back(rel);
        if (rel <= tol || rel == 0.0) {
          o.converged = 1;
          break;
        }
      }
    }
  }
  CK(cudaEventRecord(h->ev[1], h->stream));
  CK(cudaEventSynchronize(h->ev[1]));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]));
  h->last_pcg_ms = ms;
  o.seconds = ms * 1e-3;
}

int finish(H* h, const TmgError& e) {
  if (h) {
    h->err = e.msg;
    h->err_row = e.row;
  }
  return e.code;
}

template <class F>
int guarded(H* h, F&& fn) {
  if (!h) return TMG_ERR_DIMENSION;
  try {
    CK(cudaSetDevice(h->device));
    fn();
    h->err.clear();
    h->err_row = -1;
    return TMG_OK;
  } catch (const TmgError& e) {
    return finish(h, e);
  } catch (const std::exception& e) {
    return finish(h, TmgError{TMG_ERR_CUDA, e.what(), -1});
  }
}

void copy_out_hist(const SolveOut& o, double* history, int cap, int* len) {
  const int n = static_cast<int>(o.hist.size());
  const int m = (history && cap > 0) ? (n < cap ? n : cap) : 0;
  if (m) std::memcpy(history, o.hist.data(), sizeof(double) * m);
  if (len) *len = m;
}

}  // namespace

// =================================================================== ABI ==

extern "C" {

int tmg_gpu_create(int nx, int ny, int num_coarsenings, int dofs_per_node, int device,
                   tmg_gpu_handle** out) {
  if (!out) return TMG_ERR_DIMENSION;
  *out = nullptr;
  // build_hierarchy validation (grid.cpp:55-80)
  auto h = std::make_unique<tmg_gpu_handle>();
  h->device = device;
  auto cfg = [&](const std::string& m) {
    h->err = m;
    *out = h.release();
    return TMG_ERR_CONFIG;
  };
  if (nx < 1 || ny < 1)
    return cfg("grid must have at least one element per direction, got " + std::to_string(nx) +
               "x" + std::to_string(ny));
  if (num_coarsenings < 0) return cfg("num_coarsenings must be non-negative");
  if (dofs_per_node != 2)
    return cfg("dofs_per_node must be 2: the GPU path solves the plane-elasticity system");
  if (num_coarsenings > 24) return cfg("num_coarsenings too large");
  const int factor = 1 << num_coarsenings;
  if (nx % factor != 0)
    return cfg("nx = " + std::to_string(nx) + " is not divisible by 2^" +
               std::to_string(num_coarsenings) + " = " + std::to_string(factor));
  if (ny % factor != 0)
    return cfg("ny = " + std::to_string(ny) + " is not divisible by 2^" +
               std::to_string(num_coarsenings) + " = " + std::to_string(factor));
  const int n0 = 2 * (nx / factor + 1) * (ny / factor + 1);
  if (n0 > 2048) {
    return cfg("coarsest level has " + std::to_string(n0) +
               " dofs; the device coarse solve supports <= 2048 (add coarsenings)");
  }
  H* hp = h.get();
  const int st = guarded(hp, [&] {
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) fail(TMG_ERR_CUDA, "CUDA device " + std::to_string(device) + " not present");
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
      fail(TMG_ERR_CUDA, std::string("libtmg_gpu is built for sm_100a; device is ") + prop.name);
    }
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&hp->stream, cudaStreamNonBlocking));
    for (cudaEvent_t& e : hp->ev) CK(cudaEventCreate(&e));
    hp->nx = nx;
    hp->ny = ny;
    hp->nc = num_coarsenings;
    hp->lev.resize(num_coarsenings + 1);
    for (int l = 0; l <= num_coarsenings; ++l) {
      Level& L = hp->lev[l];
      const int s = 1 << (num_coarsenings - l);
      L.g = make_grid(nx / s, ny / s);
      L.ndof = 2L * (L.g.nx + 1) * (L.g.ny + 1);
      const size_t vb = sizeof(double2) * (L.g.size + kSlackNodes);
      CK(cudaMalloc(&L.u[0], vb));
      CK(cudaMalloc(&L.u[1], vb));
      CK(cudaMalloc(&L.res, vb));
      CK(cudaMemsetAsync(L.u[0], 0, vb, hp->stream));
      CK(cudaMemsetAsync(L.u[1], 0, vb, hp->stream));
      CK(cudaMemsetAsync(L.res, 0, vb, hp->stream));
      if (l < num_coarsenings) {
        CK(cudaMalloc(&L.f, vb));
        CK(cudaMemsetAsync(L.f, 0, vb, hp->stream));
        const size_t sb = sizeof(double) * kStencilPlanes * L.g.size;
        CK(cudaMalloc(&L.S, sb));
        CK(cudaMemsetAsync(L.S, 0, sb, hp->stream));
      }
    }
    Level& F = hp->fine();
    const size_t vb = sizeof(double2) * (F.g.size + kSlackNodes);
    for (double2** v : {&hp->x, &hp->r, &hp->pbuf[0], &hp->pbuf[1], &hp->ap, &hp->b, &hp->x0}) {
      CK(cudaMalloc(v, vb));
      CK(cudaMemsetAsync(*v, 0, vb, hp->stream));
    }
    F.f = hp->r;  // the finest cycle smooths against the PCG residual
    CK(cudaMalloc(&hp->E, sizeof(double) * (F.g.size + kSlackNodes)));
    CK(cudaMemsetAsync(hp->E, 0, sizeof(double) * (F.g.size + kSlackNodes), hp->stream));
    CK(cudaMalloc(&hp->M, F.g.size + kSlackNodes));
    CK(cudaMemsetAsync(hp->M, 0, F.g.size + kSlackNodes, hp->stream));
    hp->n0 = n0;
    CK(cudaMalloc(&hp->A0, sizeof(double) * n0 * n0));
    CK(cudaMalloc(&hp->LiT, sizeof(double) * n0 * n0));
    CK(cudaMalloc(&hp->Ainv, sizeof(double) * n0 * n0));
    CK(cudaMalloc(&hp->bad_row, sizeof(int)));
    const dim3 ng = node_grid(F.g);
    const long nparts = std::max<long>(static_cast<long>(ng.x) * ng.y, kRedBlocks);
    CK(cudaMalloc(&hp->partials, sizeof(double) * nparts));
    CK(cudaMalloc(&hp->ticket, sizeof(unsigned)));
    CK(cudaMemsetAsync(hp->ticket, 0, sizeof(unsigned), hp->stream));
    CK(cudaMalloc(&hp->st, sizeof(PcgState)));
    CK(cudaMemsetAsync(hp->st, 0, sizeof(PcgState), hp->stream));
    CK(cudaMalloc(&hp->scal, sizeof(double)));
    CK(cudaHostAlloc(&hp->hm, sizeof(HostMirror), cudaHostAllocMapped));
    std::memset(hp->hm, 0, sizeof(HostMirror));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hp->hm_dev), hp->hm, 0));
    CK(cudaHostAlloc(&hp->scal_host, sizeof(double), cudaHostAllocDefault));
    CK(cudaStreamSynchronize(hp->stream));
  });
  if (st != TMG_OK) {
    // keep only the message: the caller may read it, then destroys the handle
    const std::string msg = hp->err;
    free_handle(hp);
    h = std::make_unique<tmg_gpu_handle>();
    h->device = device;
    h->err = msg;
  }
  *out = h.release();
  return st;
}

void tmg_gpu_destroy(tmg_gpu_handle* h) {
  if (!h) return;
  free_handle(h);
  delete h;
}

int tmg_gpu_last_error(tmg_gpu_handle* h, char* buf, int len, int* row) {
  if (!h) return TMG_ERR_DIMENSION;
  if (buf && len > 0) std::snprintf(buf, len, "%s", h->err.c_str());
  if (row) *row = h->err_row;
  return TMG_OK;
}

int tmg_gpu_set_problem(tmg_gpu_handle* h, double nu, const int* fixed_dofs, int n_fixed) {
  return guarded(h, [&] {
    if (!h->stream) fail(TMG_ERR_CUDA, "handle has no device");
    const Grid& g = h->fine().g;
    const long ndof = h->fine().ndof;
    // BoundaryConditions::validate (fem.cpp:110-129)
    std::vector<int> cnt(ndof, 0);
    for (int k = 0; k < n_fixed; ++k) {
      const int d = fixed_dofs[k];
      if (d < 0 || d >= ndof)
        fail(TMG_ERR_CONFIG, "fixed dof " + std::to_string(d) + " outside [0, " + std::to_string(ndof) + ")");
      cnt[d]++;
    }
    std::vector<uint8_t> mask(g.size, 0);
    for (int x = 0; x <= g.nx; ++x)
      for (int y = 0; y <= g.ny; ++y) {
        const long node = static_cast<long>(x) * (g.ny + 1) + y;
        const int c0 = std::min(cnt[2 * node], 15), c1 = std::min(cnt[2 * node + 1], 15);
        mask[g.idx(x, y)] = static_cast<uint8_t>(c0 | (c1 << 4));
      }
    CK(cudaMemcpyAsync(h->M, mask.data(), g.size, cudaMemcpyHostToDevice, h->stream));
    h->nu = nu;
    tmg_element_stiffness(1.0, nu, h->ke);
    CK(cudaMemcpyToSymbolAsync(c_k8, h->ke, 8 * sizeof(double), 0, cudaMemcpyHostToDevice, h->stream));  // row 0
    CK(cudaMemcpyToSymbolAsync(c_ke64, h->ke, 64 * sizeof(double), 0, cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    h->have_problem = true;
    h->have_setup = false;
  });
}

int tmg_gpu_upload_moduli(tmg_gpu_handle* h, const double* moduli, long n_elem) {
  return guarded(h, [&] {
    const Grid& g = h->fine().g;
    if (n_elem != static_cast<long>(g.nx) * g.ny)
      fail(TMG_ERR_DIMENSION, "element modulus count " + std::to_string(n_elem) +
                                  " does not match grid with " +
                                  std::to_string(static_cast<long>(g.nx) * g.ny) + " elements");
    CK(cudaMemcpy2DAsync(h->E + g.idx(0, 0), sizeof(double) * g.P, moduli, sizeof(double) * g.ny,
                         sizeof(double) * g.ny, g.nx, cudaMemcpyHostToDevice, h->stream));
    h->have_moduli = true;
    h->have_setup = false;
  });
}

int tmg_gpu_setup(tmg_gpu_handle* h, double omega) {
  return guarded(h, [&] {
    CK(cudaEventRecord(h->ev[2], h->stream));
    setup(h, omega);
    CK(cudaEventRecord(h->ev[3], h->stream));
    CK(cudaEventSynchronize(h->ev[3]));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev[2], h->ev[3]));
    h->last_setup_ms = ms;
  });
}

int tmg_gpu_set_moduli(tmg_gpu_handle* h, const double* moduli, long n_elem, double omega) {
  const int s = tmg_gpu_upload_moduli(h, moduli, n_elem);
  if (s != TMG_OK) return s;
  return tmg_gpu_setup(h, omega);
}

int tmg_gpu_set_density(tmg_gpu_handle* h, const double* alpha, int nphases,
                        const double* phase_moduli, double penalty, double omega) {
  const int s = guarded(h, [&] {
    const Grid& g = h->fine().g;
    const long ne = static_cast<long>(g.nx) * g.ny;
    double* da = grow(h->aux, h->aux_cap, ne * nphases);
    double* dp = grow(h->aux2, h->aux2_cap, nphases);
    CK(cudaMemcpyAsync(da, alpha, sizeof(double) * ne * nphases, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(dp, phase_moduli, sizeof(double) * nphases, cudaMemcpyHostToDevice, h->stream));
    k_simp<<<dim3((g.ny + 127) / 128, g.nx), 128, 0, h->stream>>>(g, nphases, da, dp, penalty, h->E);
    CKL();
    h->count();
    h->have_moduli = true;
    h->have_setup = false;
  });
  if (s != TMG_OK) return s;
  return tmg_gpu_setup(h, omega);
}

int tmg_gpu_upload_rhs(tmg_gpu_handle* h, const double* b) {
  return guarded(h, [&] { upload_nodes(h, h->b, b, h->fine().g); });
}

int tmg_gpu_upload_x0(tmg_gpu_handle* h, const double* x0) {
  return guarded(h, [&] { upload_nodes(h, h->x0, x0, h->fine().g); });
}

int tmg_gpu_solution_to_x0(tmg_gpu_handle* h) {
  return guarded(h, [&] {
    CK(cudaMemcpyAsync(h->x0, h->x, sizeof(double2) * flat2(h->fine()), cudaMemcpyDeviceToDevice, h->stream));
  });
}

int tmg_gpu_solve_resident(tmg_gpu_handle* h, int use_x0, double tol, int max_iter, int gamma,
                           int pre_sweeps, int post_sweeps, int* iterations, double* final_residual,
                           int* converged, double* seconds, double* history, int history_cap,
                           int* history_len) {
  return guarded(h, [&] {
    SolveOut o;
    solve_resident(h, use_x0 != 0, tol, max_iter, gamma, pre_sweeps, post_sweeps, o);
    if (iterations) *iterations = o.iterations;
    if (final_residual) *final_residual = o.final_residual;
    if (converged) *converged = o.converged;
    if (seconds) *seconds = o.seconds;
    copy_out_hist(o, history, history_cap, history_len);
  });
}

int tmg_gpu_download_solution(tmg_gpu_handle* h, double* x_out) {
  return guarded(h, [&] { download_nodes(h, x_out, h->x, h->fine().g); });
}

int tmg_gpu_solve(tmg_gpu_handle* h, const double* b, const double* x0, double tol, int max_iter,
                  int gamma, int pre_sweeps, int post_sweeps, double* x_out, int* iterations,
                  double* final_residual, int* converged, double* seconds, double* history,
                  int history_cap, int* history_len) {
  return guarded(h, [&] {
    need_setup(h);
    upload_nodes(h, h->b, b, h->fine().g);
    if (x0) upload_nodes(h, h->x0, x0, h->fine().g);
    SolveOut o;
    solve_resident(h, x0 != nullptr, tol, max_iter, gamma, pre_sweeps, post_sweeps, o);
    download_nodes(h, x_out, h->x, h->fine().g);
    if (iterations) *iterations = o.iterations;
    if (final_residual) *final_residual = o.final_residual;
    if (converged) *converged = o.converged;
    if (seconds) *seconds = o.seconds;
    copy_out_hist(o, history, history_cap, history_len);
  });
}

int tmg_gpu_compliance(tmg_gpu_handle* h, const double* u, double* out) {
  return guarded(h, [&] {
    if (!h->have_moduli || !h->have_problem) fail(TMG_ERR_DIMENSION, "operator not set");
    Level& F = h->fine();
    const double2* src = h->x;
    if (u) {
      upload_nodes(h, F.res, u, F.g);
      src = F.res;
    } else if (!h->have_solution) {
      fail(TMG_ERR_DIMENSION, "no resident solution");
    }
    apply_dot_fine(h, src, F.u[1], kRedPlain, h->scal);
    CK(cudaMemcpyAsync(h->scal_host, h->scal, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    *out = *h->scal_host;
  });
}

int tmg_gpu_element_energies(tmg_gpu_handle* h, const double* u, double* out) {
  return guarded(h, [&] {
    if (!h->have_problem) fail(TMG_ERR_DIMENSION, "problem not set");
    Level& F = h->fine();
    const Grid& g = F.g;
    const long ne = static_cast<long>(g.nx) * g.ny;
    const double2* src = h->x;
    if (u) {
      upload_nodes(h, F.res, u, g);
      src = F.res;
    } else if (!h->have_solution) {
      fail(TMG_ERR_DIMENSION, "no resident solution");
    }
    double* d = grow(h->dense, h->dense_cap, ne);
    k_element_energy<<<dim3((g.ny + 127) / 128, g.nx), 128, 0, h->stream>>>(g, src, d);
    CKL();
    h->count();
    CK(cudaMemcpyAsync(out, d, sizeof(double) * ne, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  });
}

int tmg_gpu_sensitivities(tmg_gpu_handle* h, const double* u, int nphases, const double* alpha,
                          const double* phase_moduli, double penalty, double* out) {
  return guarded(h, [&] {
    if (!h->have_problem) fail(TMG_ERR_DIMENSION, "problem not set");
    Level& F = h->fine();
    const Grid& g = F.g;
    const long ne = static_cast<long>(g.nx) * g.ny;
    const double2* src = h->x;
    if (u) {
      upload_nodes(h, F.res, u, g);
      src = F.res;
    } else if (!h->have_solution) {
      fail(TMG_ERR_DIMENSION, "no resident solution");
    }
    double* en = grow(h->dense, h->dense_cap, ne * (nphases + 1));
    double* da = grow(h->aux, h->aux_cap, ne * nphases);
    double* dp = grow(h->aux2, h->aux2_cap, nphases);
    CK(cudaMemcpyAsync(da, alpha, sizeof(double) * ne * nphases, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(dp, phase_moduli, sizeof(double) * nphases, cudaMemcpyHostToDevice, h->stream));
    k_element_energy<<<dim3((g.ny + 127) / 128, g.nx), 128, 0, h->stream>>>(g, src, en);
    CKL();
    double* so = en + ne;
    k_sensitivity<<<1184, 256, 0, h->stream>>>(ne, nphases, da, en, dp, penalty, so);
    CKL();
    h->count(2);
    CK(cudaMemcpyAsync(out, so, sizeof(double) * ne * nphases, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  });
}

int tmg_gpu_filter(tmg_gpu_handle* h, int nphases, const double* alpha, int phase, double radius,
                   const double* raw, double* out) {
  return guarded(h, [&] {
    const Grid& g = h->fine().g;
    const long ne = static_cast<long>(g.nx) * g.ny;
    if (phase < 0 || phase >= nphases) fail(TMG_ERR_DIMENSION, "filter: phase out of range");
    if (radius <= 1.0) {  // only the self weight survives (mto.cpp:95)
      std::memcpy(out, raw, sizeof(double) * ne);
      return;
    }
    const int reach = static_cast<int>(std::ceil(radius)) - 1;
    double* da = grow(h->aux, h->aux_cap, ne * nphases);
    double* d = grow(h->dense, h->dense_cap, 2 * ne);
    CK(cudaMemcpyAsync(da, alpha, sizeof(double) * ne * nphases, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(d, raw, sizeof(double) * ne, cudaMemcpyHostToDevice, h->stream));
    k_filter<<<dim3((g.ny + 127) / 128, g.nx), 128, 0, h->stream>>>(g.nx, g.ny, nphases, phase, radius,
                                                                     reach, da, d, d + ne);
    CKL();
    h->count();
    CK(cudaMemcpyAsync(out, d + ne, sizeof(double) * ne, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  });
}

int tmg_gpu_apply(tmg_gpu_handle* h, int level, const double* x, double* y) {
  return guarded(h, [&] {
    check_level(h, level);
    if (level < h->nc) need_setup(h);
    if (!h->have_moduli || !h->have_problem) fail(TMG_ERR_DIMENSION, "operator not set");
    Level& L = h->lev[level];
    upload_nodes(h, L.u[0], x, L.g);
    apply_level(h, level, L.u[0], L.res);
    download_nodes(h, y, L.res, L.g);
  });
}

}  // extern "C"

namespace {
template <class Op>
__global__ void k_level_values(Op op, Grid g, long n, const int* __restrict__ off,
                               const int* __restrict__ cols, double* __restrict__ vals) {
  const long r = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (r >= n) return;
  const long node = r >> 1;
  const int c = static_cast<int>(r & 1);
  const int x = static_cast<int>(node / (g.ny + 1)), y = static_cast<int>(node % (g.ny + 1));
  const long i = g.idx(x, y);
  for (int k = off[r]; k < off[r + 1]; ++k) {
    const long cn = cols[k] >> 1;
    const int d = cols[k] & 1;
    const int ex = static_cast<int>(cn / (g.ny + 1)) - x, ey = static_cast<int>(cn % (g.ny + 1)) - y;
    double v = 0.0;
    if (ex >= -1 && ex <= 1 && ey >= -1 && ey <= 1) {
      double b[4];
      op.block(i, ex, ey, b);
      v = b[2 * c + d];
    }
    vals[k] = v;
  }
}
}  // namespace

extern "C" {

int tmg_gpu_level_values(tmg_gpu_handle* h, int level, const int* offsets, const int* cols,
                         double* vals) {
  return guarded(h, [&] {
    check_level(h, level);
    if (level < h->nc) need_setup(h);
    const Level& L = h->lev[level];
    const long n = L.ndof;
    const long nnz = offsets[n];
    int* doff = reinterpret_cast<int*>(grow(h->aux, h->aux_cap, (n + 1 + nnz + 1) / 2 + 1));
    int* dcol = doff + n + 1;
    double* dv = grow(h->dense, h->dense_cap, nnz);
    CK(cudaMemcpyAsync(doff, offsets, sizeof(int) * (n + 1), cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(dcol, cols, sizeof(int) * nnz, cudaMemcpyHostToDevice, h->stream));
    with_op(h, level, [&](auto op) {
      k_level_values<decltype(op)><<<(n + 127) / 128, 128, 0, h->stream>>>(op, L.g, n, doff, dcol, dv);
    });
    CKL();
    h->count();
    CK(cudaMemcpyAsync(vals, dv, sizeof(double) * nnz, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  });
}

int tmg_gpu_vcycle(tmg_gpu_handle* h, const double* f, double* u, int gamma, int pre_sweeps,
                   int post_sweeps) {
  return guarded(h, [&] {
    need_setup(h);
    Level& F = h->fine();
    upload_nodes(h, h->r, f, F.g);
    for (Level& L : h->lev) L.cur = 0;
    upload_nodes(h, F.u[0], u, F.g);
    enqueue_cycle(h, h->nc, false, gamma, pre_sweeps, post_sweeps);
    download_nodes(h, u, F.u[F.cur], F.g);
  });
}

int tmg_gpu_prolongate(tmg_gpu_handle* h, int level, const double* coarse, double* fine) {
  return guarded(h, [&] {
    check_level(h, level);
    if (level < 1) fail(TMG_ERR_DIMENSION, "prolongate: level " + std::to_string(level) + " has no coarser neighbor");
    Level& F = h->lev[level];
    Level& C = h->lev[level - 1];
    upload_nodes(h, C.u[0], coarse, C.g);
    prolong_level(h, level, C.u[0], F.res, false);
    download_nodes(h, fine, F.res, F.g);
  });
}

int tmg_gpu_restrict(tmg_gpu_handle* h, int level, const double* fine, double* coarse) {
  return guarded(h, [&] {
    check_level(h, level);
    if (level < 1) fail(TMG_ERR_DIMENSION, "restrict: level " + std::to_string(level) + " has no coarser neighbor");
    Level& F = h->lev[level];
    Level& C = h->lev[level - 1];
    upload_nodes(h, F.res, fine, F.g);
    restrict_level(h, level, F.res, C.res);
    download_nodes(h, coarse, C.res, C.g);
  });
}

int tmg_gpu_smooth(tmg_gpu_handle* h, int level, const double* f, double* u, int sweeps) {
  return guarded(h, [&] {
    check_level(h, level);
    if (level < h->nc) need_setup(h);
    if (!h->have_moduli || !h->have_problem) fail(TMG_ERR_DIMENSION, "operator not set");
    Level& L = h->lev[level];
    upload_nodes(h, L.f, f, L.g);
    upload_nodes(h, L.u[0], u, L.g);
    L.cur = 0;
    for (int s = 0; s < sweeps; ++s) {
      sweep_level(h, level, false, L.u[L.cur], L.u[L.cur ^ 1], L.f);
      L.cur ^= 1;
    }
    download_nodes(h, u, L.u[L.cur], L.g);
  });
}

void* tmg_gpu_stream(tmg_gpu_handle* h) { return h ? static_cast<void*>(h->stream) : nullptr; }

long tmg_gpu_launch_count(tmg_gpu_handle* h) { return h ? h->launches : 0; }

int tmg_gpu_time_kernel(tmg_gpu_handle* h, int which, int reps, double* avg_ms, double* bytes) {
  return guarded(h, [&] {
    if (!h->have_moduli || !h->have_problem) fail(TMG_ERR_DIMENSION, "operator not set");
    Level& F = h->fine();
    const double nodes = static_cast<double>(F.g.nx + 1) * (F.g.ny + 1);
    auto launch = [&] {
      if (which == 0) apply_level(h, h->nc, h->pbuf[0], h->ap);
      else sweep_level(h, h->nc, false, F.u[0], F.u[1], h->r);
    };
    for (int w = 0; w < 3; ++w) launch();
    CK(cudaEventRecord(h->ev[2], h->stream));
    for (int k = 0; k < reps; ++k) launch();
    CK(cudaEventRecord(h->ev[3], h->stream));
    CK(cudaEventSynchronize(h->ev[3]));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev[2], h->ev[3]));
    *avg_ms = ms / reps;
    // algorithmic bytes per node: apply reads u 16 + E 8 + mask 1, writes 16;
    // the sweep additionally reads f 16
    *bytes = nodes * (which == 0 ? 41.0 : 57.0);
  });
}

int tmg_gpu_last_timings(tmg_gpu_handle* h, double* setup_ms, double* pcg_ms) {
  if (!h) return TMG_ERR_DIMENSION;
  if (setup_ms) *setup_ms = h->last_setup_ms;
  if (pcg_ms) *pcg_ms = h->last_pcg_ms;
  return TMG_OK;
}

int tmg_gpu_event_record(tmg_gpu_handle* h, int slot) {
  return guarded(h, [&] {
    if (slot < 0 || slot >= 8) fail(TMG_ERR_DIMENSION, "event slot out of range");
    if (!h->uev[slot]) CK(cudaEventCreate(&h->uev[slot]));
    CK(cudaEventRecord(h->uev[slot], h->stream));
  });
}

int tmg_gpu_event_elapsed(tmg_gpu_handle* h, int a, int b, double* ms) {
  return guarded(h, [&] {
    if (a < 0 || a >= 8 || b < 0 || b >= 8 || !h->uev[a] || !h->uev[b])
      fail(TMG_ERR_DIMENSION, "event slot not recorded");
    CK(cudaEventSynchronize(h->uev[b]));
    float f = 0.f;
    CK(cudaEventElapsedTime(&f, h->uev[a], h->uev[b]));
    *ms = f;
  });
}

void* tmg_host_alloc(unsigned long bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) return nullptr;
  return p;
}

void tmg_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

}  // extern "C"
