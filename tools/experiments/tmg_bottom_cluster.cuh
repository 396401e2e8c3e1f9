// ARCHIVED EXPERIMENT (not built into the library): the V-cycle bottom as one
// thread-block-cluster kernel with global-memory stages. It was bitwise equal
// to the per-level launches and SLOWER on every config (DESIGN.md section 4,
// "Tried and not kept"); kept with tools/micro/cluster_bar.cu as the record of
// the measured stage costs. To rebuild it, copy it back into csrc/ and hook it
// into enqueue_cycle as described in DESIGN.md.
// The bottom of the V-cycle as ONE thread-block-cluster kernel.
//
// Below a few tens of thousands of nodes a coarse level is pure latency: the
// shared-memory tile kernels (tmg_stile.cuh) spend ~5-7 us per V(2,2) half
// whatever the level size (launch, one load round, three barrier-separated
// stages), and the coarsest solve another ~4-6 us, so on the optimizer meshes
// (64^2-1024^2) the levels of <= 129^2 nodes cost 25-55 us of a 70-250 us PCG
// iteration. Here one cluster of CTAs (one per SM, all on one GPC) walks every
// one of those levels, DOWN to the coarsest solve and back UP, in a single
// launch. Its stages exchange data through global memory (L2: the bottom
// levels together are a few MB) and are separated by hardware cluster
// barriers (barrier.cluster arrive.release / wait.acquire, a few hundred
// cycles) instead of kernel boundaries. Within a stage every CTA takes a
// strided share of the level's nodes.
//
// Per level l (mg_cycle, solvers.cpp:483-514, gamma = 1, 2 pre- and 2
// post-sweeps from a zero iterate) the stages are those of the tile kernels,
// with the same per-node arithmetic in the same order (s_apply, s_jacobi_r,
// the restriction sums, the prolongation means), so every result is bitwise
// that of the per-level launches (TMG_BOTTOM_MAX_NODES=0):
//
//   DOWN  x1 = omega f / D                      -> u[cur]   (the top level's
//                                                in stage 0, the others in the
//                                                restriction stage above them)
//         x2 = x1 + omega D^-1 (f - A x1)       -> u[cur^1]
//         r  = f - A x2                          -> res
//         f_c = (1/4) P^T r  (+ x1 of level l-1)
//   coarsest: u_0 = A_0^-1 f_0 (the explicit inverse, k_coarse_solve's sums)
//   UP    w  = x2 + P u_c (on the fly over the 3x3 window)
//         x3 = w + omega D^-1 (f - A w)          -> res
//         x4 = x3 + omega D^-1 (f - A x3)        -> u[cur]
//
// Buffers written by one CTA are read by others only after a cluster barrier,
// with plain loads (the barrier's acquire invalidates L1); the stencil planes
// and the coarsest inverse are invariant during the kernel and go through the
// read-only path.
#pragma once

#include <cuda_runtime.h>

#include "tmg_device.cuh"
#include "tmg_smarch.cuh"

namespace tmg {

constexpr int kBotMaxLevels = 12;
#ifndef TMG_BOT_THREADS
#define TMG_BOT_THREADS 256
#endif
constexpr int kBotThreads = TMG_BOT_THREADS;
// default size limit of the top level of the cluster bottom (nodes);
// TMG_BOTTOM_MAX_NODES overrides it (0 disables the kernel)
constexpr long kBotMaxNodes = 129L * 129L;

struct BotLevel {
  Grid g;
  const double* S;  // stencil planes, plane stride g.size
  double2* f;       // rhs (the restriction of the level above writes it, except on the top level)
  double2* u;       // x1, then x4 (the visit's result): u[cur]
  double2* x2;      // u[cur ^ 1]
  double2* r;       // residual, then x3: res
};

struct BotArgs {
  int nl;                       // stencil levels 1..nl (lev[nl] is the top)
  BotLevel lev[kBotMaxLevels];  // index 1..nl
  Grid g0;                      // coarsest level
  double2* f0;
  double2* u0;
  const double* Ainv;
  int n0;
  double omega;
};

__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_ctas() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}

// stencil planes of one node column (row index j), read-only path
struct GPlanes {
  const double* col;
  long plane;
  __device__ __forceinline__ double at(int k, int j) const { return __ldg(col + k * plane + j); }
};

__device__ __forceinline__ bool bot_in(const Grid& g, int x, int y) {
  return x >= 0 && x <= g.nx && y >= 0 && y <= g.ny;
}
// a vector value, zero outside the level (the tile kernels' region load)
__device__ __forceinline__ double2 bot_ld(const Grid& g, const double2* v, int x, int y) {
  return bot_in(g, x, y) ? v[g.idx(x, y)] : make_double2(0.0, 0.0);
}

// A v and its diagonal at (x, y) from a 3x3 window of v
__device__ __forceinline__ void bot_apply(const BotLevel& L, int x, int y, const double2 (&l)[3],
                                          const double2 (&c)[3], const double2 (&r)[3], double2& yv, double2& d) {
  const Grid& g = L.g;
  s_apply(GPlanes{L.S + g.idx(x, 0), g.size}, GPlanes{L.S + g.idx(x - 1, 0), g.size}, y, l, c, r, yv, d);
}

__device__ __forceinline__ void bot_window(const Grid& g, const double2* v, int x, int y, double2 (&l)[3],
                                           double2 (&c)[3], double2 (&r)[3]) {
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    l[q] = bot_ld(g, v, x - 1, y - 1 + q);
    c[q] = bot_ld(g, v, x, y - 1 + q);
    r[q] = bot_ld(g, v, x + 1, y - 1 + q);
  }
}

// x1 = omega f / D (the tile kernels' DOWN stage-A input)
__device__ __forceinline__ double2 bot_x1(const BotLevel& L, double2 f, int x, int y, double omega) {
  const long i = L.g.idx(x, y);
  const double2 rc = make_double2(rcp_nr(__ldg(L.S + i)), rcp_nr(__ldg(L.S + 2 * L.g.size + i)));
  return make_double2(omega * f.x * rc.x, omega * f.y * rc.y);
}

// w = x2 + P u_c at a level node (the tile kernels' UP stage-A input): coarse
// column ceil(x/2), for odd x the mean with floor(x/2); odd rows interpolate
// the two coarse rows around them
__device__ __forceinline__ double2 bot_w(const Grid& g, const Grid& gc, const double2* x2, const double2* uc, int x,
                                         int y) {
  // every load is issued unconditionally (selects instead of branches), so
  // the compiler can batch the window's loads into one round trip
  const int Y = y >> 1;
  const int Xa = (x + 1) >> 1, Xb = x >> 1;
  const double2 pa = bot_ld(gc, uc, Xa, Y), qa = bot_ld(gc, uc, Xa, Y + 1);
  const double2 pb = bot_ld(gc, uc, Xb, Y), qb = bot_ld(gc, uc, Xb, Y + 1);
  const double2 xv = bot_ld(g, x2, x, y);
  const bool oy = y & 1;
  const double2 ca = oy ? make_double2(0.5 * pa.x + 0.5 * qa.x, 0.5 * pa.y + 0.5 * qa.y) : pa;
  const double2 cb = oy ? make_double2(0.5 * pb.x + 0.5 * qb.x, 0.5 * pb.y + 0.5 * qb.y) : pb;
  const double2 pu = ((g.x0 + x) & 1) ? make_double2(0.5 * cb.x + 0.5 * ca.x, 0.5 * cb.y + 0.5 * ca.y) : ca;
  return bot_in(g, x, y) ? make_double2(xv.x + pu.x, xv.y + pu.y) : make_double2(0.0, 0.0);
}

#ifdef TMG_BOT_TRACE
// per-stage %globaltimer stamps of CTA 0, thread 0 (trace builds only)
__device__ unsigned long long g_bot_trace[64];
__device__ __forceinline__ void bot_stamp(int& k) {
  if (threadIdx.x == 0 && cluster_rank() == 0 && k < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_bot_trace[k] = t;
  }
  ++k;
}
#define BOT_STAMP() bot_stamp(stamp)
#else
#define BOT_STAMP()
#endif

__global__ void __launch_bounds__(kBotThreads, 1) k_bottom(const __grid_constant__ BotArgs a) {
  extern __shared__ double bot_fd[];  // the coarsest rhs, dof-major
  const int rank = static_cast<int>(cluster_rank());
  const int stride = static_cast<int>(cluster_ctas()) * kBotThreads;
  const int first = rank * kBotThreads + threadIdx.x;
  const double omega = a.omega;
  // nodes of a level, column-major (x = n / rows, y = n % rows)
  auto nodes = [](const Grid& g) { return (g.nx + 1) * (g.ny + 1); };
#ifdef TMG_BOT_TRACE
  int stamp = 0;
#endif
  BOT_STAMP();

  // ---- stage 0: x1 of the top level
  {
    const BotLevel& L = a.lev[a.nl];
    const int rows = L.g.ny + 1, N = nodes(L.g);
    for (int n = first; n < N; n += stride) {
      const int x = n / rows, y = n % rows;
      const long i = L.g.idx(x, y);
      L.u[i] = bot_x1(L, L.f[i], x, y, omega);
    }
  }
  cluster_barrier();
  BOT_STAMP();
  // ---- DOWN
  for (int l = a.nl; l >= 1; --l) {
    const BotLevel& L = a.lev[l];
    const Grid& g = L.g;
    const int rows = g.ny + 1, N = nodes(g);
    // x2 = x1 + omega D^-1 (f - A x1)
    for (int n = first; n < N; n += stride) {
      const int x = n / rows, y = n % rows;
      double2 wl[3], wc[3], wr[3], yv, d;
      bot_window(g, L.u, x, y, wl, wc, wr);
      bot_apply(L, x, y, wl, wc, wr, yv, d);
      const long i = g.idx(x, y);
      L.x2[i] = s_jacobi_r(wc[1], L.f[i], yv, make_double2(rcp_nr(d.x), rcp_nr(d.y)), omega);
    }
    cluster_barrier();
    BOT_STAMP();
    // r = f - A x2
    for (int n = first; n < N; n += stride) {
      const int x = n / rows, y = n % rows;
      double2 wl[3], wc[3], wr[3], yv, d;
      bot_window(g, L.x2, x, y, wl, wc, wr);
      bot_apply(L, x, y, wl, wc, wr, yv, d);
      const long i = g.idx(x, y);
      const double2 f = L.f[i];
      L.r[i] = make_double2(f.x - yv.x, f.y - yv.y);
    }
    cluster_barrier();
    BOT_STAMP();
    // f_c = (1/4) P^T r in the tile kernels' order: rows (1/2, 1, 1/2)
    // around the even level row, then columns 2X-1, 2X, 2X+1; then x1 of
    // the coarse level from f_c
    const Grid& gc = (l > 1) ? a.lev[l - 1].g : a.g0;
    double2* fc = (l > 1) ? a.lev[l - 1].f : a.f0;
    const int crows = gc.ny + 1, NC = nodes(gc);
    for (int n = first; n < NC; n += stride) {
      const int X = n / crows, Y = n % crows;
      auto rs = [&](int x) {
        const double2 rm = bot_ld(g, L.r, x, 2 * Y - 1), r0 = bot_ld(g, L.r, x, 2 * Y),
                      rp = bot_ld(g, L.r, x, 2 * Y + 1);
        return make_double2(fma(0.5, rm.x + rp.x, r0.x), fma(0.5, rm.y + rp.y, r0.y));
      };
      const double2 s0 = rs(2 * X - 1), s1 = rs(2 * X), s2 = rs(2 * X + 1);
      double2 acc = make_double2(0.5 * s0.x, 0.5 * s0.y);
      acc.x += s1.x;
      acc.y += s1.y;
      acc.x = fma(0.5, s2.x, acc.x);
      acc.y = fma(0.5, s2.y, acc.y);
      const double2 v = make_double2(0.25 * acc.x, 0.25 * acc.y);
      const long i = gc.idx(X, Y);
      fc[i] = v;
      if (l > 1) a.lev[l - 1].u[i] = bot_x1(a.lev[l - 1], v, X, Y, omega);
    }
    cluster_barrier();
    BOT_STAMP();
  }
  // ---- coarsest: u_0 = A_0^-1 f_0 (k_coarse_solve: one warp per node,
  // lane-strided partial sums, then a butterfly)
  {
    const Grid& g = a.g0;
    const int rows = g.ny + 1, nn = a.n0 / 2;
    for (int k = threadIdx.x; k < nn; k += kBotThreads) {
      const double2 v = a.f0[g.idx(k / rows, k % rows)];
      bot_fd[2 * k] = v.x;
      bot_fd[2 * k + 1] = v.y;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int warps = stride / 32;
    for (int node = first >> 5; node < nn; node += warps) {
      double s0 = 0.0, s1 = 0.0;
      for (int k = lane; k < a.n0; k += 32) {
        const double fk = bot_fd[k];
        s0 = fma(__ldg(a.Ainv + static_cast<long>(k) * a.n0 + 2 * node), fk, s0);
        s1 = fma(__ldg(a.Ainv + static_cast<long>(k) * a.n0 + 2 * node + 1), fk, s1);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      }
      if (lane == 0) a.u0[g.idx(node / rows, node % rows)] = make_double2(s0, s1);
    }
  }
  cluster_barrier();
  BOT_STAMP();
  // ---- UP
  for (int l = 1; l <= a.nl; ++l) {
    const BotLevel& L = a.lev[l];
    const Grid& g = L.g;
    const Grid& gc = (l > 1) ? a.lev[l - 1].g : a.g0;
    const double2* uc = (l > 1) ? a.lev[l - 1].u : a.u0;
    const int rows = g.ny + 1, N = nodes(g);
    // x3 = w + omega D^-1 (f - A w), w = x2 + P u_c
    for (int n = first; n < N; n += stride) {
      const int x = n / rows, y = n % rows;
      double2 wl[3], wc[3], wr[3], yv, d;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        wl[q] = bot_w(g, gc, L.x2, uc, x - 1, y - 1 + q);
        wc[q] = bot_w(g, gc, L.x2, uc, x, y - 1 + q);
        wr[q] = bot_w(g, gc, L.x2, uc, x + 1, y - 1 + q);
      }
      bot_apply(L, x, y, wl, wc, wr, yv, d);
      const long i = g.idx(x, y);
      L.r[i] = s_jacobi_r(wc[1], L.f[i], yv, make_double2(rcp_nr(d.x), rcp_nr(d.y)), omega);
    }
    cluster_barrier();
    BOT_STAMP();
    // x4 = x3 + omega D^-1 (f - A x3)
    for (int n = first; n < N; n += stride) {
      const int x = n / rows, y = n % rows;
      double2 wl[3], wc[3], wr[3], yv, d;
      bot_window(g, L.r, x, y, wl, wc, wr);
      bot_apply(L, x, y, wl, wc, wr, yv, d);
      const long i = g.idx(x, y);
      L.u[i] = s_jacobi_r(wc[1], L.f[i], yv, make_double2(rcp_nr(d.x), rcp_nr(d.y)), omega);
    }
    if (l < a.nl) cluster_barrier();
    BOT_STAMP();
  }
}

}  // namespace tmg
