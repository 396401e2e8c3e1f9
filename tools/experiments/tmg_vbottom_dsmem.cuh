// ARCHIVED EXPERIMENT (not built into the library): the V-cycle bottom as
// one cluster kernel with DSMEM-resident data. Bitwise equal to the per-level
// launches and slower ("Tried and not kept"); the
// TMG_VB_TRACE stamps gave ~2 us per stage.
// The bottom of the V-cycle (every level of at most kVbMaxNodes nodes and the
// coarsest solve) as ONE thread-block-cluster kernel with the data resident
// in distributed shared memory.
//
// Below ~65^2 nodes a V(2,2) half costs the tile kernels (tmg_stile.cuh) a
// launch, a load round from L2 and three or four barrier-separated stages,
// ~4-6 us whatever the level size, so c0/c1/c3 spend 20-30 us of a
// 60-230 us PCG iteration in the levels of <= 65^2 nodes and the coarsest
// solve. Here one cluster of kVbCTAs CTAs loads those levels' stencil planes
// once, keeps every vector in shared memory, and walks DOWN to the coarsest
// solve and back UP with hardware cluster barriers between the stages
// (measured on the B200: a DSMEM store + cluster barrier + load round is
// ~0.35 us against 1.23 us for a dependent kernel boundary in a graph and
// ~0.7 us for a global-memory stage, tools/micro/cluster_bar.cu).
//
// Layout: CTA r of the cluster owns the node columns [r w, (r+1) w) of every
// bottom level (w = ceil(ncol / CTAs)); a column is stored with one zero row
// below and above (rows + 2 entries). A neighbour's value or stencil plane in
// another CTA's columns is read through the cluster's shared-memory window.
//
// Per level the stages are the tile kernels' with the same per-node
// arithmetic in the same order (s_apply, s_jacobi_r, the restriction sums,
// the prolongation means; the coarsest solve is k_coarse_solve's), so every
// result is bitwise that of the per-level launches (TMG_VBOTTOM=0):
//   DOWN  x1 = omega f / D (folded into the restriction above; stage 0 for
//         the top level), x2 = x1 + omega D^-1 (f - A x1), r = f - A x2,
//         f_c = (1/4) P^T r and the coarse level's x1
//   coarsest  u_0 = A_0^-1 f_0 (the explicit inverse)
//   UP    w = x2 + P u_c, x3 = w + omega D^-1 (f - A w),
//         x4 = x3 + omega D^-1 (f - A x3)
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "tmg_device.cuh"
#include "tmg_smarch.cuh"

namespace tmg {

constexpr int kVbThreads = 512;
constexpr int kVbMaxLevels = 6;  // stencil levels in the bottom
// default size limit of the bottom's top level (nodes); TMG_VBOTTOM_MAX_NODES
// overrides it, TMG_VBOTTOM=0 turns the kernel off
constexpr long kVbMaxNodes = 65L * 65L;

struct VbLevel {
  Grid g;           // device (global) grid of the level
  const double* S;  // global stencil planes (plane stride g.size)
  // shared-memory offsets (bytes) of this level's arrays, identical in every CTA
  int w;       // owned columns per CTA
  int rows2;   // rows + 2 (a zero row below and above)
  int o_pl;    // planes [19][w][rows2]
  int o_f;     // f [w][rows2] (double2)
  int o_a;     // x1, then x3
  int o_b;     // x2
  int o_c;     // r, then w, then x4 (the visit's result)
};

struct VbArgs {
  int nl;  // stencil levels 1..nl
  VbLevel lev[kVbMaxLevels + 1];
  Grid g0;  // coarsest level
  int w0, rows20, o_f0, o_u0, o_fd, o_zero;
  const double* Ainv;
  int n0;
  double omega;
  const double2* f_top;  // global f of the top level
  double2* out_top;      // global u[cur] of the top level (x4)
  int zero_len;          // doubles in the zero column
  int smem;              // dynamic shared memory per CTA (bytes)
};

// stencil planes of one column (row j; rows -1 .. rows are stored)
struct VbPlanes {
  const double* b;
  int ps;
  __device__ __forceinline__ double at(int k, int j) const { return b[k * ps + j]; }
};

#ifdef TMG_VB_TRACE
__device__ unsigned long long g_vb_trace[64];
#define VB_STAMP()                                                              \
  do {                                                                          \
    if (t == 0 && rank == 0 && vb_k < 64) {                                     \
      unsigned long long tt;                                                    \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));                     \
      g_vb_trace[vb_k] = tt;                                                    \
    }                                                                           \
    ++vb_k;                                                                     \
  } while (0)
#else
#define VB_STAMP()
#endif
__global__ void __launch_bounds__(kVbThreads, 1) k_vbottom(const __grid_constant__ VbArgs a) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) unsigned char vsm[];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = static_cast<int>(cl.block_rank());
  const int t = threadIdx.x;
  const double omega = a.omega;
  const double2 z2 = make_double2(0.0, 0.0);
#ifdef TMG_VB_TRACE
  int vb_k = 0;
#endif
  VB_STAMP();

  auto ptr = [&](int off, int owner) -> unsigned char* {
    return owner == rank ? vsm + off : static_cast<unsigned char*>(cl.map_shared_rank(static_cast<void*>(vsm + off), owner));
  };
  auto in_level = [](const Grid& g, int x, int y) { return x >= 0 && x <= g.nx && y >= 0 && y <= g.ny; };
  // a node value of a level buffer (zero outside the level)
  auto val = [&](const Grid& g, int w, int rows2, int off, int x, int y) -> double2 {
    if (!in_level(g, x, y)) return z2;
    const int o = x / w;
    return reinterpret_cast<const double2*>(ptr(off, o))[(x - o * w) * rows2 + y + 1];
  };
  auto planes = [&](const VbLevel& L, int x) -> VbPlanes {
    if (x < 0) return VbPlanes{reinterpret_cast<const double*>(vsm + a.o_zero) + 1, 0};
    const int o = x / L.w;
    return VbPlanes{reinterpret_cast<const double*>(ptr(L.o_pl, o)) + (x - o * L.w) * L.rows2 + 1, L.w * L.rows2};
  };
  // A v at (x, y) of level L over buffer `off`, with its diagonal
  auto apply = [&](const VbLevel& L, int off, int x, int y, double2& yv, double2& d) {
    double2 l3[3], c3[3], r3[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      l3[q] = val(L.g, L.w, L.rows2, off, x - 1, y - 1 + q);
      c3[q] = val(L.g, L.w, L.rows2, off, x, y - 1 + q);
      r3[q] = val(L.g, L.w, L.rows2, off, x + 1, y - 1 + q);
    }
    s_apply(planes(L, x), planes(L, x - 1), y, l3, c3, r3, yv, d);
  };
  auto loc2 = [&](int off, int lc, int rows2, int y) -> double2& {
    return reinterpret_cast<double2*>(vsm + off)[lc * rows2 + y + 1];
  };

  // ---- zero everything, then load the stencil planes and the top level's f
  for (int i = t; i < a.smem / 16; i += kVbThreads) reinterpret_cast<double2*>(vsm)[i] = z2;
  __syncthreads();
  for (int l = 1; l <= a.nl; ++l) {
    const VbLevel& L = a.lev[l];
    const int x0 = rank * L.w, nown = max(0, min(L.w, L.g.nx + 1 - x0)), rows = L.g.ny + 1;
    double* pl = reinterpret_cast<double*>(vsm + L.o_pl);
    const int ps = L.w * L.rows2;
    for (int i = t; i < nown * rows * kStencilPlanes; i += kVbThreads) {
      const int k = i / (nown * rows), rem = i - k * nown * rows, lc = rem / rows, y = rem - lc * rows;
      pl[k * ps + lc * L.rows2 + y + 1] = __ldg(L.S + k * L.g.size + L.g.idx(x0 + lc, y));
    }
  }
  VB_STAMP();
  grid_dep_wait();
  grid_dep_launch();
  VB_STAMP();
  {
    const VbLevel& L = a.lev[a.nl];
    const int x0 = rank * L.w, nown = max(0, min(L.w, L.g.nx + 1 - x0)), rows = L.g.ny + 1;
    for (int i = t; i < nown * rows; i += kVbThreads) {
      const int lc = i / rows, y = i - lc * rows;
      loc2(L.o_f, lc, L.rows2, y) = a.f_top[L.g.idx(x0 + lc, y)];
    }
  }
  __syncthreads();
  // ---- stage 0: x1 of the top level
  auto x1_of = [&](const VbLevel& L, int lc, int y, double2 f) {
    const double* pl = reinterpret_cast<const double*>(vsm + L.o_pl) + lc * L.rows2 + y + 1;
    const int ps = L.w * L.rows2;
    const double2 rc = make_double2(rcp_nr(pl[0]), rcp_nr(pl[2 * ps]));
    return make_double2(omega * f.x * rc.x, omega * f.y * rc.y);
  };
  {
    const VbLevel& L = a.lev[a.nl];
    const int x0 = rank * L.w, nown = max(0, min(L.w, L.g.nx + 1 - x0)), rows = L.g.ny + 1;
    for (int i = t; i < nown * rows; i += kVbThreads) {
      const int lc = i / rows, y = i - lc * rows;
      loc2(L.o_a, lc, L.rows2, y) = x1_of(L, lc, y, loc2(L.o_f, lc, L.rows2, y));
    }
  }
  cl.sync();
  VB_STAMP();
  // ---- DOWN
  for (int l = a.nl; l >= 1; --l) {
    const VbLevel& L = a.lev[l];
    const int x0 = rank * L.w, nown = max(0, min(L.w, L.g.nx + 1 - x0)), rows = L.g.ny + 1;
    for (int i = t; i < nown * rows; i += kVbThreads) {
      const int lc = i / rows, y = i - lc * rows, x = x0 + lc;
      double2 yv, d;
      apply(L, L.o_a, x, y, yv, d);
      loc2(L.o_b, lc, L.rows2, y) = s_jacobi_r(loc2(L.o_a, lc, L.rows2, y), loc2(L.o_f, lc, L.rows2, y), yv,
                                               make_double2(rcp_nr(d.x), rcp_nr(d.y)), omega);
    }
    cl.sync();
    VB_STAMP();
  VB_STAMP();
    for (int i = t; i < nown * rows; i += kVbThreads) {
      const int lc = i / rows, y = i - lc * rows, x = x0 + lc;
      double2 yv, d;
      apply(L, L.o_b, x, y, yv, d);
      const double2 f = loc2(L.o_f, lc, L.rows2, y);
      loc2(L.o_c, lc, L.rows2, y) = make_double2(f.x - yv.x, f.y - yv.y);
    }
    cl.sync();
    VB_STAMP();
  VB_STAMP();
    // restriction into the coarse level's f (and its x1)
    const bool coarsest = (l == 1);
    const Grid& gc = coarsest ? a.g0 : a.lev[l - 1].g;
    const int wc = coarsest ? a.w0 : a.lev[l - 1].w;
    const int rows2c = coarsest ? a.rows20 : a.lev[l - 1].rows2;
    const int o_fc = coarsest ? a.o_f0 : a.lev[l - 1].o_f;
    const int X0 = rank * wc, nownc = max(0, min(wc, gc.nx + 1 - X0)), rowsc = gc.ny + 1;
    for (int i = t; i < nownc * rowsc; i += kVbThreads) {
      const int lc = i / rowsc, Y = i - lc * rowsc, X = X0 + lc;
      auto rs = [&](int x) {
        const double2 rm = val(L.g, L.w, L.rows2, L.o_c, x, 2 * Y - 1), r0 = val(L.g, L.w, L.rows2, L.o_c, x, 2 * Y),
                      rp = val(L.g, L.w, L.rows2, L.o_c, x, 2 * Y + 1);
        return make_double2(fma(0.5, rm.x + rp.x, r0.x), fma(0.5, rm.y + rp.y, r0.y));
      };
      const double2 s0 = rs(2 * X - 1), s1 = rs(2 * X), s2 = rs(2 * X + 1);
      double2 acc = make_double2(0.5 * s0.x, 0.5 * s0.y);
      acc.x += s1.x;
      acc.y += s1.y;
      acc.x = fma(0.5, s2.x, acc.x);
      acc.y = fma(0.5, s2.y, acc.y);
      const double2 fcv = make_double2(0.25 * acc.x, 0.25 * acc.y);
      loc2(o_fc, lc, rows2c, Y) = fcv;
      if (!coarsest) loc2(a.lev[l - 1].o_a, lc, rows2c, Y) = x1_of(a.lev[l - 1], lc, Y, fcv);
    }
    cl.sync();
    VB_STAMP();
  VB_STAMP();
  }
  // ---- coarsest: u_0 = A_0^-1 f_0 (k_coarse_solve's sums)
  {
    const Grid& g = a.g0;
    const int rows = g.ny + 1, nn = a.n0 / 2;
    double* fd = reinterpret_cast<double*>(vsm + a.o_fd);
    for (int k = t; k < nn; k += kVbThreads) {
      const double2 v = val(g, a.w0, a.rows20, a.o_f0, k / rows, k % rows);
      fd[2 * k] = v.x;
      fd[2 * k + 1] = v.y;
    }
    __syncthreads();
    const int lane = t & 31, warp = t >> 5;
    const int X0 = rank * a.w0, nown = max(0, min(a.w0, g.nx + 1 - X0));
    for (int j = warp; j < nown * rows; j += kVbThreads / 32) {
      const int lc = j / rows, Y = j - lc * rows;
      const int node = (X0 + lc) * rows + Y;
      double s0 = 0.0, s1 = 0.0;
      for (int k = lane; k < a.n0; k += 32) {
        const double fk = fd[k];
        s0 = fma(__ldg(a.Ainv + static_cast<long>(k) * a.n0 + 2 * node), fk, s0);
        s1 = fma(__ldg(a.Ainv + static_cast<long>(k) * a.n0 + 2 * node + 1), fk, s1);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      }
      if (lane == 0) loc2(a.o_u0, lc, a.rows20, Y) = make_double2(s0, s1);
    }
  }
  cl.sync();
  VB_STAMP();
  // ---- UP
  for (int l = 1; l <= a.nl; ++l) {
    const VbLevel& L = a.lev[l];
    const int x0 = rank * L.w, nown = max(0, min(L.w, L.g.nx + 1 - x0)), rows = L.g.ny + 1;
    const bool coarsest = (l == 1);
    const Grid& gc = coarsest ? a.g0 : a.lev[l - 1].g;
    const int wc = coarsest ? a.w0 : a.lev[l - 1].w;
    const int rows2c = coarsest ? a.rows20 : a.lev[l - 1].rows2;
    const int o_uc = coarsest ? a.o_u0 : a.lev[l - 1].o_c;
    // w = x2 + P u_c (the tile kernels' UP stage-A input)
    for (int i = t; i < nown * rows; i += kVbThreads) {
      const int lc = i / rows, y = i - lc * rows, x = x0 + lc;
      auto colv = [&](int X) {
        const double2 p = val(gc, wc, rows2c, o_uc, X, y >> 1);
        if (!(y & 1)) return p;
        const double2 q = val(gc, wc, rows2c, o_uc, X, (y >> 1) + 1);
        return make_double2(0.5 * p.x + 0.5 * q.x, 0.5 * p.y + 0.5 * q.y);
      };
      double2 pu = colv((x + 1) >> 1);
      if ((L.g.x0 + x) & 1) {
        const double2 q = colv(x >> 1);
        pu = make_double2(0.5 * q.x + 0.5 * pu.x, 0.5 * q.y + 0.5 * pu.y);
      }
      const double2 xv = loc2(L.o_b, lc, L.rows2, y);
      loc2(L.o_c, lc, L.rows2, y) = make_double2(xv.x + pu.x, xv.y + pu.y);
    }
    cl.sync();
    VB_STAMP();
  VB_STAMP();
    // x3 = w + omega D^-1 (f - A w)
    for (int i = t; i < nown * rows; i += kVbThreads) {
      const int lc = i / rows, y = i - lc * rows, x = x0 + lc;
      double2 yv, d;
      apply(L, L.o_c, x, y, yv, d);
      loc2(L.o_a, lc, L.rows2, y) = s_jacobi_r(loc2(L.o_c, lc, L.rows2, y), loc2(L.o_f, lc, L.rows2, y), yv,
                                               make_double2(rcp_nr(d.x), rcp_nr(d.y)), omega);
    }
    cl.sync();
    VB_STAMP();
  VB_STAMP();
    // x4 = x3 + omega D^-1 (f - A x3): into C (w is dead) and, on the top
    // level, into global memory
    for (int i = t; i < nown * rows; i += kVbThreads) {
      const int lc = i / rows, y = i - lc * rows, x = x0 + lc;
      double2 yv, d;
      apply(L, L.o_a, x, y, yv, d);
      const double2 v = s_jacobi_r(loc2(L.o_a, lc, L.rows2, y), loc2(L.o_f, lc, L.rows2, y), yv,
                                   make_double2(rcp_nr(d.x), rcp_nr(d.y)), omega);
      loc2(L.o_c, lc, L.rows2, y) = v;
      if (l == a.nl) a.out_top[L.g.idx(x, y)] = v;
    }
    // the next level's w stage reads this C; the last level's x4 ends the
    // kernel (the cluster still syncs so no CTA exits while others read it)
    cl.sync();
    VB_STAMP();
  VB_STAMP();
  }
}

}  // namespace tmg
