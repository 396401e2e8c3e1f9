// Tile kernels for the small coarse levels.
//
// The two-stage marching kernels (tmg_smarch.cuh) stream a level column by
// column through a TMA ring; on a level of a few thousand nodes a CTA marches
// one or two output columns plus the ring fill, and the pass costs ~9 us of
// pipeline latency whatever its size. Here a CTA instead loads a square
// region of the level (its nodes plus the halo the two stages read) into
// shared memory with plain loads and runs the stages over it with block
// barriers: the same V(2,2) halves as the marching kernels, with the same
// per-node arithmetic in the same order (s_apply, s_jacobi_r, the
// restriction sums), so the results are bitwise those of the marching path.
//
//   DOWN (coarse block of TC x TC nodes, level region 2 TC + 5 wide):
//     x1 = omega f / D; x2 = x1 + omega D^-1 (f - A x1) (written out);
//     r = f - A x2; f_c = (1/4) P^T r
//   UP (level block of 2 TC x 2 TC nodes, region 2 TC + 4 wide):
//     w = x2 + P u_c; x3 = w + omega D^-1 (f - A w);
//     x4 = x3 + omega D^-1 (f - A x3) (written out)
#pragma once

#include <cuda_runtime.h>

#include "tmg_device.cuh"
#include "tmg_smarch.cuh"

namespace tmg {

// Tile sizes: DOWN covers TC x TC coarse nodes per CTA, UP 2 TC x 2 TC level
// nodes. The stages of a tile are issue-bound on one SM (a %globaltimer trace
// of the 8-node tiles: ~1 us per stage for a 441-node region), so the small
// levels take small tiles spread over more SMs: the halo redundancy costs
// nothing there, the per-SM node count sets the stage time.
template <int TC>
__host__ __device__ constexpr int t_threads() { return TC >= 8 ? 512 : (TC >= 4 ? 256 : (TC >= 2 ? 128 : 64)); }
template <bool UP, int TC>
__host__ __device__ constexpr int t_side() { return UP ? 2 * TC + 4 : 2 * TC + 5; }
template <bool UP, int TC>
__host__ __device__ constexpr int t_nodes() { return t_side<UP, TC>() * t_side<UP, TC>(); }
template <int TC>
__host__ __device__ constexpr int t_uc_side() { return TC + 4; }  // UP coarse region side
// default size limit of a tile-kernel level (nodes); TMG_STILE_MAX_NODES overrides
constexpr long kTileMaxNodes = 257L * 257L;
// default tile sizes by level size (measured, c0/c1/c2/c3): 2-node tiles up to
// 65^2 nodes, 4-node tiles up to 129^2, 8-node tiles above
constexpr long kTileTC2Nodes = 65L * 65L, kTileTC4Nodes = 129L * 129L;

// shared memory: planes, f, the reciprocal diagonal, two stage buffers, then
// (DOWN) the residual block
// or (UP) x2 and the coarse correction
// planes region in doubles, padded to 16 bytes for the double2 buffers after it
template <bool UP, int TC>
__host__ __device__ constexpr int t_plane_doubles() { return (kStencilPlanes * t_nodes<UP, TC>() + 1) & ~1; }
template <bool UP, int TC>
__host__ __device__ constexpr int t_smem() {
  return t_plane_doubles<UP, TC>() * 8 + t_nodes<UP, TC>() * 4 * 16 +
         (UP ? t_nodes<true, TC>() * 16 + t_uc_side<TC>() * t_uc_side<TC>() * 16 : (2 * TC + 1) * (2 * TC + 1) * 16);
}

// plane k of the region column whose row 0 is `col` (plane stride = region nodes)
template <int N>
struct TPlanes {
  const double* col;
  __device__ __forceinline__ double at(int k, int j) const { return col[k * N + j]; }
};

template <bool UP, int TC>
__global__ void __launch_bounds__(t_threads<TC>()) k_stile(const __grid_constant__ SMarchArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int W = t_side<UP, TC>();
  constexpr int N = t_nodes<UP, TC>();
  constexpr int kTThreads = t_threads<TC>();
  constexpr int kTU = 2 * TC, kTUC = t_uc_side<TC>(), kTC = TC;
  double* pl = reinterpret_cast<double*>(smem_raw);       // [19][W][W]
  double2* fv = reinterpret_cast<double2*>(pl + t_plane_doubles<UP, TC>());
  double2* rcv = fv + N;  // 1/D of the region (rcp_nr of planes 0 and 2), formed once
  double2* sa = rcv + N;  // stage-A inputs (x1 / w)
  double2* sb = sa + N;  // stage-A outputs (x2 / x3)
  double2* ex = sb + N;  // DOWN: residual block; UP: x2 over the region, then u_c
  const Grid& g = a.g;
  const int t = threadIdx.x;
  // region origin (level node of local (0, 0))
  const int ox = UP ? blockIdx.y * kTU - 2 : 2 * blockIdx.y * kTC - 3;
  const int oy = UP ? blockIdx.x * kTU - 2 : 2 * blockIdx.x * kTC - 3;
  auto in_level = [&](int x, int y) { return g.x0 + x >= 0 && g.x0 + x <= g.nx && y >= 0 && y <= g.ny; };
  const double2 z2 = make_double2(0.0, 0.0);
  // ---- load the region (zeros outside the level, where every array is
  // zero), one node per thread. A launch with programmatic stream
  // serialization starts while its predecessor still runs; until
  // griddepcontrol.wait it only issues loads, into registers, of data no
  // kernel of the solve writes (the stencil planes, from setup) or that the
  // kernel two launches back finished (UP: f and x2, from this level's DOWN
  // half; every tile kernel lets its dependent launch only after its own
  // wait). Nothing is stored before the wait (the conservative form; see the
  // dependent-launch race in DESIGN.md section 4).
  static_assert(N <= kTThreads, "one region node per thread");
  const int n0 = t;
  const bool own = n0 < N;
  const int x0n = ox + n0 / W, y0n = oy + n0 % W;
  const bool in0 = own && in_level(x0n, y0n);
  const long i0 = in0 ? g.idx(x0n, y0n) : 0;
  double p[kStencilPlanes];
#pragma unroll
  for (int k = 0; k < kStencilPlanes; ++k) p[k] = in0 ? a.S[k * g.size + i0] : 0.0;
  double2 f0 = z2, x20 = z2;
  if (UP && in0) {
    f0 = a.f[i0];
    x20 = a.x2[i0];
  }
  grid_dep_wait();
  grid_dep_launch();
  if (own) {
#pragma unroll
    for (int k = 0; k < kStencilPlanes; ++k) pl[k * N + n0] = p[k];
    // the reciprocal diagonal (rcp_nr of planes 0 and 2, the d of s_apply),
    // formed once for the DOWN stage-A input and stage A, UP stages A and B
    rcv[n0] = make_double2(rcp_nr(p[0]), rcp_nr(p[2]));
    fv[n0] = UP ? f0 : (in0 ? a.f[i0] : z2);
    if (UP) ex[n0] = x20;
  }
  double2* uc = ex + N;  // UP: coarse region kTUC x kTUC from coarse node (cx0, cy0)
  const int cx0 = (ox >> 1) - 1, cy0 = (oy >> 1) - 1;  // ox, oy even for UP
  if (UP) {
    for (int n = t; n < kTUC * kTUC; n += kTThreads) {
      const int X = cx0 + n / kTUC, Y = cy0 + n % kTUC;
      const bool in = a.gc.x0 + X >= 0 && a.gc.x0 + X <= a.gc.nx && Y >= 0 && Y <= a.gc.ny;
      uc[n] = in ? a.uc[a.gc.idx(X, Y)] : z2;
    }
  }
  __syncthreads();
  auto D = [&](int n) { return rcv[n]; };
  // y = A v at local (i, j) over the buffer v, its diagonal in d
  auto apply = [&](const double2* v, int i, int j, double2& y, double2& d) {
    double2 l[3], c[3], r[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      l[q] = v[(i - 1) * W + j - 1 + q];
      c[q] = v[i * W + j - 1 + q];
      r[q] = v[(i + 1) * W + j - 1 + q];
    }
    s_apply(TPlanes<N>{pl + i * W}, TPlanes<N>{pl + (i - 1) * W}, j, l, c, r, y, d);
  };
  // ---- stage-A inputs over the whole region
  for (int n = t; n < N; n += kTThreads) {
    const int i = n / W, j = n % W, x = ox + i, y = oy + j;
    double2 v;
    if (!UP) {
      // x1 = omega f / D (the marching kernels' a_in_down)
      const double2 f = fv[n], rc = D(n);
      v = make_double2(a.omega * f.x * rc.x, a.omega * f.y * rc.y);
    } else {
      // w = x2 + P u_c (a_in_up): coarse column ceil(x/2), and for odd x the
      // mean with floor(x/2); odd rows interpolate the coarse rows
      const int gy = y - 2 * cy0;
      auto colv = [&](int X) {
        const double2 p = uc[(X - cx0) * kTUC + (gy >> 1)], q = uc[(X - cx0) * kTUC + (gy >> 1) + 1];
        return (gy & 1) ? make_double2(0.5 * p.x + 0.5 * q.x, 0.5 * p.y + 0.5 * q.y) : p;
      };
      const int gx = g.x0 + x;
      double2 pu = colv((x + 1) >> 1);
      if (gx & 1) {
        const double2 q = colv(x >> 1);
        pu = make_double2(0.5 * q.x + 0.5 * pu.x, 0.5 * q.y + 0.5 * pu.y);
      }
      const double2 xv = ex[n];
      v = make_double2(xv.x + pu.x, xv.y + pu.y);
    }
    sa[n] = in_level(x, y) ? v : z2;
  }
  __syncthreads();
  // ---- stage A: one damped-Jacobi sweep on the region minus one ring
  for (int n = t; n < (W - 2) * (W - 2); n += kTThreads) {
    const int i = 1 + n / (W - 2), j = 1 + n % (W - 2), x = ox + i, y = oy + j;
    const int m = i * W + j;
    double2 yv, d;
    apply(sa, i, j, yv, d);
    const double2 rc = D(m);  // = rcp_nr of d = (c00, c11), planes 0 and 2
    const double2 v = in_level(x, y) ? s_jacobi_r(sa[m], fv[m], yv, rc, a.omega) : z2;
    sb[m] = v;
    // DOWN: x2 of the level nodes this CTA owns (level block [2X0, 2X0+2kTC))
    if (!UP && i >= 3 && i < 3 + 2 * kTC && j >= 3 && j < 3 + 2 * kTC && x < g.ncol && y <= g.ny)
      a.out[g.idx(x, y)] = v;
  }
  __syncthreads();
  // ---- stage B on the region minus two rings
  for (int n = t; n < (W - 4) * (W - 4); n += kTThreads) {
    const int i = 2 + n / (W - 4), j = 2 + n % (W - 4), x = ox + i, y = oy + j;
    const int m = i * W + j;
    double2 yv, d;
    apply(sb, i, j, yv, d);
    const bool ok = in_level(x, y);
    if (UP) {
      const double2 v = ok ? s_jacobi_r(sb[m], fv[m], yv, D(m), a.omega) : z2;
      if (x < g.ncol && y <= g.ny && x >= 0) a.out[g.idx(x, y)] = v;
    } else {
      ex[(i - 2) * (W - 4) + (j - 2)] = ok ? make_double2(fv[m].x - yv.x, fv[m].y - yv.y) : z2;
    }
  }
  if (UP) return;
  __syncthreads();
  // ---- DOWN: restriction (1/4) P^T r in the marching kernel's order: rows
  // (1/2, 1, 1/2) around the even level row, then columns 2X-1, 2X, 2X+1
  constexpr int RW = W - 4;  // residual block side (level nodes 2X0-1 .. 2X0+2kTC-1)
  for (int n = t; n < kTC * kTC; n += kTThreads) {
    const int X = blockIdx.y * kTC + n / kTC, Y = blockIdx.x * kTC + n % kTC;
    if (X >= a.gc.ncol || Y > a.gc.ny) continue;
    const int ci = 2 * (n / kTC) + 1, cj = 2 * (n % kTC) + 1;  // residual-block position of (2X, 2Y)
    auto rs = [&](int i) {
      const double2 rm = ex[i * RW + cj - 1], r0 = ex[i * RW + cj], rp = ex[i * RW + cj + 1];
      return make_double2(fma(0.5, rm.x + rp.x, r0.x), fma(0.5, rm.y + rp.y, r0.y));
    };
    const double2 s0 = rs(ci - 1), s1 = rs(ci), s2 = rs(ci + 1);
    double2 acc = make_double2(0.5 * s0.x, 0.5 * s0.y);
    acc.x += s1.x;
    acc.y += s1.y;
    acc.x = fma(0.5, s2.x, acc.x);
    acc.y = fma(0.5, s2.y, acc.y);
    a.fc[a.gc.idx(X, Y)] = make_double2(0.25 * acc.x, 0.25 * acc.y);
  }
}

}  // namespace tmg
