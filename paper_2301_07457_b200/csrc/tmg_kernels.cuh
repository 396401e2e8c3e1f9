// sm_100a kernels of the pCGMG path. All fp64, HBM-bound stencils: no tensor
// cores (FP64 MMA is not a Blackwell lever and the arithmetic intensity is
// ~2-3 flop/B). See DESIGN.md section 4 for the per-kernel byte counts.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "tmg_device.cuh"

namespace tmg {

constexpr int kBX = 64;  // threads along y (contiguous) per block
constexpr int kBY = 4;   // threads along x per block
constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 148 * 8;  // fixed grid => fixed reduction order

// ------------------------------------------------------------ reductions --

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum in a fixed tree order; result valid in thread 0.
template <int NT>
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[NT / 32];
  const int t = threadIdx.x + threadIdx.y * blockDim.x;
  v = warp_sum(v);
  if ((t & 31) == 0) sh[t >> 5] = v;
  __syncthreads();
  double r = 0.0;
  if (t < 32) {
    r = (t < NT / 32) ? sh[t] : 0.0;
    r = warp_sum(r);
  }
  __syncthreads();
  return r;
}

// Scalars of the PCG recurrence (pcg_solve, solvers.cpp:332-395), resident on
// the device so iterations chain without host round trips.
struct PcgState {
  double tol;  // stopping tolerance of the running solve (device-side stopping test)
  double* hist;  // device-side loop: residual history (mapped pinned host memory)
  int max_iter;  // device-side loop: iteration cap
  double bnorm;
  double rr, zr, zr_prev, pap, alpha, beta, relres;
  int it;      // iteration being computed (1-based)
  int status;  // 0 ok, 4 preconditioner (zr <= 0), 3 definiteness (pAp <= 0)
};

// Mirror written by the reducing block to mapped pinned host memory.
struct HostMirror {
  double relres;
  double zr, pap, rr;
  int status;
  int it;
};

// Small device values the host needs mid-solve, written by a kernel into
// mapped pinned memory. A cudaMemcpyAsync D2H would queue behind any large
// device-to-host copy in flight on the same copy engine (the pipelined
// solves download the previous solution while the next one runs).
struct Readback {
  double bnorm;  // PcgState::bnorm
  double scal0;  // scal[0] (the plain value of the last reduction)
  int bad_row;   // coarsest Cholesky: first non-positive pivot, or -1
};
__global__ void k_readback(const int* bad_row, const PcgState* st, const double* scal, Readback* out) {
  if (bad_row) out->bad_row = *bad_row;
  if (st) out->bnorm = st->bnorm;
  if (scal) out->scal0 = scal[0];
}

enum RedOp { kRedNone = 0, kRedZr = 1, kRedPap = 2, kRedRr = 3, kRedB = 4, kRedPlain = 5 };

__device__ __forceinline__ void apply_scalar(RedOp op, double acc, PcgState* st, HostMirror* hm, double* out);

// Fixed-order sum of p[0 .. n): exactly 128 lanes (the first four warps of
// the block; blockDim >= 128) stride the array, then a fixed tree. The order
// depends on n only, never on the launch that calls it, so the in-kernel
// finish of a single-rank reduction and k_finish after a multi-rank
// all-reduce of the same partial array give bitwise-equal sums. Valid in
// every thread; every thread of the block must call it.
__device__ __forceinline__ double fixed_sum(const double* p, int n) {
  __shared__ double sh[4];
  const int t = threadIdx.x + threadIdx.y * blockDim.x;
  if (t < 128) {
    // eight loads in flight per lane (__ldcg is an asm volatile: one add per
    // load would expose an L2 round trip every few elements); the adds keep
    // the lane's increasing-k order, so the sum is bitwise unchanged
    double acc = 0.0;
    int k = t;
    for (; k + 7 * 128 < n; k += 8 * 128) {
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __ldcg(p + k + j * 128);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc += v[j];
    }
    for (; k < n; k += 128) acc += __ldcg(p + k);
    acc = warp_sum(acc);
    if ((t & 31) == 0) sh[t >> 5] = acc;
  }
  __syncthreads();
  const double r = (sh[0] + sh[1]) + (sh[2] + sh[3]);
  __syncthreads();
  return r;
}

// Per-CTA partial into partials[pidx]; then, with a ticket (single rank), the
// last CTA to finish sums all nparts partials in the fixed order and applies
// `op`. Without a ticket (several ranks) the partials stay for the
// all-reduce and k_finish. The partial index is a global tile index
// (DESIGN.md section 5), so 1..N ranks produce the same partial array.
template <int NT>
__device__ __forceinline__ void finish_reduction(double part, double* partials, int pidx, unsigned* ticket,
                                                 int nlocal, int nparts, RedOp op, PcgState* st,
                                                 HostMirror* hm, double* out) {
  const int t = threadIdx.x + threadIdx.y * blockDim.x;
  const double s = block_sum<NT>(part);
  __shared__ bool last;
  if (t == 0) {
    partials[pidx] = s;
    if (ticket) {
      __threadfence();
      last = (atomicAdd(ticket, 1u) == static_cast<unsigned>(nlocal - 1));
    } else {
      last = false;
    }
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const double acc = fixed_sum(partials, nparts);
  if (t != 0) return;
  *ticket = 0u;
  apply_scalar(op, acc, st, hm, out);
}

// one partial per CTA of the grid, in block order (single-rank launches)
template <int NT>
__device__ __forceinline__ void finish_reduction(double part, double* partials, unsigned* ticket, int nblocks,
                                                 RedOp op, PcgState* st, HostMirror* hm, double* out) {
  finish_reduction<NT>(part, partials, blockIdx.x + blockIdx.y * gridDim.x, ticket, nblocks, nblocks, op, st, hm,
                       out);
}

// Scalar tail of a reduction: the global sum `acc` updates the PCG state
// (single rank: called by the last block; several ranks: by k_scalar after
// the all-reduce of the per-rank partials).
__device__ __forceinline__ void apply_scalar(RedOp op, double acc, PcgState* st, HostMirror* hm, double* out) {
  if (out) *out = acc;
  if (!st) return;
  switch (op) {
    case kRedZr: {
      // solvers.cpp:360-371
      st->zr = acc;
      if (!(acc > 0.0) && st->status == 0) st->status = 4;
      st->beta = (st->it == 1) ? 0.0 : acc / st->zr_prev;
      st->zr_prev = acc;
      if (hm) {
        hm->zr = acc;
        hm->status = st->status;
      }
      break;
    }
    case kRedPap: {
      // solvers.cpp:373-382
      st->pap = acc;
      if (!(acc > 0.0) && st->status == 0) st->status = 3;
      st->alpha = st->zr / acc;
      if (hm) {
        hm->pap = acc;
        hm->status = st->status;
      }
      break;
    }
    case kRedRr: {
      // solvers.cpp:383-390 (norm2(r) / bnorm)
      st->rr = acc;
      st->relres = sqrt(acc) / st->bnorm;
      if (hm) {
        hm->rr = acc;
        hm->relres = st->relres;
        hm->status = st->status;
        hm->it = st->it;
      }
      st->it += 1;
      break;
    }
    case kRedB: {
      st->bnorm = sqrt(acc);
      break;
    }
    default:
      break;
  }
}

// Multi-rank reductions: the ranks' partial arrays (each rank fills its own
// tiles, zeros elsewhere) are summed elementwise, which is exact, then every
// rank finishes the same array in the fixed order (one block of 128).
__global__ void __launch_bounds__(128) k_finish(const double* parts, int n, RedOp op, PcgState* st,
                                                HostMirror* hm, double* out) {
  const double acc = fixed_sum(parts, n);
  if (threadIdx.x == 0) apply_scalar(op, acc, st, hm, out);
}
// in-process ranks: elementwise sum of the partial arrays in rank order
__global__ void k_sum_parts(const double* const* parts, int nr, double* const* outs, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int r = 0; r < nr; ++r) s += parts[r][i];
  for (int r = 0; r < nr; ++r) outs[r][i] = s;
}

// --------------------------------------------------------- node kernels --

struct NodeIdx {
  int x, y;
  bool ok;
};

__device__ __forceinline__ NodeIdx node_of_thread(const Grid& g) {
  NodeIdx n;
  n.y = blockIdx.x * kBX + threadIdx.x;
  n.x = blockIdx.y * kBY + threadIdx.y;
  n.ok = (n.x < g.ncol) && (n.y <= g.ny);
  return n;
}

// y = A x, optionally with partial x.y for a fused dot (K1 / K5 / K9).
template <class Op, bool DOT>
__global__ void __launch_bounds__(kBX* kBY) k_apply(Op op, Grid g, const double2* __restrict__ x,
                                                    double2* __restrict__ y, double* partials,
                                                    unsigned* ticket, RedOp rop, PcgState* st,
                                                    HostMirror* hm, double* out) {
  const NodeIdx n = node_of_thread(g);
  double part = 0.0;
  if (n.ok) {
    const long i = g.idx(n.x, n.y);
    double2 r, d;
    op.apply(x, i, r, d);
    y[i] = r;
    if (DOT) {
      const double2 xi = x[i];
      part = xi.x * r.x + xi.y * r.y;
    }
  }
  if (DOT) finish_reduction<kBX * kBY>(part, partials, ticket, gridDim.x * gridDim.y, rop, st, hm, out);
}

// Damped-Jacobi sweep x_out = x_in + omega D^-1 (f - A x_in) (jacobi_sweep,
// solvers.cpp:30-37). ZERO: x_in is the zero vector (first pre-smoothing
// sweep of a visit that starts from u = 0): x_out = omega f / D.
template <class Op, bool ZERO>
__global__ void __launch_bounds__(kBX* kBY) k_sweep(Op op, Grid g, const double2* __restrict__ xin,
                                                    double2* __restrict__ xout,
                                                    const double2* __restrict__ f, double omega) {
  const NodeIdx n = node_of_thread(g);
  if (!n.ok) return;
  const long i = g.idx(n.x, n.y);
  const double2 fi = f[i];
  double2 ax, d;
  if (ZERO) {
    d = op.diag(i);
    xout[i] = make_double2(omega * fi.x / d.x, omega * fi.y / d.y);
  } else {
    op.apply(xin, i, ax, d);
    const double2 xi = xin[i];
    xout[i] = make_double2(xi.x + omega * (fi.x - ax.x) / d.x, xi.y + omega * (fi.y - ax.y) / d.y);
  }
}

// r = f - A x (solvers.cpp:498-499)
template <class Op>
__global__ void __launch_bounds__(kBX* kBY) k_residual(Op op, Grid g, const double2* __restrict__ x,
                                                       const double2* __restrict__ f,
                                                       double2* __restrict__ r) {
  const NodeIdx n = node_of_thread(g);
  if (!n.ok) return;
  const long i = g.idx(n.x, n.y);
  double2 ax, d;
  op.apply(x, i, ax, d);
  const double2 fi = f[i];
  r[i] = make_double2(fi.x - ax.x, fi.y - ax.y);
}

// f_c = (1/4) P^T r as a gather over the 3x3 fine children of each coarse
// node (restrict, grid.cpp:122-142). Ghost fine nodes hold 0.
__global__ void __launch_bounds__(kBX* kBY) k_restrict(Grid cg, Grid fg, const double2* __restrict__ r,
                                                       double2* __restrict__ fc) {
  const NodeIdx n = node_of_thread(cg);
  if (!n.ok) return;
  const long c = fg.idx(2 * n.x, 2 * n.y);
  const double w[3] = {0.5, 1.0, 0.5};
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int dx = -1; dx <= 1; ++dx) {
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
      const double2 v = r[c + dx * fg.P + dy];
      const double ww = 0.25 * w[dx + 1] * w[dy + 1];
      s0 = fma(ww, v.x, s0);
      s1 = fma(ww, v.y, s1);
    }
  }
  fc[cg.idx(n.x, n.y)] = make_double2(s0, s1);
}

// x (+)= P u_c, bilinear (prolongate, grid.cpp:98-120 + solvers.cpp:508-509).
template <bool ADD>
__global__ void __launch_bounds__(kBX* kBY) k_prolong(Grid fg, Grid cg, const double2* __restrict__ uc,
                                                      double2* __restrict__ x) {
  const NodeIdx n = node_of_thread(fg);
  if (!n.ok) return;
  const int X0 = n.x >> 1, Y0 = n.y >> 1;
  const bool ox = n.x & 1, oy = n.y & 1;
  double s0, s1;
  const long c = cg.idx(X0, Y0);
  const double2 a = uc[c];
  if (!ox && !oy) {
    s0 = a.x;
    s1 = a.y;
  } else if (ox && !oy) {
    const double2 b = uc[c + cg.P];
    s0 = 0.5 * a.x + 0.5 * b.x;
    s1 = 0.5 * a.y + 0.5 * b.y;
  } else if (!ox && oy) {
    const double2 b = uc[c + 1];
    s0 = 0.5 * a.x + 0.5 * b.x;
    s1 = 0.5 * a.y + 0.5 * b.y;
  } else {
    const double2 b = uc[c + 1], e = uc[c + cg.P], f = uc[c + cg.P + 1];
    s0 = 0.25 * a.x + 0.25 * b.x + 0.25 * e.x + 0.25 * f.x;
    s1 = 0.25 * a.y + 0.25 * b.y + 0.25 * e.y + 0.25 * f.y;
  }
  const long i = fg.idx(n.x, n.y);
  if (ADD) {
    const double2 xi = x[i];
    x[i] = make_double2(xi.x + s0, xi.y + s1);
  } else {
    x[i] = make_double2(s0, s1);
  }
}

// ------------------------------------------------------- Galerkin (K6) --

__host__ __device__ constexpr double pw(int o) { return o == 0 ? 1.0 : 0.5; }

// Coarse stencil of node (X, Y): (1/4) sum_{i,j} P(i,I) A(i,j) P(j,J)
// (galerkin_coarse_matrix, solvers.cpp:397-458), evaluated as a gather over
// the 3x3 fine children i of I and their 3x3 fine neighbours j; the parents
// of j are always inside I's 3x3 coarse neighbourhood. Only the centre and the
// four forward blocks are stored (symmetry).
template <class Op>
__device__ __forceinline__ void galerkin_gather(const Op& fine, const Grid& fg, int X, int Y, double (&acc)[5][4]) {
#pragma unroll
  for (int a = 0; a < 5; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  // slot of coarse offset (ox, oy): centre 0, N 1, SE 2, E 3, NE 4, else -1
#pragma unroll
  for (int dx = -1; dx <= 1; ++dx) {
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
      const int fx = 2 * X + dx, fy = 2 * Y + dy;
      if (fg.x0 + fx < 0 || fg.x0 + fx > fg.nx || fy < 0 || fy > fg.ny) continue;  // global bounds
      const long i = fg.idx(fx, fy);
      const double wi = 0.25 * pw(dx) * pw(dy);
#pragma unroll
      for (int ex = -1; ex <= 1; ++ex) {
#pragma unroll
        for (int ey = -1; ey <= 1; ++ey) {
          const int jx = dx + ex, jy = dy + ey;  // fine offset of j from (2X, 2Y)
          // parents of j along each axis: even -> one (weight 1), odd -> two (1/2)
          const int nxp = (jx & 1) ? 2 : 1, nyp = (jy & 1) ? 2 : 1;
          bool any = false;
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              if (a >= nxp || c >= nyp) continue;
              const int ox = (jx & 1) ? ((jx - 1) / 2 + a) : jx / 2;
              const int oy = (jy & 1) ? ((jy - 1) / 2 + c) : jy / 2;
              const bool fwd = (ox == 0 && oy == 0) || (ox == 0 && oy == 1) || (ox == 1);
              any = any || fwd;
            }
          if (!any) continue;
          double b[4];
          fine.block(i, ex, ey, b);
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              if (a >= nxp || c >= nyp) continue;
              const int ox = (jx & 1) ? ((jx - 1) / 2 + a) : jx / 2;
              const int oy = (jy & 1) ? ((jy - 1) / 2 + c) : jy / 2;
              int slot = -1;
              if (ox == 0 && oy == 0) slot = 0;
              else if (ox == 0 && oy == 1) slot = 1;
              else if (ox == 1 && oy == -1) slot = 2;
              else if (ox == 1 && oy == 0) slot = 3;
              else if (ox == 1 && oy == 1) slot = 4;
              if (slot < 0) continue;
              const double w = wi * ((jx & 1) ? 0.5 : 1.0) * ((jy & 1) ? 0.5 : 1.0);
#pragma unroll
              for (int q = 0; q < 4; ++q) acc[slot][q] = fma(w, b[q], acc[slot][q]);
            }
        }
      }
    }
  }
}

template <class Op>
__global__ void __launch_bounds__(128) k_galerkin(Op fine, Grid fg, Grid cg, double* __restrict__ Sc,
                                                  long LSc) {
  const int Y = blockIdx.x * 32 + threadIdx.x;
  const int X = blockIdx.y * 4 + threadIdx.y;
  if (X >= cg.ncol || Y > cg.ny) return;
  double acc[5][4];
  galerkin_gather(fine, fg, X, Y, acc);
  const long I = cg.idx(X, Y);
  Sc[0 * LSc + I] = acc[0][0];
  Sc[1 * LSc + I] = acc[0][1];
  Sc[2 * LSc + I] = acc[0][3];
#pragma unroll
  for (int s = 1; s < 5; ++s)
#pragma unroll
    for (int q = 0; q < 4; ++q) Sc[(3 + 4 * (s - 1) + q) * LSc + I] = acc[s][q];
}

// Level nc-1 from the fine level, per coarse cell. Every fine element lies in
// one coarse cell C and its nodes interpolate from C's four corners only, so
// away from fixed dofs (1/4) P^T A P = sum_C sum_q E_{C,q} M_q with four
// constant 8x8 matrices M_q = (1/4) P_q^T Ke P_q (q = the element's quadrant
// of C; c_mq, built on the host from the device Ke). A coarse node's five
// stored blocks then cost 144 FMAs over the 4x4 moduli around it instead of
// the 81-block gather of k_galerkin. Nodes with a fixed dof among the 5x5
// fine nodes around them take the general gather (identity rows, masks).
__constant__ double c_mq[4][64];

__global__ void __launch_bounds__(128) k_galerkin_cells(FineOp fine, Grid fg, Grid cg, double* __restrict__ Sc,
                                                        long LSc) {
  const int Y = blockIdx.x * 32 + threadIdx.x;
  const int X = blockIdx.y * 4 + threadIdx.y;
  if (X >= cg.ncol || Y > cg.ny) return;
  const long c = fg.idx(2 * X, 2 * Y);
  bool fixed = false;
#pragma unroll
  for (int dx = -2; dx <= 2; ++dx)
#pragma unroll
    for (int dy = -2; dy <= 2; ++dy) fixed = fixed || fine.M[c + dx * fg.P + dy] != 0;
  double acc[5][4];
  if (fixed) {
    galerkin_gather(fine, fg, X, Y, acc);
  } else {
    // moduli of the 4x4 fine elements around the node: e[u][v] = element
    // (2X - 2 + u, 2Y - 2 + v)
    double e[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) e[u][v] = fine.E[c + (u - 2) * fg.P + (v - 2)];
    // block (a, b) of cell (cx, cy) (offsets 0/1 from X-1, Y-1), summed into acc[slot]
    auto cell = [&](int cx, int cy, int a, int b, double (&out)[4]) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double w = e[2 * cx + (q & 1)][2 * cy + (q >> 1)];
        out[0] = fma(w, c_mq[q][(2 * a) * 8 + 2 * b], out[0]);
        out[1] = fma(w, c_mq[q][(2 * a) * 8 + 2 * b + 1], out[1]);
        out[2] = fma(w, c_mq[q][(2 * a + 1) * 8 + 2 * b], out[2]);
        out[3] = fma(w, c_mq[q][(2 * a + 1) * 8 + 2 * b + 1], out[3]);
      }
    };
#pragma unroll
    for (int k = 0; k < 5; ++k)
#pragma unroll
      for (int m = 0; m < 4; ++m) acc[k][m] = 0.0;
    // corners: (0,0)->0 (1,0)->1 (1,1)->2 (0,1)->3; cell (1,1) is (X, Y)
    cell(0, 0, 2, 2, acc[0]);  // centre: I is corner 2 of (X-1, Y-1)
    cell(1, 0, 3, 3, acc[0]);  //         corner 3 of (X, Y-1)
    cell(1, 1, 0, 0, acc[0]);  //         corner 0 of (X, Y)
    cell(0, 1, 1, 1, acc[0]);  //         corner 1 of (X-1, Y)
    cell(0, 1, 1, 2, acc[1]);  // N
    cell(1, 1, 0, 3, acc[1]);
    cell(1, 0, 3, 1, acc[2]);  // SE
    cell(1, 0, 3, 2, acc[3]);  // E
    cell(1, 1, 0, 1, acc[3]);
    cell(1, 1, 0, 2, acc[4]);  // NE
  }
  const long I = cg.idx(X, Y);
  Sc[0 * LSc + I] = acc[0][0];
  Sc[1 * LSc + I] = acc[0][1];
  Sc[2 * LSc + I] = acc[0][3];
#pragma unroll
  for (int s = 1; s < 5; ++s)
#pragma unroll
    for (int q = 0; q < 4; ++q) Sc[(3 + 4 * (s - 1) + q) * LSc + I] = acc[s][q];
}

// ------------------------------------------------- coarsest level (K7) --

// Dense coarsest matrix in the reference dof order (row-major n x n).
template <class Op>
__global__ void k_dense_assemble(Op op, Grid g, double* __restrict__ A, int n) {
  const int y = blockIdx.x * blockDim.x + threadIdx.x;
  const int x = blockIdx.y;
  if (x >= g.ncol || y > g.ny) return;
  const long i = g.idx(x, y);
  const int ri = 2 * (x * (g.ny + 1) + y);
  for (int ex = -1; ex <= 1; ++ex)
    for (int ey = -1; ey <= 1; ++ey) {
      const int x2 = x + ex, y2 = y + ey;
      if (x2 < 0 || x2 > g.nx || y2 < 0 || y2 > g.ny) continue;
      double b[4];
      op.block(i, ex, ey, b);
      const int cj = 2 * (x2 * (g.ny + 1) + y2);
      A[static_cast<long>(ri) * n + cj] = b[0];
      A[static_cast<long>(ri) * n + cj + 1] = b[1];
      A[static_cast<long>(ri + 1) * n + cj] = b[2];
      A[static_cast<long>(ri + 1) * n + cj + 1] = b[3];
    }
}

// Singular pivot test of the coarsest factorizations. CholeskyFactor::factor
// (solvers.cpp:144-148) raises DefinitenessError at the first pivot that is
// not > 0. For a matrix that is singular in exact arithmetic (an
// unconstrained structure: three rigid motions) that pivot is a rounding
// residue of either sign, and the device's Galerkin operator is not bitwise
// the reference's, so the device also treats a pivot within 16 n eps of the
// row's original diagonal as zero: it then stops at the same (first
// dependent) row as the reference. Legitimate coarsest pivots sit far above
// it (a stiff island held only by 1e-9 void still has ~1e-9 relative pivots,
// 16 n eps = 6e-13 at n = 162).
__device__ __forceinline__ bool pivot_ok(double d, double diag0, int n) {
  return d > 0.0 && d > 16.0 * n * 2.220446049250313e-16 * fabs(diag0);
}

// Right-looking Cholesky, lower triangle in place, one CTA (n <= 2048).
// A non-positive (or numerically zero, pivot_ok) pivot records its row like
// CholeskyFactor::factor (solvers.cpp:144-148).
// SMEM: the matrix is factored in shared memory (n <= kCholSmemMax; the
// same operations in the same order, so the factor is bit-identical).
constexpr int kCholSmemMax = 168;  // 168^2 doubles = 220.5 KB
template <bool SMEM>
__global__ void __launch_bounds__(1024) k_cholesky(double* __restrict__ Ag, int n, int* bad_row) {
  extern __shared__ double As[];
  __shared__ int fail;
  const int t = threadIdx.x, nt = blockDim.x;
  const int lane = t & 31, w = t >> 5, nw = nt >> 5;
  double* A = SMEM ? As : Ag;
  if (SMEM) {
    // two barriers per column: every thread takes the pivot itself, and the
    // scaled column is also staged contiguously (cv) so the trailing update
    // reads it without the bank conflicts of the strided column
    __shared__ double cv[kCholSmemMax];
    double* dg0 = As + n * n;  // original diagonal
    for (int k = t; k < n * n; k += nt) As[k] = Ag[k];
    for (int k = t; k < n; k += nt) dg0[k] = Ag[static_cast<long>(k) * n + k];
    __syncthreads();
    int bad = -1;
    for (int k = 0; k < n; ++k) {
      const double d = A[k * n + k];
      if (!pivot_ok(d, dg0[k], n)) {  // the same d in every thread: a uniform exit
        bad = k;
        break;
      }
      // only the threads that scale an entry (and thread 0, which stores the
      // pivot) take the square root: a redundant DSQRT in all 1024 threads
      // costs more FP64 issue than the barrier it saves
      if (t == 0 || k + 1 + t < n) {
        const double piv = sqrt(d);
        for (int i = k + 1 + t; i < n; i += nt) {
          const double l = A[i * n + k] / piv;
          A[i * n + k] = l;
          cv[i] = l;
        }
        if (t == 0) A[k * n + k] = piv;
      }
      __syncthreads();
      for (int i = k + 1 + w; i < n; i += nw) {
        const double lik = cv[i];
        double* Ai = A + i * n;
        for (int j = k + 1 + lane; j <= i; j += 32) Ai[j] -= lik * cv[j];
      }
      __syncthreads();
    }
    for (int k = t; k < n * n; k += nt) Ag[k] = As[k];
    if (t == 0) *bad_row = bad;
    return;
  }
  __shared__ double dg0g[SMEM ? 1 : 2048];
  if (t == 0) fail = -1;
  for (int k = t; k < n; k += nt) dg0g[k] = Ag[static_cast<long>(k) * n + k];
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    if (t == 0) {
      const double d = A[static_cast<long>(k) * n + k];
      if (!pivot_ok(d, dg0g[k], n)) fail = k;
      else A[static_cast<long>(k) * n + k] = sqrt(d);
    }
    __syncthreads();
    if (fail >= 0) break;
    const double piv = A[static_cast<long>(k) * n + k];
    for (int i = k + 1 + t; i < n; i += nt) A[static_cast<long>(i) * n + k] /= piv;
    __syncthreads();
    for (int i = k + 1 + w; i < n; i += nw) {
      const double lik = A[static_cast<long>(i) * n + k];
      double* Ai = A + static_cast<long>(i) * n;
      for (int j = k + 1 + lane; j <= i; j += 32) Ai[j] -= lik * A[static_cast<long>(j) * n + k];
    }
    __syncthreads();
  }
  if (SMEM) {
    __syncthreads();
    for (int k = t; k < n * n; k += nt) Ag[k] = As[k];
  }
  if (t == 0) *bad_row = fail;
}

// Banded Cholesky of the coarsest matrix in one CTA. With the column-major
// node numbering the 9-point coarsest operator has lower half-bandwidth
// b = 2 (ny + 2) + 1 dofs, and its factor has no fill outside the band (the
// envelope the reference's CholeskyFactor exploits, solvers.cpp:89-148), so
// only the band is staged in shared memory (Bs[i][d] = A[i][i-d]). Step k:
// b threads form the multipliers l_{k+1..k+b} (one division each), then one
// thread per entry of the band triangle subtracts l_i l_j, with a barrier
// after each half. Inside the band every entry sees the same operations in
// the same order as in k_cholesky (outside it both leave exact zeros), so the
// factor and the failing row are bitwise those of the dense kernel. b <= 31.
// (Round 1's one-warp form took each lane's row update as 32 shuffles with a
// shared-memory read-modify-write each: 120 us at n = 162, b = 21; this form
// 79 us.)
constexpr int kCholBandThreads = 256;
__global__ void __launch_bounds__(kCholBandThreads) k_cholesky_band(double* __restrict__ Ag, int n, int b,
                                                                    int* bad_row) {
  extern __shared__ double Bs[];
  __shared__ double lv[32];  // the step's multipliers l_{k+1+a}
  const int t = threadIdx.x, W = b + 1;
  double* dg0 = Bs + n * W;  // original diagonal
  for (int e = t; e < n * W; e += kCholBandThreads) {
    const int i = e / W, d = e - i * W;
    Bs[e] = (i - d >= 0) ? Ag[static_cast<long>(i) * n + i - d] : 0.0;
  }
  for (int k = t; k < n; k += kCholBandThreads) dg0[k] = Ag[static_cast<long>(k) * n + k];
  // the update pairs (a, c), c <= a < b, of the band triangle: thread t
  // owns pair t (b(b+1)/2 <= 496 pairs for b <= 31: two rounds at most)
  int pa[2], pc[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    int q = t + r * kCholBandThreads, a = 0;
    while (a < 31 && q > a) {
      q -= a + 1;
      ++a;
    }
    pa[r] = (a < b) ? a : -1;
    pc[r] = q;
  }
  __syncthreads();
  int bad = -1;
  for (int k = 0; k < n; ++k) {
    const double dk = Bs[k * W];
    if (!pivot_ok(dk, dg0[k], n)) {  // the same value in every thread: a uniform exit
      bad = k;
      break;
    }
    if (t < b) {
      const int i = k + 1 + t;
      const double piv = sqrt(dk);
      if (i < n) {
        const double l = Bs[i * W + t + 1] / piv;  // A[i][k]
        Bs[i * W + t + 1] = l;
        lv[t] = l;
      }
      if (t == 0) Bs[k * W] = piv;
    }
    __syncthreads();
    // A[i][j] -= l_i l_j for k < j <= i: i = k+1+a, j = k+1+c (the same
    // operation on every entry as the one-warp and dense kernels)
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int aa = pa[r], cc = pc[r];
      if (aa >= 0 && k + 1 + aa < n) Bs[(k + 1 + aa) * W + aa - cc] -= lv[aa] * lv[cc];
    }
    __syncthreads();
  }
  for (int e = t; e < n * W; e += kCholBandThreads) {
    const int i = e / W, d = e - i * W;
    if (i - d >= 0) Ag[static_cast<long>(i) * n + i - d] = Bs[e];
  }
  if (t == 0) *bad_row = bad;
}

// Coarsest levels up to kDenseFactorMaxDofs dofs take the one-CTA factor
// kernels (dense, or the band in shared memory); larger ones, up to
// kCoarsestMaxDofs (three dense n x n arrays: 2.3 GB each at the limit),
// factor the band in L2 and form the explicit inverse with the banded /
// tiled kernels (k_cholesky_band_g, k_lower_inverse_band, k_gram_tiled).
constexpr int kDenseFactorMaxDofs = 2048;
constexpr int kCoarsestMaxDofs = 16900;
constexpr int kLargeCoarsestMaxBand = 300;  // lower half-bandwidth (dofs) the one-CTA L2 band factor takes

// Banded Cholesky of a large coarsest matrix (n > 2048: reference configs
// with few coarsenings, e.g. 256^2 with the default num_coarsenings = 2,
// solvers.hpp:25), in place on the band of the dense row-major matrix, one
// CTA. The band (n (b + 1) doubles, a few MB) lives in L2; step k forms the
// b multipliers (one thread each, kept in shared memory) and then one warp
// per row of the band triangle subtracts l_i l_j along the row. The same
// operation on every entry in the same order as k_cholesky / k_cholesky_band.
// dg0: n doubles of scratch for the original diagonal (pivot_ok).
constexpr int kCholBandGThreads = 1024;
__global__ void __launch_bounds__(kCholBandGThreads) k_cholesky_band_g(double* A, int n, int b, double* dg0,
                                                                       int* bad_row) {
  extern __shared__ double lvg[];  // b multipliers
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  constexpr int nw = kCholBandGThreads / 32;
  for (int k = t; k < n; k += kCholBandGThreads) dg0[k] = A[static_cast<long>(k) * n + k];
  __syncthreads();
  int bad = -1;
  for (int k = 0; k < n; ++k) {
    const double dk = A[static_cast<long>(k) * n + k];
    if (!pivot_ok(dk, dg0[k], n)) {  // the same value in every thread: a uniform exit
      bad = k;
      break;
    }
    const double piv = sqrt(dk);
    const int m = min(b, n - 1 - k);  // rows below the pivot inside the band
    for (int a = t; a < m; a += kCholBandGThreads) {
      double* p = A + static_cast<long>(k + 1 + a) * n + k;
      const double l = *p / piv;
      *p = l;
      lvg[a] = l;
    }
    __syncthreads();  // also orders the read of A[k][k] above before its overwrite below
    if (t == 0) A[static_cast<long>(k) * n + k] = piv;
    for (int a = w; a < m; a += nw) {
      const double la = lvg[a];
      double* Ai = A + static_cast<long>(k + 1 + a) * n + k + 1;
      for (int c = lane; c <= a; c += 32) Ai[c] -= la * lvg[c];
    }
    __syncthreads();
  }
  if (t == 0) *bad_row = bad;
}

// Column j of L^-1 for a banded L of any half-bandwidth b (large coarsest
// levels), one warp per column. y_i = -(sum_{k in [max(j, i-b), i)} L_ik y_k)
// / L_ii only reads the last b entries of the column, which are kept in a
// shared-memory ring of RW >= b + 1 doubles per warp (RW a power of two), so
// every column of the matrix has a resident warp at once and the L2 latency
// of a row is hidden by the other columns. Entries above the diagonal are
// written as zeros (k_gram and k_coarse_solve read full rows).
__global__ void k_lower_inverse_band(const double* __restrict__ L, double* __restrict__ LiT, int n, int b,
                                     int RW) {
  extern __shared__ double yring[];
  const int wpb = blockDim.x >> 5;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * wpb + w;
  if (j >= n) return;
  double* yr = yring + static_cast<long>(w) * RW;
  double* out = LiT + static_cast<long>(j) * n;
  for (int i = lane; i < j; i += 32) out[i] = 0.0;
  const double yj = 1.0 / L[static_cast<long>(j) * n + j];
  if (lane == 0) {
    yr[j & (RW - 1)] = yj;
    out[j] = yj;
  }
  __syncwarp();
  for (int i = j + 1; i < n; ++i) {
    const double* Li = L + static_cast<long>(i) * n;
    const double dg = Li[i];
    double s = 0.0;
    for (int k = max(j, i - b) + lane; k < i; k += 32) s = fma(Li[k], yr[k & (RW - 1)], s);
    s = warp_sum(s);
    __syncwarp();  // every lane has read the ring before slot i (= slot i - RW) is rewritten
    if (lane == 0) {
      const double yi = -s / dg;
      yr[i & (RW - 1)] = yi;
      out[i] = yi;
    }
    __syncwarp();
  }
}

// Ainv = L^-T L^-1 for large n: 64x64 tiles of the lower triangle (mirrored
// into the upper one), 4x4 entries per thread, 16 columns of LiT per step
// staged in shared memory. Every entry sums its products in increasing k by
// fma like k_gram; the steps before max(i, j) add exact zeros (LiT is upper
// triangular), so the result is bitwise k_gram's.
constexpr int kGramTile = 64, kGramK = 16;
__global__ void __launch_bounds__(256) k_gram_tiled(const double* __restrict__ LiT, double* __restrict__ Ainv,
                                                    int n) {
  const int bi = blockIdx.y, bj = blockIdx.x;
  if (bj > bi) return;
  __shared__ double As[kGramK][kGramTile + 1];
  __shared__ double Bs[kGramK][kGramTile + 1];
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  const int i0 = bi * kGramTile, j0 = bj * kGramTile;
  double acc[4][4];
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[p][q] = 0.0;
  // rows i >= i0 of LiT are zero left of column i0 (i0 >= j0)
  for (int k0 = i0 / kGramK * kGramK; k0 < n; k0 += kGramK) {
    // 64 rows x 16 columns per operand: thread t loads 4 entries of each
    for (int e = t; e < kGramTile * kGramK; e += 256) {
      const int r = e / kGramK, kk = e % kGramK;
      const int k = k0 + kk;
      const int ia = i0 + r, jb = j0 + r;
      As[kk][r] = (ia < n && k < n) ? LiT[static_cast<long>(ia) * n + k] : 0.0;
      Bs[kk][r] = (jb < n && k < n) ? LiT[static_cast<long>(jb) * n + k] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kGramK; ++kk) {
      double av[4], bv[4];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        av[p] = As[kk][ty * 4 + p];
        bv[p] = Bs[kk][tx * 4 + p];
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = fma(av[p], bv[q], acc[p][q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + ty * 4 + p, j = j0 + tx * 4 + q;
      if (i < n && j < n) {
        Ainv[static_cast<long>(i) * n + j] = acc[p][q];
        if (bi != bj) Ainv[static_cast<long>(j) * n + i] = acc[p][q];
      }
    }
}

// Column j of L^-1 (stored as row j of LiT), one warp per column, the
// running column kept in shared memory.
// b: lower half-bandwidth of L (>= n - 1 when dense); with b <= 31 a row's
// non-zeros left of the diagonal fit one 32-lane chunk.
__global__ void k_lower_inverse(const double* __restrict__ L, double* __restrict__ LiT, int n, int b) {
  extern __shared__ double ycol[];
  const int wpb = blockDim.x >> 5;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * wpb + w;
  if (j >= n) return;
  double* yv = ycol + static_cast<long>(w) * n;
  for (int i = lane; i < n; i += 32) yv[i] = 0.0;
  __syncwarp();
  if (lane == 0) yv[j] = 1.0 / L[static_cast<long>(j) * n + j];
  __syncwarp();
  if (b <= 31) {
    // banded L: row i has non-zeros in columns [i - b, i]; one chunk per row,
    // fetched one step ahead, the diagonal as a precomputed reciprocal
    double cur = 0.0, nxt = 0.0, dcur = 0.0, dnxt = 0.0;
    auto fetch = [&](int i, double& v, double& dg) {
      const double* Li = L + static_cast<long>(i) * n;
      const int k = max(j, i - b) + lane;
      v = (k < i) ? Li[k] : 0.0;
      dg = 1.0 / Li[i];
    };
    if (j + 1 < n) fetch(j + 1, cur, dcur);
    for (int i = j + 1; i < n; ++i) {
      if (i + 1 < n) fetch(i + 1, nxt, dnxt);
      const int k = max(j, i - b) + lane;
      double s = (k < i) ? cur * yv[k] : 0.0;
      s = warp_sum(s);
      if (lane == 0) yv[i] = -s * dcur;
      __syncwarp();
      cur = nxt;
      dcur = dnxt;
    }
  } else if (n <= 192) {
    // rows held in registers one step ahead: the L2 latency of row i+1
    // overlaps the dependent reduction of row i (whose diagonal enters as a
    // precomputed reciprocal)
    double cur[6], nxt[6], dcur = 0.0, dnxt = 0.0;
    auto fetch = [&](int i, double (&v)[6], double& dg) {
      const double* Li = L + static_cast<long>(i) * n;
#pragma unroll
      for (int m = 0; m < 6; ++m) {
        const int k = j + lane + 32 * m;
        v[m] = (k < i) ? Li[k] : 0.0;
      }
      dg = 1.0 / Li[i];  // reciprocal of the diagonal, off the dependent chain
    };
    if (j + 1 < n) fetch(j + 1, cur, dcur);
    for (int i = j + 1; i < n; ++i) {
      if (i + 1 < n) fetch(i + 1, nxt, dnxt);
      double s = 0.0;
#pragma unroll
      for (int m = 0; m < 6; ++m) {
        const int k = j + lane + 32 * m;
        if (k < i) s = fma(cur[m], yv[k], s);
      }
      s = warp_sum(s);
      if (lane == 0) yv[i] = -s * dcur;
      __syncwarp();
#pragma unroll
      for (int m = 0; m < 6; ++m) cur[m] = nxt[m];
      dcur = dnxt;
    }
  } else {
    for (int i = j + 1; i < n; ++i) {
      const double* Li = L + static_cast<long>(i) * n;
      double s = 0.0;
      for (int k = j + lane; k < i; k += 32) s = fma(Li[k], yv[k], s);
      s = warp_sum(s);
      if (lane == 0) yv[i] = -s / Li[i];
      __syncwarp();
    }
  }
  for (int i = lane; i < n; i += 32) LiT[static_cast<long>(j) * n + i] = yv[i];
}

// Ainv = L^-T L^-1 (symmetric), Ainv[i][j] = sum_k LiT[i][k] LiT[j][k].
__global__ void k_gram(const double* __restrict__ LiT, double* __restrict__ Ainv, int n) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (j >= n) return;
  const int k0 = i > j ? i : j;
  const double* a = LiT + static_cast<long>(i) * n;
  const double* b = LiT + static_cast<long>(j) * n;
  double s = 0.0;
  for (int k = k0; k < n; ++k) s = fma(a[k], b[k], s);
  Ainv[static_cast<long>(i) * n + j] = s;
}

// u0 = A0^-1 f0 on the coarsest grid (CholeskyFactor::solve, solvers.cpp:154).
// One warp per node: lanes stride over the input dofs (staged in smem) and
// the warp sums its partials. A thread-per-node loop over all n inputs was a
// 40 us latency chain per V-cycle at n = 162.
constexpr int kCoarseSolveThreads = 256;
__global__ void __launch_bounds__(kCoarseSolveThreads) k_coarse_solve(const double* __restrict__ Ainv, int n,
                                                                      Grid g, const double2* __restrict__ f,
                                                                      double2* __restrict__ u) {
  extern __shared__ double fd[];
  grid_dep_wait();  // f comes from the restriction just before (tile kernels launch this early)
  grid_dep_launch();
  const int rows = g.ny + 1, nodes = n / 2;
  for (int k = threadIdx.x; k < nodes; k += blockDim.x) {
    const double2 v = f[g.idx(k / rows, k % rows)];
    fd[2 * k] = v.x;
    fd[2 * k + 1] = v.y;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int node = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (node >= nodes) return;
  // Ainv is bitwise symmetric (k_gram forms (i, j) and (j, i) with the same
  // operations), so the node's two columns are read as its two rows: the
  // same values in the same order, contiguous across the lanes
  const double* r0 = Ainv + static_cast<long>(2 * node) * n;
  const double* r1 = r0 + n;
  double s0 = 0.0, s1 = 0.0;
  for (int k = lane; k < n; k += 32) {
    const double fk = fd[k];
    s0 = fma(r0[k], fk, s0);
    s1 = fma(r1[k], fk, s1);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  if (lane == 0) u[g.idx(node / rows, node % rows)] = make_double2(s0, s1);
}

// --------------------------------------------------- PCG vector ops (K8) --

// Grid-stride dot over flat padded vectors (ghosts are 0 and add exactly 0).
// Tile geometry of the fine-level reductions: row tiles of kRedRows rows and
// global column tiles of `tx` node columns (the marching kernels' tiles), so
// a partial covers the same nodes, summed in the same order, whatever the
// slab partition. Partial index = row tile + TY * global column tile.
constexpr int kRedRows = 128;
struct RedTiles {
  int tx;      // node columns per tile
  int ctile0;  // global column tile of local column 0 (g.x0 / tx)
  int nparts;  // TY * global column tiles
};

// a.b over the owned nodes; thread = row, marching the tile's columns
__global__ void __launch_bounds__(kRedRows) k_dot(const double2* __restrict__ a, const double2* __restrict__ b,
                                                  Grid g, RedTiles rt, double* partials, unsigned* ticket,
                                                  RedOp op, PcgState* st, HostMirror* hm, double* out) {
  const int y = blockIdx.x * kRedRows + threadIdx.x;
  const int xlo = blockIdx.y * rt.tx, xhi = min(xlo + rt.tx, g.ncol);
  double s = 0.0;
  if (y <= g.ny) {
    for (int x = xlo; x < xhi; ++x) {
      const long i = g.idx(x, y);
      const double2 u = a[i], v = b[i];
      s = fma(u.x, v.x, s);
      s = fma(u.y, v.y, s);
    }
  }
  finish_reduction<kRedRows>(s, partials, blockIdx.x + gridDim.x * (rt.ctile0 + blockIdx.y), ticket,
                             gridDim.x * gridDim.y, rt.nparts, op, st, hm, out);
}

// x += alpha p; r -= alpha Ap; rr = r.r (solvers.cpp:383-386)
__global__ void __launch_bounds__(kRedRows) k_update_xr(double2* __restrict__ x, double2* __restrict__ r,
                                                        const double2* __restrict__ p,
                                                        const double2* __restrict__ ap, Grid g, RedTiles rt,
                                                        double* partials, unsigned* ticket, RedOp rop,
                                                        PcgState* st, HostMirror* hm, double* out) {
  const double alpha = st->alpha;
  const int y = blockIdx.x * kRedRows + threadIdx.x;
  const int xlo = blockIdx.y * rt.tx, xhi = min(xlo + rt.tx, g.ncol);
  double s = 0.0;
  if (y <= g.ny) {
    for (int xc = xlo; xc < xhi; ++xc) {
      const long k = g.idx(xc, y);
      const double2 pp = p[k], aa = ap[k];
      double2 xx = x[k], rr = r[k];
      xx.x += alpha * pp.x;
      xx.y += alpha * pp.y;
      rr.x += -alpha * aa.x;
      rr.y += -alpha * aa.y;
      x[k] = xx;
      r[k] = rr;
      s = fma(rr.x, rr.x, s);
      s = fma(rr.y, rr.y, s);
    }
  }
  finish_reduction<kRedRows>(s, partials, blockIdx.x + gridDim.x * (rt.ctile0 + blockIdx.y), ticket,
                             gridDim.x * gridDim.y, rt.nparts, rop, st, hm, out);
}

// r = b - t (t = A x0) ; plain copy when t == nullptr
__global__ void k_sub(const double2* __restrict__ b, const double2* __restrict__ t,
                      double2* __restrict__ r, long n2) {
  for (long k = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; k < n2;
       k += static_cast<long>(gridDim.x) * blockDim.x) {
    const double2 bb = b[k];
    if (t) {
      const double2 tt = t[k];
      r[k] = make_double2(bb.x - tt.x, bb.y - tt.y);
    } else {
      r[k] = bb;
    }
  }
}

__global__ void k_pcg_begin(PcgState* st, double tol, int max_iter, double* hist) {
  st->tol = tol;
  st->max_iter = max_iter;
  st->hist = hist;
  st->it = 1;
  st->status = 0;
  st->zr_prev = 0.0;
  st->beta = 0.0;
}

// Device-side stopping test between the fused update pass and the rest of a
// PCG iteration graph: r_{it-1} is complete once StSweep01U has run, and when
// it meets the test (solvers.cpp:388) the rest of the iteration (the V-cycle
// and the p-update, speculative work the host would discard) is skipped by
// the graph's conditional node.
__global__ void k_set_continue(cudaGraphConditionalHandle hc, const PcgState* st) {
  const double rel = st->relres;
  cudaGraphSetConditional(hc, (rel <= st->tol || rel == 0.0) ? 0u : 1u);
}

// ---- the whole PCG loop as one graph (a conditional WHILE node whose body
// runs two iterations, one per direction-buffer parity). The host launches it
// once per solve and reads this record when it completes.
struct LoopRecord {
  int iterations;  // completed iterations
  int converged;
  int status;      // 0, or the first breakdown (PcgState::status codes)
  int err_it;      // iteration of the breakdown
  double zr, pap;  // their values (error messages)
  int heads, rests;  // executed heads (update + test) and rests (instrumentation)
};

// After the fused update that completes iteration st->it - 1: record its
// relative residual (residual_history, solvers.cpp:388-391) and run the rest
// of iteration st->it unless the stopping test holds or max_iter iterations
// are complete (pcg_solve's loop bound, solvers.cpp:359); stopping also ends
// the WHILE loop.
__global__ void k_loop_head(cudaGraphConditionalHandle rest, cudaGraphConditionalHandle loop, const PcgState* st,
                            LoopRecord* rec) {
  const int done = st->it - 1;
  const double rel = st->relres;
  st->hist[done] = rel;
  rec->iterations = done;
  rec->heads += 1;
  const bool conv = rel <= st->tol || rel == 0.0;
  rec->converged = conv ? 1 : 0;
  const bool go = !conv && done < st->max_iter;
  cudaGraphSetConditional(rest, go ? 1u : 0u);
  if (!go) cudaGraphSetConditional(loop, 0u);
}

// After the rest of iteration st->it: a breakdown (z.r <= 0 or p.Ap <= 0,
// solvers.cpp:362-380) ends the loop; otherwise `next` (the following
// iteration's guard, or the WHILE handle) lets it continue.
__global__ void k_loop_tail(cudaGraphConditionalHandle next, cudaGraphConditionalHandle loop, const PcgState* st,
                            LoopRecord* rec) {
  rec->rests += 1;
  const bool ok = st->status == 0;
  if (!ok) {
    rec->status = st->status;
    rec->err_it = st->it;
    rec->zr = st->zr;
    rec->pap = st->pap;
    cudaGraphSetConditional(loop, 0u);
  }
  cudaGraphSetConditional(next, ok ? 1u : 0u);
}

// ------------------------------------------------------ consumers (K9-K11)

// u_e^T khat u_e (fem.cpp:292-318), unmasked u, dense element-major output.
__global__ void k_element_energy(Grid g, const double2* __restrict__ u, double* __restrict__ out) {
  const int ey = blockIdx.x * blockDim.x + threadIdx.x;
  const int ex = blockIdx.y;
  if (ey >= g.ny) return;
  const long i = g.idx(ex, ey);
  double ue[8];
  const double2 a = u[i], b = u[i + g.P], c = u[i + g.P + 1], d = u[i + 1];
  ue[0] = a.x; ue[1] = a.y; ue[2] = b.x; ue[3] = b.y;
  ue[4] = c.x; ue[5] = c.y; ue[6] = d.x; ue[7] = d.y;
  double s = 0.0;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    double row = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) row = fma(c_ke64[r * 8 + q], ue[q], row);
    s = fma(ue[r], row, s);
  }
  out[static_cast<long>(ex) * g.ny + ey] = s;
}

// -p alpha^(p-1) E0 * energy for every phase (mto.cpp:61-85)
__global__ void k_sensitivity(long ne, int np, const double* __restrict__ alpha,
                              const double* __restrict__ energy, const double* __restrict__ pm,
                              double pen, double* __restrict__ out) {
  for (long e = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; e < ne;
       e += static_cast<long>(gridDim.x) * blockDim.x) {
    const double en = energy[e];
    for (int i = 0; i < np; ++i) {
      const double a = alpha[e * np + i];
      const double pw1 = (pen == 3.0) ? a * a : pow(a, pen - 1.0);
      out[i * ne + e] = -pen * pw1 * pm[i] * en;
    }
  }
}

// E_e = sum_i alpha_i^p E_i (density.cpp:68-85) into the padded modulus grid
__global__ void k_simp(Grid g, int np, const double* __restrict__ alpha,
                       const double* __restrict__ pm, double pen, double* __restrict__ E) {
  const int ey = blockIdx.x * blockDim.x + threadIdx.x;
  const int ex = blockIdx.y;
  if (ey >= g.ny) return;
  const long e = static_cast<long>(ex) * g.ny + ey;
  double v = 0.0;
  for (int i = 0; i < np; ++i) {
    const double a = alpha[e * np + i];
    const double ap = (pen == 3.0) ? a * a * a : pow(a, pen);
    v += ap * pm[i];
  }
  E[g.idx(ex, ey)] = v;
}

// density-weighted cone sensitivity filter (mto.cpp:87-117)
__global__ void k_filter(int nx, int ny, int np, int phase, double radius, int reach,
                         const double* __restrict__ alpha, const double* __restrict__ raw,
                         double* __restrict__ out) {
  const int ey = blockIdx.x * blockDim.x + threadIdx.x;
  const int ex = blockIdx.y;
  if (ey >= ny) return;
  double acc = 0.0, ws = 0.0;
  const int x0 = max(0, ex - reach), x1 = min(nx - 1, ex + reach);
  const int y0 = max(0, ey - reach), y1 = min(ny - 1, ey + reach);
  for (int jx = x0; jx <= x1; ++jx)
    for (int jy = y0; jy <= y1; ++jy) {
      const double w = radius - sqrt(static_cast<double>((ex - jx) * (ex - jx) + (ey - jy) * (ey - jy)));
      if (w <= 0.0) continue;
      const long j = static_cast<long>(jx) * ny + jy;
      acc += w * alpha[j * np + phase] * raw[j];
      ws += w;
    }
  const long e = static_cast<long>(ex) * ny + ey;
  out[e] = acc / (alpha[e * np + phase] * ws);
}

// values of a level operator at the entries of a CSR pattern (parity tests)
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

}  // namespace tmg
