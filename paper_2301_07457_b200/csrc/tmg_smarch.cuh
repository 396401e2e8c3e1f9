// Two-stage (temporally blocked) marching kernels for the coarse levels.
//
// A coarse level's operator is the exact Galerkin stencil, 19 doubles per
// node (tmg_device.cuh). Streaming it is the dominant cost of a coarse level
// (152 of ~200 bytes per node and pass), so each kernel here applies the
// stencil TWICE per HBM read of it. A CTA owns a tile of rows (one consumer
// thread per row) and marches along x; a producer warp streams every column
// (19 planes + vectors) HBM -> smem with TMA bulk copies into a ring that
// keeps the last four columns resident. Per ring entry c:
//
//   DOWN (the first half of a visit that starts from u = 0, mg_cycle
//   solvers.cpp:492-500, 2 pre-sweeps):
//     x1(c)   = omega f / D                       (sweep 1 from zero)
//     x2(c-1) = x1 + omega D^-1 (f - A x1)        (sweep 2; written out)
//     r(c-2)  = f - A x2, f_c += (1/4) P^T r      (residual + restriction)
//   UP (prolongation + 2 post-sweeps, solvers.cpp:508-513):
//     w(c)    = x2 + P u_c
//     x3(c-1) = w + omega D^-1 (f - A w)
//     x4(c-2) = x3 + omega D^-1 (f - A x3)        (written out)
//
// Intermediate columns are exchanged between rows through small shared
// buffers (one consumer barrier per stage); each thread keeps the 3x3 window
// of both stages in rotating registers, so the stencil is read from smem once
// per application and from HBM once per kernel. Bytes per node of the level:
// DOWN 152 + 16 (f) + 16 (x2) + 4 (f_c) = 188, UP 152 + 16 + 4 + 16 + 16 =
// 204, against ~904 for the unfused visit.
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda.h>
#include <cuda_runtime.h>

#include "tmg_device.cuh"
#include "tmg_march.cuh"

namespace tmg {

#ifndef TMG_SY
#define TMG_SY 96
#endif
constexpr int kSY = TMG_SY;             // consumer threads (rows) per CTA (per stage group in k_smarch2)
constexpr int kSWarps = kSY / 32;
constexpr int kSThreads = kSY + 32;     // + one producer warp
// ring depth: 4 resident columns + 2 in flight, the most that keeps two
// CTAs per SM
#ifndef TMG_SSTAGES
#define TMG_SSTAGES 6
#endif
template <bool UP>
__host__ __device__ constexpr int s_stages() { return TMG_SSTAGES; }
constexpr int kSRows = kSY + 2;         // streamed rows per column
// every coarse level runs the two-stage V(2,2) halves (measured on c1-c4:
// one-pass kernels for the small levels were 1-13 % slower per PCG
// iteration): these marching kernels above kTileMaxNodes, the shared-memory
// tiles of tmg_stile.cuh below; the one-pass kernels remain for W-cycle
// revisits and other sweep counts
constexpr long kSMinNodes = 0;

struct SMarchArgs {
  // the stencil planes as a 3-D tensor (padded row, storage column, plane):
  // one TMA box of kSRows rows x 1 column x 19 planes per ring entry
  CUtensorMap tmS;
  Grid g;   // the level
  Grid gc;  // its coarse level (restriction target / prolongation source)
  int tx;   // output columns per CTA (coarse columns for DOWN)
  const double* S;  // stencil planes, plane stride g.size
  const double2* f;
  const double2* x2;  // UP: the pre-smoothed iterate
  const double2* uc;  // UP: coarse correction
  double2* out;       // DOWN: x2, UP: x4
  double2* fc;        // DOWN: restricted rhs
  double omega;
};

// Slot layout: planes [19][kSRows] (the TMA box, dense), then f, then (UP)
// the coarse column; slots are 128-byte aligned for the tensor copy. The UP
// kernel's x2 is read by the threads directly (one column ahead) so that six
// stages still fit two CTAs per SM.
// A box must start on a 16-byte boundary (an odd FP64 start row traps as an
// illegal instruction), so it starts at the even row at or below the first
// stream row and spans two extra rows; misS skips the leading one.
constexpr int kSBoxRows = kSRows + 2;
constexpr int kSPlane = kSBoxRows * 8;
static_assert(kSPlane % 16 == 0, "TMA box rows must be a multiple of 16 bytes");
constexpr int kSO_F = kStencilPlanes * kSPlane;
constexpr int kSO_C = kSO_F + sbytes(kSRows, 16);
constexpr int kSCoarseRows = kSRows / 2 + 3;
constexpr int round128(int b) { return (b + 127) / 128 * 128; }
constexpr int kSSlotDown = round128(kSO_C);
constexpr int kSSlotUp = round128(kSO_C + sbytes(kSCoarseRows, 16));

// 2x2-block stencil application at row j of the centre column (cs = its
// slot, ls = the left column's slot, both smem), window w (cols x-1..x+1,
// rows y-1..y+1). Blocks as StencilOp::apply (tmg_device.cuh).
struct SPlanes {
  const unsigned char* base;
  int mis;
  __device__ __forceinline__ double at(int k, int j) const {
    return *reinterpret_cast<const double*>(base + k * kSPlane + mis + j * 8);
  }
};

template <class PL>
__device__ __forceinline__ void s_fwd(const PL& p, int k, int j, double2 v, double& y0, double& y1) {
  y0 = fma(p.at(k, j), v.x, y0);
  y0 = fma(p.at(k + 1, j), v.y, y0);
  y1 = fma(p.at(k + 2, j), v.x, y1);
  y1 = fma(p.at(k + 3, j), v.y, y1);
}
template <class PL>
__device__ __forceinline__ void s_bwd(const PL& p, int k, int j, double2 v, double& y0, double& y1) {
  y0 = fma(p.at(k, j), v.x, y0);
  y0 = fma(p.at(k + 2, j), v.y, y0);
  y1 = fma(p.at(k + 1, j), v.x, y1);
  y1 = fma(p.at(k + 3, j), v.y, y1);
}

// Stage B's left-column blocks held in registers: planes 7-18 of the left
// column at rows j+1 (7-10), j (11-14) and j-1 (15-18), the only ones
// s_apply reads through its L accessor
struct LCache {
  const double* v;
  __device__ __forceinline__ double at(int k, int) const { return v[k - 7]; }
};

// Three independent accumulator pairs (centre/N/SE, E/NE/S, NW/W/SW) keep
// three FMA chains in flight per thread; with two resident CTAs a single
// chain per dof left the FP64 pipe waiting on its own latency.
template <class CP, class LP>
__device__ __forceinline__ void s_apply(const CP& C, const LP& L, int j, const double2 (&l)[3],
                                        const double2 (&c)[3], const double2 (&r)[3], double2& y, double2& d) {
  const double c00 = C.at(0, j), c01 = C.at(1, j), c11 = C.at(2, j);
  double a0 = c00 * c[1].x, a1 = c01 * c[1].x;
  a0 = fma(c01, c[1].y, a0);
  a1 = fma(c11, c[1].y, a1);
  double b0 = 0.0, b1 = 0.0, e0 = 0.0, e1 = 0.0;
  s_fwd(C, 3, j, c[2], a0, a1);       // N
  s_fwd(C, 11, j, r[1], b0, b1);      // E
  s_bwd(L, 7, j + 1, l[2], e0, e1);   // NW = SE of (x-1, y+1)
  s_fwd(C, 7, j, r[0], a0, a1);       // SE
  s_fwd(C, 15, j, r[2], b0, b1);      // NE
  s_bwd(L, 11, j, l[1], e0, e1);      // W  = E of (x-1, y)
  s_bwd(C, 3, j - 1, c[0], b0, b1);   // S  = N of (x, y-1)
  s_bwd(L, 15, j - 1, l[0], e0, e1);  // SW = NE of (x-1, y-1)
  y = make_double2((a0 + b0) + e0, (a1 + b1) + e1);
  d = make_double2(c00, c11);
}

// barrier among this kernel's consumer warps only (named barrier 2)
__device__ __forceinline__ void s_consumer_sync() {
  asm volatile("bar.sync 2, %0;" ::"n"(kSY) : "memory");
}

// one damped-Jacobi update from the reciprocal diagonal (rcp_nr from
// tmg_march.cuh, one per component: coarse diagonals differ between the dofs)
__device__ __forceinline__ double2 s_jacobi_r(double2 x, double2 f, double2 y, double2 r, double omega) {
  return make_double2(fma(omega * r.x, f.x - y.x, x.x), fma(omega * r.y, f.y - y.y, x.y));
}

// one box of the 3-D stencil tensor (all 19 planes of a column's row range)
__device__ __forceinline__ void tma_planes(void* dst, const CUtensorMap* map, int row, int col, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(row), "r"(col), "r"(0), "r"(smem_u32(bar))
      : "memory");
}

// first stream row relative to y0 (R0 - 1, R0 = -1 UP / -2 DOWN)
template <bool UP>
__host__ __device__ constexpr int r0c() { return (UP ? -1 : -2) - 1; }
static_assert(kOY % 2 == 0 && (kSY - 2) % 2 == 0 && (kSY - 4) % 2 == 0, "even row tiles");

template <bool UP>
__global__ void __launch_bounds__(kSThreads) k_smarch(const __grid_constant__ SMarchArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int kSStages = s_stages<UP>();
  __shared__ uint64_t full[kSStages], empty[kSStages];
  // row-exchange columns; one buffer each suffices: between a step's reads
  // of a buffer and the next step's writes to it lies a consumer barrier
  __shared__ double2 xa[kSY + 2];  // stage-A inputs (x1 / w), written in H1
  __shared__ double2 xb[kSY + 2];  // stage-A outputs (x2 / x3), written in H2
  __shared__ double2 rb[kSY];      // DOWN: stage-B residual rows, written in H2
  constexpr int kSlot = UP ? kSSlotUp : kSSlotDown;

  const Grid& g = a.g;
  const int t = threadIdx.x;
  // rows: thread t <-> yt = y0 + R0 + t; stage A on all threads, stage B on
  // t in [1, kSY-1); stage-A inputs also on the halo rows y0+R0-1, y0+R0+kSY
  constexpr int R0 = UP ? -1 : -2;
  constexpr int kOwned = UP ? kSY - 2 : kSY - 4;  // DOWN: 46 coarse rows
  const int y0 = blockIdx.x * kOwned;
  int cf, cl, xlo, xhi;  // entries [cf, cl]; stage-B output columns [xlo, xhi]
  if (!UP) {
    const int X0 = blockIdx.y * a.tx, X1 = min(X0 + a.tx, a.gc.ncol);
    xlo = 2 * X0 - 1;
    xhi = 2 * X1 - 1;
    cf = xlo - 2;
    cl = xhi + 2;
  } else {
    xlo = blockIdx.y * a.tx;
    xhi = min(xlo + a.tx, g.ncol) - 1;
    cf = xlo - 2;
    cl = xhi + 2;
  }
  const int nent = cl - cf + 1;
  auto slot = [&](int j) { return smem_raw + static_cast<size_t>(j % kSStages) * kSlot; };
  auto in_storage = [&](int c) { return c >= -kGX && c < g.ncol + kGX; };
  // stream rows start at y0 + R0 - 1 (planes, f, x2); coarse rows at y0/2 + R0/2 - 2
  constexpr int r0 = r0c<UP>();
  static_assert(r0 == R0 - 1, "stream row offset");
  const int cr0 = (UP ? -2 : 0);

  if (t == 0) {
    for (int s = 0; s < kSStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kSWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = t; i < kSY + 2; i += kSThreads) {
    xa[i] = xb[i] = make_double2(0.0, 0.0);
    if (i < kSY) rb[i] = make_double2(0.0, 0.0);
  }
  __syncthreads();

  const uintptr_t pf = reinterpret_cast<uintptr_t>(a.f);
  // first stream row y0 + r0 in padded storage is y0 + r0 + kOY; y0 is even
  // (kOwned is even), so its parity is that of r0 + kOY
  constexpr int misS = ((r0c<UP>() + kOY) & 1) ? 8 : 0;
  const int misF = static_cast<int>((pf + static_cast<uintptr_t>(g.idx(0, y0 + r0)) * 16) & 15u);
  int misC = 0;
  if (UP) {
    misC = static_cast<int>((reinterpret_cast<uintptr_t>(a.uc) +
                             static_cast<uintptr_t>(a.gc.idx(0, (y0 >> 1) + cr0)) * 16) & 15u);
  }

  // producer warp (identified through a shuffle, so the branch and the copy
  // operands are warp-uniform and stay in uniform registers); lane 0 issues
  if (__shfl_sync(0xffffffffu, t >> 5, 0) == kSWarps) {
    const bool leader = (t == kSY);
    const uint32_t bf = (kSRows * 16 + misF + 15) / 16 * 16;
    const uint32_t bc = (kSCoarseRows * 16 + misC + 15) / 16 * 16;
    const uint32_t total = kStencilPlanes * kSPlane + bf + (UP ? bc : 0u);
    if (leader) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.tmS)) : "memory");
    for (int j = 0; j < nent; ++j) {
      const int s = j % kSStages;
      if (j >= kSStages) mbar_wait(&empty[s], ((j / kSStages) - 1) & 1);
      const int c = cf + j;
      if (!in_storage(c)) {
        if (leader) mbar_arrive(&full[s]);
        continue;
      }
      unsigned char* sl = slot(j);
      const long ri = g.idx(c, y0 + r0);
      if (leader) {
        mbar_expect_tx(&full[s], total);
        // padded row index y + kOY, storage column c + kGX (Grid::idx)
        tma_planes(sl, &a.tmS, y0 + r0 + kOY - misS / 8, c + kGX, &full[s]);
        bulk_g2s(sl + kSO_F, reinterpret_cast<const unsigned char*>(a.f + ri) - misF, bf, &full[s]);
        if (UP) {
          const long ci = a.gc.idx((c + 1) >> 1, (y0 >> 1) + cr0);
          bulk_g2s(sl + kSO_C, reinterpret_cast<const unsigned char*>(a.uc + ci) - misC, bc, &full[s]);
        }
      }
      __syncwarp();
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  // Schedule per ring entry e (column c = cf + e), two consumer barriers:
  //   H1: stage-A inputs of column c (-> xa); the stage-A column c-2 from xb
  //       into the stage-B window; DOWN: restriction of the stage-B rows of
  //       column c-4 (rb)
  //   --- barrier ---
  //   H2: stage A at column c-1 (-> xb) and stage B at column c-3 (-> out /
  //       rb): independent, so their FMA chains interleave
  //   --- barrier ---
  // Stage B reads the transposed blocks of its left column from registers
  // (cached when that column was its centre), so the ring still holds four
  // columns (c-3 .. c). Nodes outside the level are masked by selects, not
  // branches: the stencil is zero there (S is zero-filled and only level
  // nodes are assembled), so the unmasked arithmetic is finite and discarded.
  const int yt = y0 + R0 + t;
  const int lane = t & 31;
  const int j = t + 1;  // stream row index of yt (streams start at yt - 1 for t = 0)
  // halo stream row of the stage-A inputs this thread also computes (only
  // threads 0 and kSY-1 store it; the rest compute it to stay convergent)
  const int jh = (t == 0) ? 0 : kSY + 1;
  const int yh = y0 + r0 + jh;
  auto row_in = [&](int y) { return y >= 0 && y <= g.ny; };
  auto col_in = [&](int x) { return g.x0 + x >= 0 && g.x0 + x <= g.nx; };
  const bool rin = row_in(yt), hin = row_in(yh);
  const bool tB = t >= 1 && t < kSY - 1;  // rows of stage B
  auto fat = [&](const unsigned char* s, int jj) {
    return *reinterpret_cast<const double2*>(s + kSO_F + misF + jj * 16);
  };
  const double2 z2 = make_double2(0.0, 0.0);
  auto sel = [](bool p, double2 v) { return p ? v : make_double2(0.0, 0.0); };
  // DOWN stage-A input: x1 = omega f / D (sweep 1 from zero); rc = 1/D
  auto a_in_down = [&](const unsigned char* s, int jj, double2& rc) {
    const SPlanes P{s, misS};
    const double2 f = fat(s, jj);
    rc = make_double2(rcp_nr(P.at(0, jj)), rcp_nr(P.at(2, jj)));
    return make_double2(a.omega * f.x * rc.x, a.omega * f.y * rc.y);
  };
  // UP stage-A input: w = x2 + P u_c (bilinear, grid.cpp:20-46); coarse
  // column ceil(c/2) in s, floor(c/2) in ps for odd columns
  auto a_in_up = [&](const unsigned char* s, const unsigned char* ps, bool odd_col, int jj, double2 xv) {
    const int y = y0 + r0 + jj;
    const int gy = y - 2 * ((y0 >> 1) + cr0);  // fine row relative to the coarse stream start
    auto crow = [&](const unsigned char* sl, int k) {
      return *reinterpret_cast<const double2*>(sl + kSO_C + misC + k * 16);
    };
    auto colv = [&](const unsigned char* sl) {
      const double2 p = crow(sl, gy >> 1), q = crow(sl, (gy >> 1) + 1);
      return (gy & 1) ? make_double2(0.5 * p.x + 0.5 * q.x, 0.5 * p.y + 0.5 * q.y) : p;
    };
    double2 pu = colv(s);
    if (odd_col) {
      const double2 q = colv(ps);
      pu = make_double2(0.5 * q.x + 0.5 * pu.x, 0.5 * q.y + 0.5 * pu.y);
    }
    return make_double2(xv.x + pu.x, xv.y + pu.y);
  };

  // UP: x2 of the own row and of the halo row for the next column, loaded
  // while the current one is processed
  // (the column three entries further is prefetched into L2 at the same
  // time: one step of lead alone left the warps waiting on HBM latency)
  double2 x2o = z2, x2h = z2;
  auto fetch_x2 = [&](int c) {
    x2o = a.x2[g.idx(c, yt)];
    x2h = a.x2[g.idx(c, yh)];
    if (c + 3 <= cl) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.x2 + g.idx(c + 3, yt)));
  };
  if (UP) {
    for (int k = 1; k < 3; ++k) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.x2 + g.idx(cf + k, yt)));
    fetch_x2(cf);
  }

  // rotating windows: A over stage-A inputs (columns c-2, c-1, c), B over
  // stage-A outputs (c-4, c-3, c-2). The entry loop is unrolled by 3 so the
  // windows rotate by compile-time index: at phase P the window columns are
  // w[P], w[P+1], w[P+2] (mod 3), w[P+2] being the column read this step.
  double2 wa[3][3], wb[3][3];
  double2 rd[3];  // DOWN: 1/D of the own row at the stage-A window columns
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    rd[p] = z2;
#pragma unroll
    for (int q = 0; q < 3; ++q) wa[p][q] = wb[p][q] = z2;
  }
  double lc[12];  // stage B: planes 7-10 at j+1, 11-14 at j, 15-18 at j-1 of its left column
#pragma unroll
  for (int k = 0; k < 12; ++k) lc[k] = 0.0;
  double2 acc = z2, bres = z2;  // DOWN: restriction accumulator, own stage-B residual

  // ring position of entry e (slot index, mbarrier phase) and the slots of
  // entries e-1 .. e-3, advanced incrementally
  int si = 0;
  uint32_t ph = 0;
  const unsigned char* sp1 = nullptr;
  const unsigned char* sp2 = nullptr;
  const unsigned char* sp3 = nullptr;
  int srel = kSStages - 3;  // slot of entry e-3 (mod kSStages)

  auto step = [&](auto phase, int e) {
    constexpr int P = decltype(phase)::value;
    constexpr int IL = P, IC = (P + 1) % 3, IR = (P + 2) % 3;
    const int c = cf + e;
    const bool enter = e < nent;
    const unsigned char* s0 = smem_raw + static_cast<size_t>(si) * kSlot;
    // ---------------------------------------------------------------- H1
    if (enter) {
      mbar_wait(&full[si], ph);
      const bool ci = col_in(c);
      double2 v, vh;
      if (!UP) {
        double2 rc, rch;
        v = a_in_down(s0, j, rc);
        vh = a_in_down(s0, jh, rch);
        rd[IR] = rc;
      } else {
        const bool odd = (g.x0 + c) & 1;
        const double2 xo = x2o, xh = x2h;
        if (e + 1 < nent) fetch_x2(c + 1);
        v = a_in_up(s0, sp1, odd, j, xo);
        vh = a_in_up(s0, sp1, odd, jh, xh);
      }
      xa[t + 1] = sel(ci && rin, v);
      if (t == 0) xa[0] = sel(ci && hin, vh);
      if (t == kSY - 1) xa[kSY + 1] = sel(ci && hin, vh);
    }
    // stage-B window column c-2 (stage A ran there last step)
#pragma unroll
    for (int q = 0; q < 3; ++q) wb[IR][q] = tB ? xb[t + q] : z2;
    if (!UP && e >= 4) {
      // restriction of column x = c-4: rows (1/2, 1, 1/2) around even fine
      // rows, columns the same
      const int x = c - 4;
      if (x >= xlo && x <= xhi) {
        const double2 rm = rb[t > 0 ? t - 1 : 0], rp = rb[t < kSY - 1 ? t + 1 : kSY - 1];
        const double2 rs = make_double2(fma(0.5, rm.x + rp.x, bres.x), fma(0.5, rm.y + rp.y, bres.y));
        if (((g.x0 + x) & 1) == 0) {
          acc.x += rs.x;
          acc.y += rs.y;
        } else {
          if (x != xlo) {
            acc.x = fma(0.5, rs.x, acc.x);
            acc.y = fma(0.5, rs.y, acc.y);
            const int X = (x - 1) >> 1, Y = yt >> 1;
            if ((yt & 1) == 0 && t >= 2 && t < kSY - 2 && yt >= y0 && yt < y0 + kOwned && Y <= a.gc.ny)
              a.fc[a.gc.idx(X, Y)] = make_double2(0.25 * acc.x, 0.25 * acc.y);
          }
          acc = make_double2(0.5 * rs.x, 0.5 * rs.y);
        }
      }
    }
    s_consumer_sync();
    // ---------------------------------------------------------------- H2
    if (enter) {
#pragma unroll
      for (int q = 0; q < 3; ++q) wa[IR][q] = xa[t + q];
    }
    const bool runA = enter && e >= 2, runB = e >= 3 && e <= nent;
    double2 va = z2, vb = z2;
    double2 ya, da, yb, db;
    if (runA) s_apply(SPlanes{sp1, misS}, SPlanes{sp2, misS}, j, wa[IL], wa[IC], wa[IR], ya, da);
    if (runB) s_apply(SPlanes{sp3, misS}, LCache{lc}, j, wb[IL], wb[IC], wb[IR], yb, db);
    if (runA) {
      const int x = c - 1;
      const double2 f = fat(sp1, j);
      const double2 r = UP ? make_double2(rcp_nr(da.x), rcp_nr(da.y)) : rd[IC];
      va = sel(col_in(x) && rin, s_jacobi_r(wa[IC][1], f, ya, r, a.omega));
      // x2 of the nodes this CTA owns: rows [y0, y0+kOwned), fine columns
      // [2 X0, 2 X1) of its coarse columns
      if (!UP && t >= 2 && t < 2 + kOwned && x > xlo && x <= xhi && x < g.ncol && yt <= g.ny)
        a.out[g.idx(x, yt)] = va;
      xb[t + 1] = va;
    }
    if (runB) {
      const int x = c - 3;
      const SPlanes C{sp3, misS};
      const double2 f = fat(sp3, j);
      const bool ok = tB && col_in(x) && rin;
      if (UP) {
        vb = sel(ok, s_jacobi_r(wb[IC][1], f, yb, make_double2(rcp_nr(db.x), rcp_nr(db.y)), a.omega));
        if (tB && x >= xlo && x <= xhi && yt <= g.ny) a.out[g.idx(x, yt)] = vb;
      } else {
        bres = sel(ok, make_double2(f.x - yb.x, f.y - yb.y));
        rb[t] = bres;
      }
      // the transposed blocks of column x for stage B at x+1
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        lc[k] = C.at(7 + k, j + 1);
        lc[4 + k] = C.at(11 + k, j);
        lc[8 + k] = C.at(15 + k, j - 1);
      }
      // column c-3 is no longer needed
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[srel]);
    }
    s_consumer_sync();
    // advance the ring position
    sp3 = sp2;
    sp2 = sp1;
    sp1 = s0;
    srel = (srel + 1 == kSStages) ? 0 : srel + 1;
    if (++si == kSStages) {
      si = 0;
      ph ^= 1u;
    }
  };

  // entries 0 .. nent-1 plus drain steps: stage B trails the last entry by
  // one step, the DOWN restriction by two
  const int nsteps = nent + (UP ? 1 : 2);
  int e = 0;
  for (; e + 2 < nsteps; e += 3) {
    step(std::integral_constant<int, 0>{}, e);
    step(std::integral_constant<int, 1>{}, e + 1);
    step(std::integral_constant<int, 2>{}, e + 2);
  }
  if (e < nsteps) step(std::integral_constant<int, 0>{}, e);
  if (e + 1 < nsteps) step(std::integral_constant<int, 1>{}, e + 1);
}

}  // namespace tmg
