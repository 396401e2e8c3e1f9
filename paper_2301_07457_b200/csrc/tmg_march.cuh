// Column-marching engine for the matrix-free fine level.
//
// A CTA owns a tile of rows y (one consumer thread per row; y is the
// contiguous direction of the reference numbering, grid.hpp:19) and marches
// over node columns x. Column data is streamed HBM -> shared memory by TMA
// bulk copies (cp.async.bulk ... mbarrier::complete_tx) into a kStages-deep
// ring. Warp-specialised: one producer warp issues the copies, kTY/32 consumer
// warps compute; full/empty mbarriers hand slots back and forth, so no
// CTA-wide barrier sits on the per-column critical path and every byte of the
// streamed fields is read from HBM once.
//
// Each consumer keeps the 3x3 neighbourhood of its node in registers in three
// rotating column slots (period 3, the loop is unrolled by 3 so the window
// shifts without register moves). A stage decides which streams a ring entry
// carries, how a column is turned into window values (load) and what a node
// computes from its window (run). The fused stages cover one V-cycle visit of
// the finest level (mg_cycle, solvers.cpp:483-514) in four passes and the PCG
// direction update + K p + p.Kp in one (solvers.cpp:367-382):
//
//   StSweep01       two damped-Jacobi sweeps from u = 0; the first sweep
//                   (omega f / D) is evaluated on the fly for the neighbours
//   StResidRestrict r = f - A u and f_c = (1/4) P^T r (grid.cpp:122-142) with
//                   one shared-memory row exchange per column
//   StProlongSweep  u + P u_c (grid.cpp:98-120) on the fly, then one sweep
//   StSweep<DOT>    one sweep, optionally with z.r for PCG (solvers.cpp:361)
//   StPupd          p = z + beta p on the fly, Ap = A p, p.Ap
//   StApply/StResidual  the plain operator and residual
//
// Element moduli: ring entry c carries element column c (rows around the
// tile); node column c uses element columns c-1 (previous slot) and c.
// Rows that touch a fixed dof anywhere in their 3x3 neighbourhood take a
// (rare, warp-local) masked path; every other node runs the plain 64-DFMA
// element gather with the 8 Ke constants held in uniform registers.
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "tmg_device.cuh"
#include "tmg_kernels.cuh"

namespace tmg {

constexpr int kTY = 128;                 // consumer threads (rows) per CTA
constexpr int kConsumerWarps = kTY / 32;
constexpr int kMarchThreads = kTY + 32;  // + one producer warp
constexpr int kStages = 6;
// ring depth of the fused PCG-update pass (StSweep01U): its slots carry six
// streams, so six stages left room for three CTAs per SM; four stages give
// the register limit's four (same-box A/B, TMG_UPD_STAGES builds: c4 6.37 ->
// 6.21 ms per PCG iteration, c3 0.230 -> 0.224 ms, c1 unchanged; 5 stages in
// between)
#ifndef TMG_UPD_STAGES
#define TMG_UPD_STAGES 4
#endif
constexpr long kSlackNodes = 1024;  // every field is over-allocated by this

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// The suspend-time hint parks a waiting warp until the phase completes
// instead of the short default limit: without it the producer warp spins on
// its empty slots and takes issue slots from the consumer warps it shares a
// scheduler with (ncu showed ~20% of a fine stage's instructions there).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680u)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// barrier among the consumer warps only (named barrier 1)
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kTY) : "memory");
}

// ---------------------------------------------------------------- streams --

struct MarchArgs {
  Grid g;   // fine grid
  Grid gc;  // next coarser grid (prolongation / restriction)
  int tx;   // output columns per CTA
  const double2* u;   // primary window field (halo rows)
  const double2* u2;  // second window field (StPupd: old p)
  const double* E;
  const uint8_t* M;
  const double2* f;   // own-row field
  const double2* uc;  // coarse field (StProlongSweep)
  double2* out0;
  double2* out1;
  double2* out2;      // StSweep01U: x (read and written, own rows)
  double omega;
  double* partials;
  unsigned* ticket;   // null: leave the partials for the multi-rank all-reduce
  RedTiles rt;        // global tile geometry of the partials (reducing stages)
  RedOp rop;
  PcgState* st;
  HostMirror* hm;
  double* red_out;
};

// One bulk copy per ring entry: rows [y0 + r0, y0 + r0 + n) of node column c
// (fine streams) or coarse column ceil(c/2), rows [y0/2 + r0, ...) (coarse).
struct StreamDesc {
  const unsigned char* base;
  int esize;
  int r0;
  int n;
  bool coarse;
};

__host__ __device__ constexpr int sbytes(int n, int esize) { return ((n * esize + 16) + 15) / 16 * 16; }

__device__ __forceinline__ long stream_row_index(const MarchArgs& a, const StreamDesc& d, int c, int y0) {
  if (d.coarse) return a.gc.idx((c + 1) >> 1, (y0 >> 1) + d.r0);
  return a.g.idx(c, y0 + d.r0);
}
// byte misalignment of the first row; identical for every column of a CTA
// because pitches are multiples of 16 nodes
__device__ __forceinline__ int stream_mis(const MarchArgs& a, const StreamDesc& d, int y0) {
  const uintptr_t p = reinterpret_cast<uintptr_t>(d.base) +
                      static_cast<uintptr_t>(stream_row_index(a, d, 1, y0) * d.esize);
  return static_cast<int>(p & 15u);
}

// CTA order of a pass. The hardware starts CTAs in increasing linear block
// index (x fastest), so the columns a pass finishes with are the ones still
// in L2 when the next pass starts. Stages that declare kReverse take their
// tiles in the opposite order, so that a pass begins on the strips its
// predecessor touched last: the fused update F, the residual + restriction
// R | the prolongation + sweep R, the second post-sweep F, the direction
// update R, and the next iteration's fused update F again. The logical tile
// (and with it every reduction partial's index) does not change.
#ifndef TMG_CLAMP_ROWS
#define TMG_CLAMP_ROWS 1
#endif
#ifndef TMG_SERPENTINE
#define TMG_SERPENTINE 1
#endif
template <class Stage, class = void>
struct ReverseOf {
  static constexpr bool value = false;
};
template <class Stage>
struct ReverseOf<Stage, std::void_t<decltype(Stage::kReverse)>> {
  static constexpr bool value = Stage::kReverse && TMG_SERPENTINE;
};
template <class Stage>
__device__ __forceinline__ int tile_x() {
  return ReverseOf<Stage>::value ? static_cast<int>(gridDim.x - 1 - blockIdx.x) : static_cast<int>(blockIdx.x);
}
template <class Stage>
__device__ __forceinline__ int tile_y() {
  return ReverseOf<Stage>::value ? static_cast<int>(gridDim.y - 1 - blockIdx.y) : static_cast<int>(blockIdx.y);
}

// ------------------------------------------------------------ node helpers --

__device__ __forceinline__ uint32_t fixbits(uint32_t byte) {
  return ((byte & 0x0Fu) ? 1u : 0u) | ((byte & 0xF0u) ? 2u : 0u);
}
__device__ __forceinline__ double2 masked2(double2 v, uint32_t byte) {
  if (byte & 0x0Fu) v.x = 0.0;
  if (byte & 0xF0u) v.y = 0.0;
  return v;
}

// rows (2A, 2A+1) of e * Ke times the element's corner values q0..q3; EX:
// the exact quadrature Ke (the system's operator), else the 8-value form
// (the V-cycle's smoothing passes; tmg_device.cuh)
#define TMG_KE(r, b) (EX ? c_kex_at((r), (b)) : c_ke_at((r), (b)))
template <int A, bool EX>
__device__ __forceinline__ void erows(double e, const double2& q0, const double2& q1, const double2& q2,
                                      const double2& q3, double& y0, double& y1) {
  double s0 = TMG_KE(2 * A, 0) * q0.x;
  s0 = fma(TMG_KE(2 * A, 1), q0.y, s0);
  s0 = fma(TMG_KE(2 * A, 2), q1.x, s0);
  s0 = fma(TMG_KE(2 * A, 3), q1.y, s0);
  s0 = fma(TMG_KE(2 * A, 4), q2.x, s0);
  s0 = fma(TMG_KE(2 * A, 5), q2.y, s0);
  s0 = fma(TMG_KE(2 * A, 6), q3.x, s0);
  s0 = fma(TMG_KE(2 * A, 7), q3.y, s0);
  double s1 = TMG_KE(2 * A + 1, 0) * q0.x;
  s1 = fma(TMG_KE(2 * A + 1, 1), q0.y, s1);
  s1 = fma(TMG_KE(2 * A + 1, 2), q1.x, s1);
  s1 = fma(TMG_KE(2 * A + 1, 3), q1.y, s1);
  s1 = fma(TMG_KE(2 * A + 1, 4), q2.x, s1);
  s1 = fma(TMG_KE(2 * A + 1, 5), q2.y, s1);
  s1 = fma(TMG_KE(2 * A + 1, 6), q3.x, s1);
  s1 = fma(TMG_KE(2 * A + 1, 7), q3.y, s1);
  y0 = fma(e, s0, y0);
  y1 = fma(e, s1, y1);
}

// K w at the centre of the 3x3 window (l/c/r = columns x-1/x/x+1, index
// 0/1/2 = rows y-1/y/y+1). Elements (x-1,y-1) eA, (x,y-1) eB, (x,y) eC,
// (x-1,y) eD hold the node at their corners 2, 3, 0, 1 (fem.cpp:83-86).
template <bool EX>
__device__ __forceinline__ void gather9(const double2 (&l)[3], const double2 (&c)[3], const double2 (&r)[3],
                                        double eA, double eB, double eC, double eD, double& y0,
                                        double& y1) {
  y0 = 0.0;
  y1 = 0.0;
  erows<2, EX>(eA, l[0], c[0], c[1], l[1], y0, y1);
  erows<3, EX>(eB, c[0], r[0], r[1], c[1], y0, y1);
  erows<0, EX>(eC, c[1], r[1], r[2], c[2], y0, y1);
  erows<1, EX>(eD, l[1], c[1], c[2], l[2], y0, y1);
}

// (A w)_i and diag(A)_i of Z K Z + I_fixed (fem.cpp:89-106) for the window.
// mL/mC/mR: the three mask bytes (rows y-1, y, y+1) of each column.
template <bool EX = false>
__device__ __forceinline__ void fine_apply(const double2 (&l)[3], const double2 (&c)[3], const double2 (&r)[3],
                                           uint32_t mL, uint32_t mC, uint32_t mR, double eA, double eB,
                                           double eC, double eD, double2& y, double2& d) {
  double y0, y1;
  if ((mL | mC | mR) == 0u) {
    gather9<EX>(l, c, r, eA, eB, eC, eD, y0, y1);
  } else {
    double2 ml[3], mc[3], mr[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      ml[q] = masked2(l[q], (mL >> (8 * q)) & 0xFFu);
      mc[q] = masked2(c[q], (mC >> (8 * q)) & 0xFFu);
      mr[q] = masked2(r[q], (mR >> (8 * q)) & 0xFFu);
    }
    gather9<EX>(ml, mc, mr, eA, eB, eC, eD, y0, y1);
  }
  const double2 kd = ke_diag(eA, eB, eC, eD);  // the reference's diagonal, bitwise
  double d0 = kd.x, d1 = kd.y;
  const uint32_t own = (mC >> 8) & 0xFFu;
  if (own) {
    const int k0 = own & 15, k1 = (own >> 4) & 15;
    if (k0) {
      y0 = k0 * c[1].x;
      d0 = k0;
    }
    if (k1) {
      y1 = k1 * c[1].y;
      d1 = k1;
    }
  }
  y = make_double2(y0, y1);
  d = make_double2(d0, d1);
}

// diagonal of a node from its four element moduli and own mask byte
__device__ __forceinline__ double2 fine_diag(double eA, double eB, double eC, double eD, uint32_t own) {
  const double2 kd = ke_diag(eA, eB, eC, eD);
  double d0 = kd.x, d1 = kd.y;
  if (own) {
    const int k0 = own & 15, k1 = (own >> 4) & 15;
    if (k0) d0 = k0;
    if (k1) d1 = k1;
  }
  return make_double2(d0, d1);
}

// 1/d from the MUFU seed and two Newton steps (error well below 1 ulp of
// the final product; no subroutine call like IEEE division)
__device__ __forceinline__ double rcp_nr(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

// x + omega D^-1 (f - y) (jacobi_sweep, solvers.cpp:35): one reciprocal per
// node when both dofs share the diagonal
__device__ __forceinline__ double2 jacobi_update(double2 x, double2 f, double2 y, double2 d, double omega) {
  const double s0 = omega * rcp_nr(d.x);
  const double s1 = (d.y == d.x) ? s0 : omega * rcp_nr(d.y);
  return make_double2(fma(s0, f.x - y.x, x.x), fma(s1, f.y - y.y, x.y));
}

// smem readers for slot data
template <class T>
__device__ __forceinline__ const T& sat(const unsigned char* slot, int off, int mis, int j) {
  return *reinterpret_cast<const T*>(slot + off + mis + j * static_cast<int>(sizeof(T)));
}
__device__ __forceinline__ uint32_t mask3(const unsigned char* slot, int off, int mis, int j) {
  const uint8_t* p = slot + off + mis + j;
  return static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8) | (static_cast<uint32_t>(p[2]) << 16);
}

// ------------------------------------------------------------------ stages --
// Thread t handles row yt = y0 + kRow0 + t. A column slot `Col` holds only
// the window data of one node column (rows yt-1 .. yt+1 of the window field,
// the element moduli of element column c at rows yt-1, yt and three mask
// bytes). Centre-only data (f, ...) is read from the centre column's ring slot
// in run(); the engine keeps that slot (and the previous one, for stages
// whose load() needs it) until the centre is done.

struct Col {
  double2 u[3];
  double e1, e2;  // element column c, rows yt-1, yt
  uint32_t m3;    // mask bytes of rows yt-1, yt, yt+1
  double2 w;      // StSweep01: omega / D of the own row (reused by the 2nd sweep)
};

// window field u (rows -1..TY), E (rows -1..TY), M (rows -1..TY)
#define TMG_WINDOW_STREAMS(ufield)                                                    \
  if (k == 0) return {reinterpret_cast<const unsigned char*>(ufield), 16, kRow0 - 1, kTY + 2, false}; \
  if (k == 1) return {reinterpret_cast<const unsigned char*>(a.E), 8, kRow0 - 1, kTY + 2, false};     \
  if (k == 2) return {reinterpret_cast<const unsigned char*>(a.M), 1, kRow0 - 1, kTY + 2, false};

__device__ __forceinline__ void load_window(const unsigned char* s, int ou, int oe, int om, const int* mis,
                                            int t, Col& c) {
  c.u[0] = sat<double2>(s, ou, mis[0], t);
  c.u[1] = sat<double2>(s, ou, mis[0], t + 1);
  c.u[2] = sat<double2>(s, ou, mis[0], t + 2);
  c.e1 = sat<double>(s, oe, mis[1], t);
  c.e2 = sat<double>(s, oe, mis[1], t + 1);
  c.m3 = mask3(s, om, mis[2], t);
}

#ifndef TMG_EXACT_SMOOTHER
#define TMG_EXACT_SMOOTHER 0
#endif
template <bool EX = TMG_EXACT_SMOOTHER>
__device__ __forceinline__ void window_apply(const Col& L, const Col& C, const Col& R, double2& y, double2& d) {
  fine_apply<EX>(L.u, C.u, R.u, L.m3, C.m3, R.m3, L.e1, C.e1, C.e2, L.e2, y, d);
}

// y = A u (K1); optional partial u.Au
template <bool DOT>
struct StApply {
  static constexpr int NS = 3, kRow0 = 0, kOwned = kTY, kLead = 0;
  static constexpr int O_U = 0, O_E = O_U + sbytes(kTY + 2, 16), O_M = O_E + sbytes(kTY + 2, 8);
  static constexpr int kSlot = O_M + sbytes(kTY + 2, 1);
  __device__ static StreamDesc stream(const MarchArgs& a, int k) {
    TMG_WINDOW_STREAMS(a.u)
    return {};
  }
  __device__ static int off(int k) { return k == 0 ? O_U : (k == 1 ? O_E : O_M); }
  __device__ static void load(const MarchArgs&, const unsigned char* s, const unsigned char*, const int* mis,
                              int t, int, Col& c) {
    load_window(s, O_U, O_E, O_M, mis, t, c);
  }
  __device__ static void run(const MarchArgs& a, const Col& L, const Col& C, const Col& R, const unsigned char*,
                             const int*, int x, int yt, int, bool live, double& part, double2&) {
    if (!live) return;
    double2 y, d;
    window_apply<true>(L, C, R, y, d);
    a.out0[a.g.idx(x, yt)] = y;
    if (DOT) part = fma(C.u[1].x, y.x, fma(C.u[1].y, y.y, part));
  }
};

// window streams + own-row f
template <int ROW0>
struct WithF {
  static constexpr int NS = 4, kRow0 = ROW0;
  static constexpr int O_U = 0, O_E = O_U + sbytes(kTY + 2, 16), O_M = O_E + sbytes(kTY + 2, 8);
  static constexpr int O_F = O_M + sbytes(kTY + 2, 1);
  static constexpr int kSlot = O_F + sbytes(kTY, 16);
  __device__ static StreamDesc stream(const MarchArgs& a, int k) {
    TMG_WINDOW_STREAMS(a.u)
    return {reinterpret_cast<const unsigned char*>(a.f), 16, kRow0, kTY, false};
  }
  __device__ static int off(int k) { return k == 0 ? O_U : (k == 1 ? O_E : (k == 2 ? O_M : O_F)); }
  __device__ static void load(const MarchArgs&, const unsigned char* s, const unsigned char*, const int* mis,
                              int t, int, Col& c) {
    load_window(s, O_U, O_E, O_M, mis, t, c);
  }
  __device__ static double2 fc(const unsigned char* s, const int* mis, int t) {
    return sat<double2>(s, O_F, mis[3], t);
  }
};

// x_out = u + omega D^-1 (f - A u) (jacobi_sweep, solvers.cpp:30-37); DOT adds
// x_out . f (z.r of pcg_solve, solvers.cpp:361, when f is the PCG residual)
template <bool DOT>
struct StSweep : WithF<0> {
  static constexpr int kOwned = kTY, kLead = 0;
  __device__ static void run(const MarchArgs& a, const Col& L, const Col& C, const Col& R,
                             const unsigned char* cs, const int* mis, int x, int yt, int t, bool live,
                             double& part, double2&) {
    if (!live) return;
    double2 y, d;
    window_apply(L, C, R, y, d);
    const double2 f = fc(cs, mis, t);
    const double2 z = jacobi_update(C.u[1], f, y, d, a.omega);
    a.out0[a.g.idx(x, yt)] = z;
    if (DOT) part = fma(z.x, f.x, fma(z.y, f.y, part));
  }
};

// r = f - A u (solvers.cpp:498-499)
struct StResidual : WithF<0> {
  static constexpr int kOwned = kTY, kLead = 0;
  __device__ static void run(const MarchArgs& a, const Col& L, const Col& C, const Col& R,
                             const unsigned char* cs, const int* mis, int x, int yt, int t, bool live, double&,
                             double2&) {
    if (!live) return;
    double2 y, d;
    window_apply(L, C, R, y, d);
    const double2 f = fc(cs, mis, t);
    a.out0[a.g.idx(x, yt)] = make_double2(f.x - y.x, f.y - y.y);
  }
};

// Two sweeps from u = 0. The first, x1 = omega f / D, is formed at load time
// for the thread's own row (one division per node) and shared with the
// neighbouring rows through a shared-memory column exchange; then
// x2 = x1 + omega D^-1 (f - A x1). The streamed window field is f.
//
// UPD additionally finishes the previous PCG iteration first (pcg_solve,
// solvers.cpp:383-386): the window field is r_old with A p_old beside it,
// f = r = r_old - alpha A p is formed wherever f is read, and the own rows
// write r (out1) and x += alpha p (x in out2, p streamed from uc) and
// reduce r.r. This moves the x/r update off its own 96-byte-per-node pass
// into the (compute-bound) first smoothing pass.
template <bool UPD>
struct StSweep01T {
  static constexpr int NS = UPD ? 6 : 3, kRow0 = 0, kOwned = kTY, kLead = 1;
  static constexpr int kRing = UPD ? TMG_UPD_STAGES : kStages;
  static constexpr int O_F = 0, O_E = O_F + sbytes(kTY + 2, 16), O_M = O_E + sbytes(kTY + 4, 8);
  static constexpr int O_A = O_M + sbytes(kTY + 2, 1);  // UPD: A p_old, window rows
  static constexpr int O_X = O_A + sbytes(kTY + 2, 16);  // UPD: x, own rows
  static constexpr int O_P = O_X + sbytes(kTY, 16);      // UPD: p_old, own rows
  static constexpr int kSlot = UPD ? O_P + sbytes(kTY, 16) : O_A;
  __device__ static StreamDesc stream(const MarchArgs& a, int k) {
    if (k == 0) return {reinterpret_cast<const unsigned char*>(a.f), 16, -1, kTY + 2, false};
    if (k == 1) return {reinterpret_cast<const unsigned char*>(a.E), 8, -2, kTY + 4, false};
    if (k == 2) return {reinterpret_cast<const unsigned char*>(a.M), 1, -1, kTY + 2, false};
    if (k == 3) return {reinterpret_cast<const unsigned char*>(a.u2), 16, -1, kTY + 2, false};
    if (k == 4) return {reinterpret_cast<const unsigned char*>(a.out2), 16, 0, kTY, false};
    return {reinterpret_cast<const unsigned char*>(a.uc), 16, 0, kTY, false};
  }
  __device__ static int off(int k) {
    return k == 0 ? O_F : (k == 1 ? O_E : (k == 2 ? O_M : (k == 3 ? O_A : (k == 4 ? O_X : O_P))));
  }
  // f at stream row index j (row y0 - 1 + j); UPD: r_old - alpha A p_old
  // (the same fma as k_update_xr, so r is bit-identical to the unfused path)
  __device__ static double2 f_at(const unsigned char* s, const int* mis, int j, double alpha) {
    const double2 r = sat<double2>(s, O_F, mis[0], j);
    if (!UPD) return r;
    const double2 q = sat<double2>(s, O_A, mis[3], j);
    return make_double2(fma(-alpha, q.x, r.x), fma(-alpha, q.y, r.y));
  }
  // x1 at stream row index j of column c; *w = omega / D
  __device__ static double2 x1_at(const MarchArgs& a, const unsigned char* s, const unsigned char* ps,
                                  const int* mis, int j, double alpha, double2* w) {
    // node rows r = y0-1+j: elements (c-1, r-1), (c, r-1), (c, r), (c-1, r)
    // sit at E-stream indices j and j+1 (stream starts at row y0-2)
    const double eA = ps ? sat<double>(ps, O_E, mis[1], j) : 0.0;
    const double eD = ps ? sat<double>(ps, O_E, mis[1], j + 1) : 0.0;
    const double eB = sat<double>(s, O_E, mis[1], j), eC = sat<double>(s, O_E, mis[1], j + 1);
    const uint32_t m = *(s + O_M + mis[2] + j);
    const double2 d = fine_diag(eA, eB, eC, eD, m);
    // ghost nodes have no elements: D = 0 and x1 = 0
    if (d.x == 0.0) {
      if (w) *w = make_double2(0.0, 0.0);
      return make_double2(0.0, 0.0);
    }
    const double2 f = f_at(s, mis, j, alpha);
    const double s0 = a.omega * rcp_nr(d.x);
    const double s1 = (d.y == d.x) ? s0 : a.omega * rcp_nr(d.y);
    if (w) *w = make_double2(s0, s1);
    return make_double2(s0 * f.x, s1 * f.y);
  }
  // Own row x1 per thread, shared with the neighbouring rows through a
  // double-buffered smem column (one consumer barrier per column); the first
  // and last thread also evaluate the halo rows of the tile.
  __device__ static void load(const MarchArgs& a, const unsigned char* s, const unsigned char* ps,
                              const int* mis, int t, int c, Col& col) {
    __shared__ double2 xb[2][kTY + 2];
    const double alpha = UPD ? a.st->alpha : 0.0;
    double2* buf = xb[c & 1];
    buf[t + 1] = x1_at(a, s, ps, mis, t + 1, alpha, &col.w);
    if (t == 0) buf[0] = x1_at(a, s, ps, mis, 0, alpha, nullptr);
    if (t == kTY - 1) buf[kTY + 1] = x1_at(a, s, ps, mis, kTY + 1, alpha, nullptr);
    consumer_sync();
    col.u[0] = buf[t];
    col.u[1] = buf[t + 1];
    col.u[2] = buf[t + 2];
    col.e1 = sat<double>(s, O_E, mis[1], t + 1);
    col.e2 = sat<double>(s, O_E, mis[1], t + 2);
    col.m3 = mask3(s, O_M, mis[2], t);
  }
  __device__ static void run(const MarchArgs& a, const Col& L, const Col& C, const Col& R,
                             const unsigned char* cs, const int* mis, int x, int yt, int t, bool live, double& part,
                             double2&) {
    if (!live) return;
    double2 y, d;
    window_apply(L, C, R, y, d);
    const double alpha = UPD ? a.st->alpha : 0.0;
    const double2 f = f_at(cs, mis, t + 1, alpha);
    const double2 x1 = C.u[1];
    const long i = a.g.idx(x, yt);
    a.out0[i] = make_double2(fma(C.w.x, f.x - y.x, x1.x), fma(C.w.y, f.y - y.y, x1.y));
    if (UPD) {
      a.out1[i] = f;
      const double2 xo = sat<double2>(cs, O_X, mis[4], t), pp = sat<double2>(cs, O_P, mis[5], t);
      a.out2[i] = make_double2(fma(alpha, pp.x, xo.x), fma(alpha, pp.y, xo.y));
      part = fma(f.x, f.x, part);
      part = fma(f.y, f.y, part);
    }
  }
};
using StSweep01 = StSweep01T<false>;
using StSweep01U = StSweep01T<true>;

// f_c = (1/4) P^T (f - A u) in one pass. Thread t owns fine row
// yt = y0 - 1 + t so the 63 coarse rows Y = y0/2 .. y0/2 + 62 see their three
// fine rows 2Y-1 .. 2Y+1 inside the tile; a CTA owns coarse columns
// [X0, X0 + tx) and marches fine columns 2 X0 - 1 .. 2 (X0 + tx) - 1.
struct StResidRestrict : WithF<-1> {
  static constexpr int kOwned = kTY - 2, kLead = 0;
  static constexpr bool kReverse = true;
  // acc: this row's residual summed over the fine columns of the coarse
  // column being accumulated, with weights (1/2, 1, 1/2) in x; the rows are
  // combined ((1/2, 1, 1/2) in y) once per coarse column through smem
  __device__ static void run(const MarchArgs& a, const Col& L, const Col& C, const Col& R,
                             const unsigned char* cs, const int* mis, int x, int yt, int t, bool live, double&,
                             double2& acc) {
    __shared__ double2 rbuf[2][kTY];
    double2 r = make_double2(0.0, 0.0);
    if (a.g.x0 + x >= 0 && a.g.x0 + x <= a.g.nx && yt >= 0 && yt <= a.g.ny) {  // global bounds
      double2 y, d;
      window_apply(L, C, R, y, d);
      const double2 f = fc(cs, mis, t);
      r = make_double2(f.x - y.x, f.y - y.y);
    }
    if ((x & 1) == 0) {  // fine column 2X: weight 1
      acc.x += r.x;
      acc.y += r.y;
      return;
    }
    // fine column 2X+1 closes coarse column X = (x-1)/2 and opens X+1
    const int xlo = 2 * (tile_y<StResidRestrict>() * a.tx) - 1;
    if (x != xlo) {
      acc.x = fma(0.5, r.x, acc.x);
      acc.y = fma(0.5, r.y, acc.y);
      const int X = (x - 1) >> 1;
      double2* buf = rbuf[X & 1];
      buf[t] = acc;
      consumer_sync();
      // even fine rows (odd t) carry the coarse rows
      if ((t & 1) && t < kTY - 1) {
        const double2 m = buf[t - 1], p = buf[t + 1];
        const int Y = yt >> 1;
        if (live && Y <= a.gc.ny)
          a.out0[a.gc.idx(X, Y)] = make_double2(0.25 * fma(0.5, m.x + p.x, acc.x), 0.25 * fma(0.5, m.y + p.y, acc.y));
      }
    }
    acc = make_double2(0.5 * r.x, 0.5 * r.y);
  }
};

// w = u + P u_c formed at load time (prolongate + add, grid.cpp:98-120,
// solvers.cpp:508-509), then one sweep. The coarse stream of entry c is
// coarse column ceil(c/2), rows y0/2 - 1 ..; odd columns also read the
// previous entry's coarse column floor(c/2) from its (still held) slot.
struct StProlongSweep : WithF<0> {
  static constexpr int NS = 5, kOwned = kTY, kLead = 1;
  static constexpr bool kReverse = true;
  static constexpr int O_C = WithF<0>::kSlot;
  static constexpr int kSlot = O_C + sbytes(kTY / 2 + 3, 16);
  __device__ static StreamDesc stream(const MarchArgs& a, int k) {
    if (k < 4) return WithF<0>::stream(a, k);
    return {reinterpret_cast<const unsigned char*>(a.uc), 16, -1, kTY / 2 + 3, true};
  }
  __device__ static int off(int k) { return k < 4 ? WithF<0>::off(k) : O_C; }
  // coarse rows Yb-1 .. Yb+1 (Yb = yt >> 1) -> values at fine rows yt-1 .. yt+1
  __device__ static void rows_of(const unsigned char* s, const int* mis, int t, double2 (&v)[3]) {
    const int j = t >> 1;  // coarse row Yb - 1 at stream index j (y0 even)
    const double2 c0 = sat<double2>(s, O_C, mis[4], j), c1 = sat<double2>(s, O_C, mis[4], j + 1),
                  c2 = sat<double2>(s, O_C, mis[4], j + 2);
    const double2 h01 = make_double2(0.5 * c0.x + 0.5 * c1.x, 0.5 * c0.y + 0.5 * c1.y);
    const double2 h12 = make_double2(0.5 * c1.x + 0.5 * c2.x, 0.5 * c1.y + 0.5 * c2.y);
    const bool odd = t & 1;  // yt = y0 + t with y0 even
    v[0] = odd ? c1 : h01;
    v[1] = odd ? h12 : c1;
    v[2] = odd ? c2 : h12;
  }
  // The interpolated coarse column of the last loaded entry: entries 2X-1,
  // 2X and 2X+1 all use coarse column X (as ceil(c/2) for the first two, as
  // floor(c/2) for the odd 2X+1), so each is interpolated once per thread
  // instead of three times (same values: the same coarse data and formula).
  struct Carry {
    double2 v[3];
    int col = -0x40000000;
  };
  __device__ static void load(const MarchArgs&, const unsigned char* s, const unsigned char*, const int* mis,
                              int t, int c, Col& col, Carry& cy) {
    load_window(s, O_U, O_E, O_M, mis, t, col);
    const bool have = (cy.col == c - 1);
    double2 cur[3];
    if (c & 1) {
      // odd: the mean of coarse columns (c-1)/2 (the previous entry's) and (c+1)/2
      double2 prv[3] = {};
      if (have) {
#pragma unroll
        for (int q = 0; q < 3; ++q) prv[q] = cy.v[q];
      }
      rows_of(s, mis, t, cur);
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        col.u[q].x += 0.5 * prv[q].x + 0.5 * cur[q].x;
        col.u[q].y += 0.5 * prv[q].y + 0.5 * cur[q].y;
      }
    } else {
      // even: coarse column c/2, which the previous (odd) entry interpolated
      if (have) {
#pragma unroll
        for (int q = 0; q < 3; ++q) cur[q] = cy.v[q];
      } else {
        rows_of(s, mis, t, cur);
      }
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        col.u[q].x += cur[q].x;
        col.u[q].y += cur[q].y;
      }
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) cy.v[q] = cur[q];
    cy.col = c;
  }
  __device__ static void run(const MarchArgs& a, const Col& L, const Col& C, const Col& R,
                             const unsigned char* cs, const int* mis, int x, int yt, int t, bool live, double&,
                             double2&) {
    if (!live) return;
    double2 y, d;
    window_apply(L, C, R, y, d);
    a.out0[a.g.idx(x, yt)] = jacobi_update(C.u[1], fc(cs, mis, t), y, d, a.omega);
  }
};

// PCG direction: p = z + beta p_old formed at load time, Ap = A p, partial
// p.Ap (solvers.cpp:367-382). out0 = p (the other buffer), out1 = Ap; beta
// comes from the device PCG state.
struct StPupd {
  static constexpr int NS = 4, kRow0 = 0, kOwned = kTY, kLead = 0;
  static constexpr bool kReverse = true;
  static constexpr int O_U = 0, O_E = O_U + sbytes(kTY + 2, 16), O_M = O_E + sbytes(kTY + 2, 8);
  static constexpr int O_P = O_M + sbytes(kTY + 2, 1);
  static constexpr int kSlot = O_P + sbytes(kTY + 2, 16);
  __device__ static StreamDesc stream(const MarchArgs& a, int k) {
    TMG_WINDOW_STREAMS(a.u)
    return {reinterpret_cast<const unsigned char*>(a.u2), 16, -1, kTY + 2, false};
  }
  __device__ static int off(int k) { return k == 0 ? O_U : (k == 1 ? O_E : (k == 2 ? O_M : O_P)); }
  __device__ static void load(const MarchArgs& a, const unsigned char* s, const unsigned char*, const int* mis,
                              int t, int, Col& c) {
    load_window(s, O_U, O_E, O_M, mis, t, c);
    const double beta = a.st->beta;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double2 p = sat<double2>(s, O_P, mis[3], t + q);
      c.u[q] = make_double2(fma(beta, p.x, c.u[q].x), fma(beta, p.y, c.u[q].y));
    }
  }
  __device__ static void run(const MarchArgs& a, const Col& L, const Col& C, const Col& R, const unsigned char*,
                             const int*, int x, int yt, int, bool live, double& part, double2&) {
    if (!live) return;
    double2 y, d;
    window_apply<true>(L, C, R, y, d);
    const long i = a.g.idx(x, yt);
    a.out0[i] = C.u[1];
    a.out1[i] = y;
    part = fma(C.u[1].x, y.x, fma(C.u[1].y, y.y, part));
  }
};

// ------------------------------------------------------------------ kernel --

// Stages may declare a `Carry` type (state carried between consecutive loads)
template <class Stage, class = void>
struct CarryOf {
  struct type {};
  static constexpr bool used = false;
};
template <class Stage>
struct CarryOf<Stage, std::void_t<typename Stage::Carry>> {
  using type = typename Stage::Carry;
  static constexpr bool used = true;
};

// Ring depth of a stage: Stage::kRing where declared, else kStages
template <class Stage, class = void>
struct RingOf {
  static constexpr int value = kStages;
};
template <class Stage>
struct RingOf<Stage, std::void_t<decltype(Stage::kRing)>> {
  static constexpr int value = Stage::kRing;
};

// Column range of one CTA: ring entries [cf, cl]; run() is called for every
// window centre x in [xlo, xhi] (restriction stage: every fine column it
// marches; others: the owned node columns).
template <class Stage>
__device__ __forceinline__ void march_range(const MarchArgs& a, int& cf, int& cl, int& xlo, int& xhi) {
  if constexpr (Stage::kRow0 == -1) {
    const int X0 = tile_y<Stage>() * a.tx;
    const int X1 = min(X0 + a.tx, a.gc.ncol);
    xlo = 2 * X0 - 1;
    xhi = 2 * X1 - 1;  // inclusive
    cf = xlo - 1;
    cl = xhi + 1;
  } else {
    xlo = tile_y<Stage>() * a.tx;
    xhi = min(xlo + a.tx, a.g.ncol) - 1;
    cf = xlo - 1 - Stage::kLead;
    cl = xhi + 1;
  }
}

template <class Stage, bool RED>
__global__ void __launch_bounds__(kMarchThreads) k_march(MarchArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int kStages = RingOf<Stage>::value;
  __shared__ uint64_t full[kStages], empty[kStages];

  const Grid& g = a.g;
  const int t = threadIdx.x;
  const int y0 = tile_x<Stage>() * Stage::kOwned;
  int cf, cl, xlo, xhi;
  march_range<Stage>(a, cf, cl, xlo, xhi);
  const int nent = cl - cf + 1;
  auto slot = [&](int j) { return smem_raw + static_cast<size_t>(j % kStages) * Stage::kSlot; };
  auto in_storage = [&](int c) { return c >= -kGX && c < g.ncol + kGX; };

  if (t == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  double part = 0.0;
  // warp index through a shuffle: provably warp-uniform, so the producer
  // branch is uniform and its values can stay in uniform registers
  const int warp = __shfl_sync(0xffffffffu, t >> 5, 0);
  if (warp == kConsumerWarps) {
    // ---------------- producer warp: every lane runs the loop, so the copy
    // operands are warp-uniform and live in uniform registers; lane 0 issues
    // (a single-lane loop made the compiler move each operand into a uniform
    // register through a per-copy waterfall, ~25 instructions per copy)
    const bool leader = (t == kTY);
    int mis[Stage::NS];
    uint32_t bytes[Stage::NS];
    uint32_t total = 0;
#pragma unroll
    for (int k = 0; k < Stage::NS; ++k) {
      const StreamDesc d = Stage::stream(a, k);
      mis[k] = stream_mis(a, d, y0);
      // rows past ny + 2 feed no live node: the top row tile of a mesh with
      // ny + 1 = 128 k + 1 rows (every BASELINE mesh) holds one live row and
      // would copy 130 (1.5 % of a pass's bulk-copy bytes, mostly L2 hits on
      // the next column's first rows)
      const int top = (d.coarse ? a.gc.ny : g.ny) + 2;
      const int first = (d.coarse ? (y0 >> 1) : y0) + d.r0;
      const int rows = TMG_CLAMP_ROWS ? max(1, min(d.n, top - first + 1)) : d.n;
      bytes[k] = static_cast<uint32_t>((rows * d.esize + mis[k] + 15) / 16 * 16);
      total += bytes[k];
    }
    for (int j = 0; j < nent; ++j) {
      const int s = j % kStages;
      if (j >= kStages) mbar_wait(&empty[s], ((j / kStages) - 1) & 1);
      const int c = cf + j;
      // columns outside the padded storage (-1 .. nx+1) are not loaded
      if (!in_storage(c)) {
        if (leader) mbar_arrive(&full[s]);
        continue;
      }
      unsigned char* sl = slot(j);
      if (leader) {
        mbar_expect_tx(&full[s], total);
#pragma unroll
        for (int k = 0; k < Stage::NS; ++k) {
          const StreamDesc d = Stage::stream(a, k);
          const unsigned char* src = d.base + stream_row_index(a, d, c, y0) * d.esize - mis[k];
          bulk_g2s(sl + Stage::off(k), src, bytes[k], &full[s]);
        }
      }
      __syncwarp();
    }
  } else {
    // ---------------- consumers
    const int yt = y0 + Stage::kRow0 + t;
    const bool live = (yt >= y0) && (yt < y0 + Stage::kOwned) && (yt <= g.ny);
    const int lane = t & 31;
    int mis[Stage::NS];
#pragma unroll
    for (int k = 0; k < Stage::NS; ++k) mis[k] = stream_mis(a, Stage::stream(a, k), y0);
    double2 acc = make_double2(0.0, 0.0);
    auto release = [&](int j) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[j % kStages]);
    };
    // per-thread state a stage carries from one loaded entry to the next
    typename CarryOf<Stage>::type carry{};
    // load entry j into dst (needs entry j-1's slot as `prev`)
    auto fetch = [&](int j, Col& dst) {
      mbar_wait(&full[j % kStages], (j / kStages) & 1);
      const int c = cf + j;
      const unsigned char* prev = (j > 0 && in_storage(c - 1)) ? slot(j - 1) : nullptr;
      if (in_storage(c)) {
        if constexpr (CarryOf<Stage>::used) Stage::load(a, slot(j), prev, mis, t, c, dst, carry);
        else Stage::load(a, slot(j), prev, mis, t, c, dst);
      } else {
        dst = Col{};
      }
    };
    // window centred on entry j-1 (column cf + j - 1), then free its slot
    auto step = [&](const Col& L, const Col& Cc, const Col& R, int j) {
      const int x = cf + j - 1;
      if (x >= xlo && x <= xhi) Stage::run(a, L, Cc, R, slot(j - 1), mis, x, yt, t, live, part, acc);
      release(j - 1);
    };
    Col A, B, C;  // rotating column slots
    fetch(0, A);
    fetch(1, B);
    release(0);
    int j = 2;
    for (; j + 2 < nent; j += 3) {
      fetch(j, C);
      step(A, B, C, j);
      fetch(j + 1, A);
      step(B, C, A, j + 1);
      fetch(j + 2, B);
      step(C, A, B, j + 2);
    }
    if (j < nent) {
      fetch(j, C);
      step(A, B, C, j);
      ++j;
      if (j < nent) {
        fetch(j, A);
        step(B, C, A, j);
      }
    }
  }
  if constexpr (RED) {
    static_assert(Stage::kOwned == kRedRows && Stage::kRow0 == 0, "reducing stages use the reduction tiles");
    finish_reduction<kMarchThreads>(part, a.partials, tile_x<Stage>() + gridDim.x * (a.rt.ctile0 + tile_y<Stage>()), a.ticket,
                                    gridDim.x * gridDim.y, a.rt.nparts, a.rop, a.st, a.hm, a.red_out);
  }
}

}  // namespace tmg
