// Warp-specialised variant of the two-stage coarse marching kernels
// (tmg_smarch.cuh): the same schedule, ring, arithmetic and results, with
// stage A and stage B on DIFFERENT consumer warps.
//
// In k_smarch every consumer thread runs both stages of a ring entry between
// two CTA-wide consumer barriers, so a CTA holds both 3x3 windows plus the
// cached left-column blocks (226 registers) and two CTAs per SM leave ~8
// warps to hide the FP64 and shared-memory latencies of two stencil
// applications (ncu: issue ~30 %, stalls on long/short scoreboard and fixed
// latency). Here a CTA has
//
//   warps 0..2   stage A: the stage-A inputs of column c (x1 or w = x2 + P u_c)
//                and stage A at column c-1; they wait on the ring's full
//                barriers and hand their outputs to B through a
//                double-buffered shared column (named barriers
//                full/empty, producer/consumer style);
//   warps 3..5   stage B at column c-3 (and the DOWN restriction of column
//                c-4); they release the ring slots;
//   warp 6       the TMA producer, unchanged.
//
// Each group holds one window, so a thread needs about half the registers and
// an SM runs 14 warps instead of 8 at the same shared memory. A and B are
// decoupled by one column of buffering, so a slow B step no longer stalls the
// next A step. Every per-node operation is the one k_smarch performs in the
// same order, so the results are bitwise those of k_smarch
// (tests/test_gpu_parity.py::test_specialised_coarse_kernels_are_bitwise).
#pragma once

#include "tmg_smarch.cuh"

namespace tmg {

constexpr int kS2Threads = 2 * kSY + 32;  // A group, B group, producer warp

// named barriers: 1 = A group, 2 = B group, 3 + k = xb[k] full, 5 + k = xb[k] empty
// (immediate ids, so ptxas reserves only the barriers used)
template <int ID, int N>
__device__ __forceinline__ void nb_sync() {
  asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(N) : "memory");
}
template <int ID, int N>
__device__ __forceinline__ void nb_arrive() {
  asm volatile("bar.arrive %0, %1;" ::"n"(ID), "n"(N) : "memory");
}
// wait for an mbarrier phase that has (or will have) completed, without the
// suspend hint: B only re-checks a phase A has already seen complete
__device__ __forceinline__ void mbar_wait_done(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITD_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITD_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <bool UP>
__global__ void __launch_bounds__(kS2Threads, 2) k_smarch2(const __grid_constant__ SMarchArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int kSStages = s_stages<UP>();
  __shared__ uint64_t full[kSStages], empty[kSStages];
  __shared__ double2 xa[2][kSY + 2];  // stage-A inputs (x1 / w), A group only
  __shared__ double2 xb[2][kSY + 2];  // stage-A outputs (x2 / x3), A -> B
  __shared__ double2 rb[2][kSY];      // DOWN: stage-B residual rows, B group only
  constexpr int kSlot = UP ? kSSlotUp : kSSlotDown;
  constexpr int kN = 2 * kSY;  // threads of a full/empty hand-off

  const Grid& g = a.g;
  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const bool isA = warp < kSWarps;
  const bool isB = !isA && warp < 2 * kSWarps;
  const int t = isA ? tid : tid - kSY;  // row index within the tile for A and B
  constexpr int R0 = UP ? -1 : -2;
  constexpr int kOwned = UP ? kSY - 2 : kSY - 4;
  const int y0 = blockIdx.x * kOwned;
  int cf, cl, xlo, xhi;
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
  constexpr int r0 = r0c<UP>();
  const int cr0 = (UP ? -2 : 0);

  if (tid == 0) {
    for (int s = 0; s < kSStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kSWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < kSY + 2; i += kS2Threads) {
    xa[0][i] = xa[1][i] = xb[0][i] = xb[1][i] = make_double2(0.0, 0.0);
    if (i < kSY) rb[0][i] = rb[1][i] = make_double2(0.0, 0.0);
  }
  __syncthreads();

  const uintptr_t pf = reinterpret_cast<uintptr_t>(a.f);
  constexpr int misS = ((r0c<UP>() + kOY) & 1) ? 8 : 0;
  const int misF = static_cast<int>((pf + static_cast<uintptr_t>(g.idx(0, y0 + r0)) * 16) & 15u);
  int misC = 0;
  if (UP) {
    misC = static_cast<int>((reinterpret_cast<uintptr_t>(a.uc) +
                             static_cast<uintptr_t>(a.gc.idx(0, (y0 >> 1) + cr0)) * 16) & 15u);
  }

  if (!isA && !isB) {
    // ---------------------------------------------------------- producer
    const bool leader = (tid == 2 * kSY);
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

  const int yt = y0 + R0 + t;
  const int lane = tid & 31;
  const int j = t + 1;
  const int jh = (t == 0) ? 0 : kSY + 1;
  const int yh = y0 + r0 + jh;
  auto row_in = [&](int y) { return y >= 0 && y <= g.ny; };
  auto col_in = [&](int x) { return g.x0 + x >= 0 && g.x0 + x <= g.nx; };
  const bool rin = row_in(yt), hin = row_in(yh);
  const bool tB = t >= 1 && t < kSY - 1;
  auto fat = [&](const unsigned char* s, int jj) {
    return *reinterpret_cast<const double2*>(s + kSO_F + misF + jj * 16);
  };
  const double2 z2 = make_double2(0.0, 0.0);
  auto sel = [](bool p, double2 v) { return p ? v : make_double2(0.0, 0.0); };
  const int nsteps = nent + (UP ? 1 : 2);

  if (isA) {
    // ------------------------------------------------------------ stage A
    auto a_in_down = [&](const unsigned char* s, int jj, double2& rc) {
      const SPlanes P{s, misS};
      const double2 f = fat(s, jj);
      rc = make_double2(rcp_nr(P.at(0, jj)), rcp_nr(P.at(2, jj)));
      return make_double2(a.omega * f.x * rc.x, a.omega * f.y * rc.y);
    };
    auto a_in_up = [&](const unsigned char* s, const unsigned char* ps, bool odd_col, int jj, double2 xv) {
      const int y = y0 + r0 + jj;
      const int gy = y - 2 * ((y0 >> 1) + cr0);
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
    double2 wa[3][3];
    double2 rd[3];
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      rd[p] = z2;
#pragma unroll
      for (int q = 0; q < 3; ++q) wa[p][q] = z2;
    }
    int si = 0;
    uint32_t ph = 0;
    const unsigned char* sp1 = nullptr;
    const unsigned char* sp2 = nullptr;
    auto step = [&](auto phase, int e) {
      constexpr int P = decltype(phase)::value;
      constexpr int IL = P, IC = (P + 1) % 3, IR = (P + 2) % 3;
      const int c = cf + e;
      if (e >= nent) return;  // A has no drain steps
      const unsigned char* s0 = smem_raw + static_cast<size_t>(si) * kSlot;
      double2* xin = xa[e & 1];
      mbar_wait(&full[si], ph);
      {
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
        xin[t + 1] = sel(ci && rin, v);
        if (t == 0) xin[0] = sel(ci && hin, vh);
        if (t == kSY - 1) xin[kSY + 1] = sel(ci && hin, vh);
      }
      nb_sync<1, kSY>();
#pragma unroll
      for (int q = 0; q < 3; ++q) wa[IR][q] = xin[t + q];
      double2 va = z2;
      if (e >= 2) {
        double2 ya, da;
        s_apply(SPlanes{sp1, misS}, SPlanes{sp2, misS}, j, wa[IL], wa[IC], wa[IR], ya, da);
        const int x = c - 1;
        const double2 f = fat(sp1, j);
        const double2 r = UP ? make_double2(rcp_nr(da.x), rcp_nr(da.y)) : rd[IC];
        va = sel(col_in(x) && rin, s_jacobi_r(wa[IC][1], f, ya, r, a.omega));
        if (!UP && t >= 2 && t < 2 + kOwned && x > xlo && x <= xhi && x < g.ncol && yt <= g.ny)
          a.out[g.idx(x, yt)] = va;
      }
      // hand column c-1 to B (B frees xb[e&1] after reading column c-3)
      if (e & 1) {
        nb_sync<6, kN>();
        xb[1][t + 1] = va;
        nb_arrive<4, kN>();
      } else {
        nb_sync<5, kN>();
        xb[0][t + 1] = va;
        nb_arrive<3, kN>();
      }
      sp2 = sp1;
      sp1 = s0;
      if (++si == kSStages) {
        si = 0;
        ph ^= 1u;
      }
    };
    int e = 0;
    for (; e + 2 < nsteps; e += 3) {
      step(std::integral_constant<int, 0>{}, e);
      step(std::integral_constant<int, 1>{}, e + 1);
      step(std::integral_constant<int, 2>{}, e + 2);
    }
    if (e < nsteps) step(std::integral_constant<int, 0>{}, e);
    if (e + 1 < nsteps) step(std::integral_constant<int, 1>{}, e + 1);
    return;
  }

  // -------------------------------------------------------------- stage B
  // both xb buffers start free
  nb_arrive<5, kN>();
  nb_arrive<6, kN>();
  double2 wb[3][3];
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int q = 0; q < 3; ++q) wb[p][q] = z2;
  double lc[12];
#pragma unroll
  for (int k = 0; k < 12; ++k) lc[k] = 0.0;
  double2 acc = z2, bres = z2;
  // ring position of entry e-3 (slot, phase)
  int sb = kSStages - 3;
  uint32_t phb = 1;  // entry -3's phase parity (never waited on: e >= 3)

  auto step = [&](auto phase, int e) {
    constexpr int P = decltype(phase)::value;
    constexpr int IL = P, IC = (P + 1) % 3, IR = (P + 2) % 3;
    const int c = cf + e;
    // stage-B window column c-2 (stage A ran there at step e-1)
    if (e >= 1 && e <= nent) {
      const int k = (e - 1) & 1;
      if (k) nb_sync<4, kN>();
      else nb_sync<3, kN>();
#pragma unroll
      for (int q = 0; q < 3; ++q) wb[IR][q] = tB ? xb[k][t + q] : z2;
      if (e + 1 <= nent - 1) {  // A writes xb[k] again at step e+1
        if (k) nb_arrive<6, kN>();
        else nb_arrive<5, kN>();
      }
    } else {
#pragma unroll
      for (int q = 0; q < 3; ++q) wb[IR][q] = z2;
    }
    if (!UP) {
      // rb[(e-1)&1] was written by stage B at step e-1
      nb_sync<2, kSY>();
      if (e >= 4) {
        const int x = c - 4;
        if (x >= xlo && x <= xhi) {
          const double2* rbp = rb[(e - 1) & 1];
          const double2 rm = rbp[t > 0 ? t - 1 : 0], rp = rbp[t < kSY - 1 ? t + 1 : kSY - 1];
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
    }
    if (e >= 3 && e <= nent) {
      const unsigned char* sp3 = smem_raw + static_cast<size_t>(sb) * kSlot;
      mbar_wait_done(&full[sb], phb);
      double2 yb, db;
      s_apply(SPlanes{sp3, misS}, LCache{lc}, j, wb[IL], wb[IC], wb[IR], yb, db);
      const int x = c - 3;
      const SPlanes C{sp3, misS};
      const double2 f = fat(sp3, j);
      const bool ok = tB && col_in(x) && rin;
      if (UP) {
        const double2 vb = sel(ok, s_jacobi_r(wb[IC][1], f, yb, make_double2(rcp_nr(db.x), rcp_nr(db.y)), a.omega));
        if (tB && x >= xlo && x <= xhi && yt <= g.ny) a.out[g.idx(x, yt)] = vb;
      } else {
        bres = sel(ok, make_double2(f.x - yb.x, f.y - yb.y));
        rb[e & 1][t] = bres;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        lc[k] = C.at(7 + k, j + 1);
        lc[4 + k] = C.at(11 + k, j);
        lc[8 + k] = C.at(15 + k, j - 1);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[sb]);
    } else if (!UP) {
      // keep the restriction input of this step defined (no stage B here)
      rb[e & 1][t] = bres;
    }
    if (++sb == kSStages) {
      sb = 0;
      phb ^= 1u;
    }
  };
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
