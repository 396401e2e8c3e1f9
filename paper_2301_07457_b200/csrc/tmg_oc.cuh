// OC exchange between two phases on the device (oc_update_pair,
// mto.cpp:142-227).
//
// The reference bisects for the volume multiplier: up to 101 full element
// passes, each a clamp(a * (max(floor, gain) / lambda)^damping) (or a clamp of
// a uniform shift when no element prefers phase a) followed by the mean. Here
//   k_oc_prep   reads the element-major density once (phases a, b), forms
//               {a, gain} and {lo, hi} per element in scratch (two 16-byte
//               streams) and the per-CTA maxima of gain and of the move limit;
//   k_oc_gain   turns gain into the lambda-independent factor once the
//               global maximum is known (multiplicative branch);
//   k_oc_bisect runs the whole bisection in one cooperatively launched
//               persistent grid: per step every CTA reduces its elements,
//               publishes one partial, crosses a grid barrier and sums the
//               partials in index order itself, so every CTA takes the same
//               (deterministic) branch; at the end it writes phases a and b
//               back into the element-major density.
// Bytes per element and step: {a, gain, lo, hi} = 32 (the reference streams
// the same plus its cand write).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "tmg_kernels.cuh"

namespace tmg {

constexpr int kOcThreads = 256;
constexpr unsigned kOcMaxStaged = 1536;  // step partials staged in shared memory (148 SMs x 8 CTAs = 1184)

struct OcArgs {
  long ne;
  int np;            // phases per element (element-major stride)
  int pa, pb;
  double* alpha;     // element-major density, device (in/out)
  const double* sa;  // filtered sensitivities of phases a and b
  const double* sb;
  const double* mv;  // per-element move limits
  double eps;        // density floor
  double target;
  double damping;
  // scratch per element as two 16-byte streams, {alpha_a, gain} and {lo, hi}:
  // a warp's load of either is 512 contiguous bytes (one 32-byte record per
  // element read as two 16-byte halves used half of every sector per request)
  double2* el0;
  double2* el1;
  double* pmax;      // per-CTA [max gain, max move] (prep) -> 2 * gridDim
  double* part;      // per-CTA step partials, 2 * gridDim (double-buffered)
  unsigned* bar;     // grid barrier [arrivals, generation]
  int* met;          // out: [0] 1 when the volume target was met, [1] bisection steps
};

__device__ __forceinline__ double s_max(double a, double b) { return (a < b) ? b : a; }  // std::max
__device__ __forceinline__ double s_min(double a, double b) { return (b < a) ? b : a; }  // std::min
__device__ __forceinline__ double s_clamp(double v, double lo, double hi) { return s_min(hi, s_max(lo, v)); }

__global__ void __launch_bounds__(kOcThreads) k_oc_prep(OcArgs a) {
  double mg = -1e300, mm = 0.0;
  for (long e = blockIdx.x * static_cast<long>(kOcThreads) + threadIdx.x; e < a.ne;
       e += static_cast<long>(gridDim.x) * kOcThreads) {
    const double g = a.sb[e] - a.sa[e];
    const double m = a.mv[e];
    const double x = a.alpha[e * a.np + a.pa];
    const double pair = x + a.alpha[e * a.np + a.pb];
    mg = s_max(mg, g);
    mm = s_max(mm, m);
    a.el0[e] = make_double2(x, g);
    a.el1[e] = make_double2(s_max(a.eps, x - m), s_min(pair - a.eps, x + m));
  }
  // block maxima (max is exact in any order)
  __shared__ double smg[kOcThreads], smm[kOcThreads];
  smg[threadIdx.x] = mg;
  smm[threadIdx.x] = mm;
  __syncthreads();
  for (int o = kOcThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      smg[threadIdx.x] = s_max(smg[threadIdx.x], smg[threadIdx.x + o]);
      smm[threadIdx.x] = s_max(smm[threadIdx.x], smm[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    a.pmax[2 * blockIdx.x] = smg[0];
    a.pmax[2 * blockIdx.x + 1] = smm[0];
  }
}

// grid-wide barrier of a cooperatively launched (co-resident) grid
__device__ __forceinline__ void oc_grid_sync(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*reinterpret_cast<volatile unsigned*>(bar + 1) == gen) __nanosleep(64);
    }
    __threadfence();
  }
  ++gen;
  __syncthreads();
}

// The candidate of element e for the current step (mto.cpp:176-181,
// 198-204). In the multiplicative branch a.gain holds q = sqrt(max(floor,
// gain)) for the reference's default damping 0.5 (so the step is a multiply
// by the uniform 1/sqrt(lambda)), else log(max(floor, gain)) (one exp per
// element instead of a pow). Both agree with the reference's
// pow(max(floor, gain) / lambda, damping) to a few ulp.
struct OcStep {
  bool shift, half;
  double t;       // shift branch
  double scale;   // 1/sqrt(lambda) (half) or log(lambda)
  double damping;
};
template <int MODE>  // 0: uniform shift, 1: damping 0.5, 2: any damping
__device__ __forceinline__ double oc_cand(const double4 v, const OcStep& s) {
  // v = {alpha_a, lo, hi, q}
  if (MODE == 0) return s_clamp(v.x + s.t, v.y, v.z);
  const double p = (MODE == 1) ? v.w * s.scale : exp(s.damping * (v.w - s.scale));
  return s_clamp(v.x * p, v.y, v.z);
}
// The records are read-only inside k_oc_bisect (k_oc_gain, a launch of its
// own, finishes them), so they go through the non-coherent path and the
// compiler is free to issue a whole batch of loads before the first use
// (__ldcg is an asm volatile: the loads kept their program order between the
// candidates and only three or four were in flight per thread).
__device__ __forceinline__ double4 ld_el(const double2* __restrict__ el0, const double2* __restrict__ el1, long e) {
  const double2 u = __ldg(el0 + e), w = __ldg(el1 + e);
  return make_double4(u.x, w.x, w.y, u.y);
}

// global maxima of gain and move limit from the prep partials
__device__ __forceinline__ void oc_maxima(const OcArgs& a, int prep_blocks, double& max_gain, double& max_move) {
  max_gain = -1e300;
  max_move = 0.0;
  for (int k = 0; k < prep_blocks; ++k) {
    max_gain = s_max(max_gain, __ldcg(a.pmax + 2 * k));
    max_move = s_max(max_move, __ldcg(a.pmax + 2 * k + 1));
  }
}

// The lambda-independent part of every element's factor (multiplicative
// branch): gain -> sqrt(max(floor, gain)) for damping 0.5, else its log.
__global__ void __launch_bounds__(kOcThreads) k_oc_gain(OcArgs a, int prep_blocks) {
  double max_gain, max_move;
  oc_maxima(a, prep_blocks, max_gain, max_move);
  if (!(max_gain > 0.0)) return;  // shift branch: the gain is not used
  const double floor_gain = 1e-4 * max_gain;
  const bool half = a.damping == 0.5;
  for (long e = blockIdx.x * static_cast<long>(kOcThreads) + threadIdx.x; e < a.ne;
       e += static_cast<long>(gridDim.x) * kOcThreads) {
    double2 v = a.el0[e];  // whole 16-byte record in and out: full sectors both ways
    const double g = s_max(floor_gain, v.y);
    v.y = half ? sqrt(g) : log(g);
    a.el0[e] = v;
  }
}

// One bisection step's sum over the elements a thread owns: kOcU records
// (2 kOcU 16-byte loads) issued as one batch per round, one partial sum per
// slot, a fixed pairwise tree at the end (deterministic). The mode is a
// template argument so the common damping-0.5 loop carries no exp()
// registers. The kernel is bound by loads in flight (ncu: > 90 % of cycles
// without an eligible warp), and its speed follows the compiler's schedule
// of that batch: at 80 registers and three CTAs per SM the eight loads go
// out back to back and the kernel streams at 0.83 of the DRAM peak (ncu);
// tighter register caps (48, 40) serialise part of the batch behind the
// first candidates (0.54-0.63 of HBM end to end), and eight records per
// round or a CTA-contiguous element order were slower as well (same-box A/B,
// tools/ab_oc.sh). A shared-memory ring filled by bulk copies (one producer
// warp, 512-element entries) was correct but slower still (10.5-12.7 ms
// against 7.5 ms at 8192^2): with two elements per thread and ring entry the
// mbarrier hand-off dominates.
#ifndef TMG_OC_U
#define TMG_OC_U 4
#endif
#ifndef TMG_OC_MINB
#define TMG_OC_MINB 3
#endif
constexpr int kOcU = TMG_OC_U;
template <int MODE>
__device__ __forceinline__ double oc_step_sum(const double2* __restrict__ el0, const double2* __restrict__ el1,
                                              long ne, const OcStep& st, long e, long stride) {
  double s[kOcU];
#pragma unroll
  for (int k = 0; k < kOcU; ++k) s[k] = 0.0;
#pragma unroll 1
  for (; e + (kOcU - 1) * stride < ne; e += kOcU * stride) {
    double4 v[kOcU];
#pragma unroll
    for (int k = 0; k < kOcU; ++k) v[k] = ld_el(el0, el1, e + k * stride);
#pragma unroll
    for (int k = 0; k < kOcU; ++k) s[k] += oc_cand<MODE>(v[k], st);
  }
#pragma unroll 1
  for (; e < ne; e += stride) s[0] += oc_cand<MODE>(ld_el(el0, el1, e), st);
#pragma unroll
  for (int w = 1; w < kOcU; w *= 2)
#pragma unroll
    for (int k = 0; k + w < kOcU; k += 2 * w) s[k] += s[k + w];
  return s[0];
}

__global__ void __launch_bounds__(kOcThreads, TMG_OC_MINB) k_oc_bisect(OcArgs a, int prep_blocks) {
  __shared__ double red[kOcThreads / 32];
  __shared__ double sparts[kOcMaxStaged];
  __shared__ double s_mean;
  __shared__ unsigned s_gen;
  if (threadIdx.x == 0) s_gen = *reinterpret_cast<volatile unsigned*>(a.bar + 1);
  // global maxima from the prep partials (identical in every CTA)
  double max_gain, max_move;
  oc_maxima(a, prep_blocks, max_gain, max_move);
  const double2* __restrict__ el0 = a.el0;
  const double2* __restrict__ el1 = a.el1;
  __syncthreads();
  unsigned gen = s_gen;
  OcStep st{};
  st.shift = !(max_gain > 0.0);  // mto.cpp:170: max_gain <= 0
  st.half = a.damping == 0.5;
  st.damping = a.damping;
  const double vol_tol = 1e-6;
  double t_lo = -max_move, t_hi = max_move, l_lo = 1e-10, l_hi = 1e10;
  bool met = false;
  const long stride = static_cast<long>(gridDim.x) * kOcThreads;
  for (int it = 0; it <= 100; ++it) {
    if (st.shift) {
      st.t = 0.5 * (t_lo + t_hi);
    } else {
      const double lambda = sqrt(l_lo * l_hi);
      st.scale = st.half ? 1.0 / sqrt(lambda) : log(lambda);
      st.t = lambda;  // kept for the bound update below
    }
    const long e0 = blockIdx.x * static_cast<long>(kOcThreads) + threadIdx.x;
    double s = st.shift ? oc_step_sum<0>(el0, el1, a.ne, st, e0, stride)
                        : (st.half ? oc_step_sum<1>(el0, el1, a.ne, st, e0, stride)
                                   : oc_step_sum<2>(el0, el1, a.ne, st, e0, stride));
    // fixed-shape block tree
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = 0.0;
      for (int w = 0; w < kOcThreads / 32; ++w) b += red[w];
      a.part[(it & 1) * gridDim.x + blockIdx.x] = b;
    }
    oc_grid_sync(a.bar, gen);
    // every CTA sums all partials in index order. The block first stages them
    // in shared memory with one coalesced load: thread 0 reading them from L2
    // one after another put load latency on every step.
    const double* parts = a.part + (it & 1) * gridDim.x;
    const bool staged = gridDim.x <= kOcMaxStaged;
    if (staged) {
      for (unsigned k = threadIdx.x; k < gridDim.x; k += kOcThreads) sparts[k] = __ldcg(parts + k);
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      double sum = 0.0;
      if (staged) {
        for (unsigned k = 0; k < gridDim.x; ++k) sum += sparts[k];
      } else {
        for (unsigned k = 0; k < gridDim.x; ++k) sum += __ldcg(parts + k);
      }
      s_mean = sum / static_cast<double>(a.ne);
    }
    __syncthreads();
    const double mean = s_mean;
    if (blockIdx.x == 0 && threadIdx.x == 0) a.met[1] = it + 1;
    if (fabs(mean - a.target) <= vol_tol) {
      met = true;
      break;
    }
    if (st.shift) (mean > a.target ? t_hi : t_lo) = st.t;
    else (mean > a.target ? l_lo : l_hi) = st.t;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) a.met[0] = met ? 1 : 0;
  if (!met) return;
  for (long e = blockIdx.x * static_cast<long>(kOcThreads) + threadIdx.x; e < a.ne; e += stride) {
    const double4 v = ld_el(el0, el1, e);
    const double c = st.shift ? oc_cand<0>(v, st) : (st.half ? oc_cand<1>(v, st) : oc_cand<2>(v, st));
    const double pair = v.x + a.alpha[e * a.np + a.pb];
    a.alpha[e * a.np + a.pa] = c;
    a.alpha[e * a.np + a.pb] = pair - c;
  }
}

}  // namespace tmg

namespace tmg {

// ------------------------------------------ optimizer loop (mto.cpp:229-354)

// DensityField::uniform (density.cpp:33-42)
__global__ void k_fill_uniform(long ne, int np, const double* __restrict__ fractions, double* __restrict__ alpha) {
  for (long k = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; k < ne * np;
       k += static_cast<long>(gridDim.x) * blockDim.x)
    alpha[k] = fractions[k % np];
}

// DensityField::max_change (density.cpp:60-66) into *out as the bits of a
// non-negative double (uint64 order = double order: the max is exact and
// independent of the order of the atomics)
__global__ void k_max_abs_diff(long n, const double* __restrict__ a, const double* __restrict__ b,
                               unsigned long long* out) {
  double m = 0.0;
  for (long k = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<long>(gridDim.x) * blockDim.x)
    m = s_max(m, fabs(a[k] - b[k]));
  for (int o = 16; o > 0; o >>= 1) m = s_max(m, __shfl_down_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(m)));
}

// per-element move limits: halved when a phase's change reverses, regrown by
// 5 % on a consistent move (mto.cpp:325-343)
__global__ void k_move_adapt(long ne, int np, const double* __restrict__ after, const double* __restrict__ before,
                             double* __restrict__ last, double* __restrict__ move, double move_limit) {
  for (long e = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; e < ne;
       e += static_cast<long>(gridDim.x) * blockDim.x) {
    bool flipped = false, moved = false;
    for (int i = 0; i < np; ++i) {
      const double delta = after[e * np + i] - before[e * np + i];
      const double l = last[e * np + i];
      if (fabs(delta) > 1e-12) moved = true;
      if (delta * l < -1e-12) flipped = true;
      last[e * np + i] = delta;
    }
    double mv = move[e];
    if (flipped) mv = s_max(1e-4, 0.5 * mv);
    else if (moved) mv = s_min(move_limit, 1.05 * mv);
    move[e] = mv;
  }
}

}  // namespace tmg
