// Microbenchmark: cost of one cluster-barrier-separated stage on B200
// (barrier only / + global store-load round trip / + DSMEM store) for the
// V-cycle-bottom design.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void bar_rel_acq() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void bar_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned crank() { unsigned r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
template <int MODE>
__global__ void k(double* g, int iters, long long* out) {
  const unsigned nc = gridDim.x;
  __shared__ double sm[1024];
  const unsigned r = crank();
  double acc = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) { bar_rel_acq(); }
    if (MODE == 1) { bar_relaxed(); }
    if (MODE == 2) {  // global: write own slot, barrier, read the neighbour's
      g[(r * blockDim.x + threadIdx.x) + (i & 1) * 8192] = acc;
      bar_rel_acq();
      acc += g[(((r + 1) % nc) * blockDim.x + threadIdx.x) + (i & 1) * 8192];
    }
    if (MODE == 3) {  // DSMEM: store into the neighbour's smem, barrier, read own
      unsigned dst;
      unsigned src = (unsigned)__cvta_generic_to_shared(&sm[threadIdx.x + (i & 1) * 512]);
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst) : "r"(src), "r"((r + 1) % nc));
      asm volatile("st.shared::cluster.f64 [%0], %1;" :: "r"(dst), "d"(acc) : "memory");
      bar_rel_acq();
      acc += sm[threadIdx.x + (i & 1) * 512];
    }
    if (MODE == 4) {  // DSMEM remote load after barrier
      sm[threadIdx.x + (i & 1) * 512] = acc;
      bar_rel_acq();
      unsigned a;
      unsigned src = (unsigned)__cvta_generic_to_shared(&sm[threadIdx.x + (i & 1) * 512]);
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(src), "r"((r + 1) % nc));
      double v;
      asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
      acc += v;
    }
    if (MODE == 5) { __syncthreads(); }
    if (MODE == 6 || MODE == 7) {  // x1-like stage over 4225 nodes (MODE 7: + 9-point window of u)
      const int N = 4225, stride = nc * blockDim.x;
      double2* f = reinterpret_cast<double2*>(g);
      double2* u = f + 8192 * (1 + (i & 1));
      const double2* uo = f + 8192 * (2 - (i & 1));
      const double* S = g + 6 * 8192;
      for (int n = r * blockDim.x + threadIdx.x; n < N; n += stride) {
        const int x = n / 65, y = n % 65;
        const int id = x * 80 + y + 8;
        double2 fv = f[id];
        if (MODE == 7) {
          for (int q = 0; q < 9; ++q) { const double2 w = uo[id + (q / 3 - 1) * 80 + q % 3 - 1]; fv.x += w.x; fv.y += w.y; }
        }
        const double d0 = __ldg(S + id), d2 = __ldg(S + 8192 + id);
        u[id] = make_double2(fv.x / d0, fv.y / d2);
      }
      bar_rel_acq();
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && r == 0) { out[0] = t1 - t0; out[1] = (long long)acc; }
}
template <int MODE>
void run(double* g, long long* o, int cs, const char* name) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(cs); cfg.blockDim = dim3(256); cfg.attrs = at; cfg.numAttrs = 1;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int iters = MODE >= 6 ? 200 : 2000;
  cudaError_t e0 = cudaLaunchKernelEx(&cfg, k<MODE>, g, iters, o);
  cudaError_t e1 = cudaDeviceSynchronize();
  if (e0 != cudaSuccess || e1 != cudaSuccess) { printf("%s cs=%d launch %s / %s\n", name, cs, cudaGetErrorString(e0), cudaGetErrorString(e1)); return; }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, k<MODE>, g, iters, o);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  long long h[2]; cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
  printf("%-28s cs=%2d  %7.1f cycles/stage  %6.3f us/stage  err=%s\n", name, cs, (double)h[0] / iters, ms * 1e3 / iters,
         cudaGetErrorString(cudaGetLastError()));
}
// empty-kernel chain in a graph, for the per-launch floor
__global__ void kempty(double* g) { if (threadIdx.x == 0 && blockIdx.x == 0) g[0] += 1.0; }
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); fflush(stdout); return 1; } } while (0)
int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  double* g; long long* o;
  CK(cudaMalloc(&g, 1 << 21)); CK(cudaMalloc(&o, 64)); CK(cudaMemset(g, 0, 1 << 21));
  for (int cs : {8, 16}) {
    run<0>(g, o, cs, "barrier release/acquire");
    run<1>(g, o, cs, "barrier relaxed");
    run<2>(g, o, cs, "global st + bar + ld");
    run<3>(g, o, cs, "dsmem st + bar + ld");
    run<4>(g, o, cs, "st + bar + dsmem ld");
    run<5>(g, o, cs, "__syncthreads");
    run<6>(g, o, cs, "x1-like stage, 4225 nodes");
    run<7>(g, o, cs, "+ 9-point window");
  }
  cudaStream_t s; cudaStreamCreate(&s);
  for (int blocks : {1, 16, 148}) {
    cudaGraph_t gr; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 100; ++i) kempty<<<blocks, 512, 0, s>>>(g);
    cudaStreamEndCapture(s, &gr);
    cudaGraphInstantiate(&ge, gr, 0);
    cudaGraphLaunch(ge, s);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s); cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("graph of 100 dependent empty kernels, %3d CTAs: %.3f us per kernel\n", blocks, ms * 10);
  }
  return 0;
}
