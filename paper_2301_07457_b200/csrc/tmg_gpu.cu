// libtmg_gpu.so -- host orchestration of the B200 pCGMG solve behind the C ABI
// of include/tmg_gpu.h.
//
// A handle drives one or more *ranks*. A rank owns an x-slab of every
// distributed level (contiguous node columns of the reference's column-major
// numbering, grid.hpp:19) plus kGX ghost columns per side, and a full copy of
// every replicated (small) level. One process per GPU uses one local rank and
// NCCL for the exchanges; a single process can also drive several ranks on
// one device (LocalComm), which is how the decomposition is tested on one
// B200. With one rank every level is global and nothing is exchanged.
//
// Per outer iteration of the reference optimizer (mto.cpp:267-283):
//   setup : Galerkin hierarchy (K6) + coarsest factor/inverse (K7) on device
//   solve : PCG (K8) preconditioned by one gamma-cycle (K1-K5, K7) per
//           iteration; one PCG iteration is a captured CUDA graph, the host
//           only reads a 40-byte mirror of the PCG scalars to run the
//           reference's stopping test (solvers.cpp:388) and error checks.
#include <cudaTypedefs.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <memory>
#include <string>
#include <vector>

#include "../../include/tmg_gpu.h"
#include "tmg_kernels.cuh"
#include "tmg_march.cuh"
#include "tmg_smarch.cuh"
#include "tmg_smarch2.cuh"
#include "tmg_stile.cuh"
#include "tmg_oc.cuh"

using namespace tmg;

namespace tmgi {

struct TmgError {
  int code;
  std::string msg;
  int row;
};

[[noreturn]] void fail(int code, const std::string& msg, int row = -1) {
  throw TmgError{code, msg, row};
}

// NVTX range for the phases the reference times with steady_clock
// (solvers.cpp:335, 393; mto.cpp:264-350): setup, solve, outer iteration, OC
// exchange. Header-only NVTX v3: free unless a profiler is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

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
  Grid g{};         // as stored by this rank (slab or global)
  bool dist = false;
  long ndof = 0;    // global dofs of the level
  double2* u[2] = {nullptr, nullptr};  // iterate (ping-pong for Jacobi)
  double2* f = nullptr;                // right-hand side of this level
  double2* res = nullptr;              // residual scratch
  double* S = nullptr;                 // stencil planes (coarse levels)
  int cur = 0;
};

dim3 node_block() { return dim3(kBX, kBY); }
dim3 node_grid(const Grid& g) {
  return dim3((g.ny + 1 + kBX - 1) / kBX, (g.ncol + kBY - 1) / kBY);
}

Grid make_grid(int nx, int ny, int x0, int ncol) {
  Grid g;
  g.nx = nx;
  g.ny = ny;
  // y in [-1, ny+1] at offset kOY; a multiple of 16 nodes keeps every column
  // start 16-byte aligned for the TMA bulk copies of the byte-wide mask
  g.P = ((ny + 2 + kOY) + 15) / 16 * 16;
  g.x0 = x0;
  g.ncol = ncol;
  g.size = static_cast<long>(ncol + 2 * kGX) * g.P;
  return g;
}

// ---------------------------------------------------------------- NCCL ------
// libnccl is bound at run time (the process may already hold torch's copy of
// libnccl.so.2; dlopen then returns that same library).
struct NcclApi {
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (lib) {
      api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(lib, "ncclGetUniqueId"));
      api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(lib, "ncclCommInitRank"));
      api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(lib, "ncclCommDestroy"));
      api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(lib, "ncclAllReduce"));
      api.broadcast = reinterpret_cast<decltype(api.broadcast)>(dlsym(lib, "ncclBroadcast"));
      api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(lib, "ncclAllGather"));
      api.send = reinterpret_cast<decltype(api.send)>(dlsym(lib, "ncclSend"));
      api.recv = reinterpret_cast<decltype(api.recv)>(dlsym(lib, "ncclRecv"));
      api.groupStart = reinterpret_cast<decltype(api.groupStart)>(dlsym(lib, "ncclGroupStart"));
      api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(dlsym(lib, "ncclGroupEnd"));
      api.errorString = reinterpret_cast<decltype(api.errorString)>(dlsym(lib, "ncclGetErrorString"));
    }
  }
  if (!api.commInitRank) fail(TMG_ERR_NCCL, "libnccl.so.2 not available");
  return api;
}

#define NK(call)                                                                      \
  do {                                                                                \
    ncclResult_t r_ = (call);                                                         \
    if (r_ != ncclSuccess) fail(TMG_ERR_NCCL, std::string(#call) + ": " + nccl().errorString(r_)); \
  } while (0)

}  // namespace tmgi
using namespace tmgi;

// ------------------------------------------------------------------ rank ----

struct Rank {
  int index = 0;  // global rank
  int nx = 0, ny = 0, nc = 0;
  std::vector<Level> lev;  // lev[0] coarsest ... lev[nc] finest (grid.hpp:47)
  double* E = nullptr;
  uint8_t* M = nullptr;
  // coarsest level (K7), replicated on every rank
  int n0 = 0;
  double *A0 = nullptr, *LiT = nullptr, *Ainv = nullptr;
  int* bad_row = nullptr;
  // PCG (K8)
  double2 *x = nullptr, *r = nullptr, *ap = nullptr, *b = nullptr, *x0 = nullptr;
  double2* r2 = nullptr;  // second residual buffer: the fused update alternates r / r2
  double2* pbuf[2] = {nullptr, nullptr};  // PCG directions (old / new alternate)
  double* partials = nullptr;  // fine-level reduction partials, global tile layout
  double* gparts = nullptr;    // several ranks: the all-reduced partial array
  unsigned* ticket = nullptr;
  unsigned* rticket = nullptr;  // ticket for reducing launches (null with several ranks)
  PcgState* st = nullptr;
  HostMirror* hm = nullptr;      // pinned, mapped
  HostMirror* hm_dev = nullptr;  // device alias of hm
  // device-side PCG loop: its record and residual history (pinned, mapped)
  LoopRecord* lrec = nullptr;
  LoopRecord* lrec_dev = nullptr;
  Readback* rbk = nullptr;  // mid-solve readbacks (pinned, mapped)
  Readback* rbk_dev = nullptr;
  double* hist = nullptr;
  double* hist_dev = nullptr;
  int hist_cap = 0;
  double* scal = nullptr;        // device scalars: [0] result, [1] rank partial, [2] global sum
  double* scal_host = nullptr;   // pinned
  // scratch for consumers
  double* dense = nullptr;
  long dense_cap = 0;
  double* aux = nullptr;
  long aux_cap = 0;
  double* aux2 = nullptr;
  long aux2_cap = 0;
  double* ocbuf = nullptr;  // OC exchange scratch (tmg_oc.cuh)
  long ocbuf_cap = 0;
  // pipelined solves (tmg_gpu_stage_inputs / tmg_gpu_solve_staged): two
  // staging slots of moduli + rhs and the solution's staging copy, in the
  // resident arrays' padded layouts (allocated on first use)
  double* Es[2] = {nullptr, nullptr};
  double2* bs[2] = {nullptr, nullptr};
  double2* us = nullptr;

  Level& fine() { return lev[nc]; }
  double2* rbuf(int k) const { return k ? r2 : r; }
  FineOp fine_op() const { return FineOp{E, M, lev[nc].g.P}; }
  StencilOp stencil_op(int l) const { return StencilOp{lev[l].S, lev[l].g.size, lev[l].g.P}; }
};

namespace tmgi {

// Halo exchange and all-reduce between the ranks of one solve.
struct Comm {
  virtual ~Comm() = default;
  // ghost columns of a distributed level: `wl` columns on the left from the
  // left neighbour's last owned columns, `wr` on the right from the right
  // neighbour's first ones; a node column is P elements of `esize` bytes
  // starting at field(rank).
  virtual void halo(std::vector<Rank*>& rs, int level, const std::function<void*(Rank&)>& field, size_t esize,
                    int wl, int wr, cudaStream_t s) = 0;
  // owned column ranges [X0_r, X0_r + n_r) of a replicated level's planes
  // (plane stride in elements) from every rank to every rank's full copy
  virtual void gather_columns(std::vector<Rank*>& rs, int level, const std::function<void*(Rank&)>& field,
                              size_t esize, long plane_stride, int planes, const std::vector<int>& X0,
                              const std::vector<int>& ncol, cudaStream_t s) = 0;
  // several ghost exchanges at one point of the schedule (same fields and
  // widths as the separate calls, in this order): NCCL issues them as one
  // group, one launch and one latency instead of one per field
  struct HaloReq {
    int level;
    std::function<void*(Rank&)> field;
    size_t esize;
    int wl, wr;
  };
  virtual void halo_many(std::vector<Rank*>& rs, const std::vector<HaloReq>& reqs, cudaStream_t s) {
    for (const HaloReq& q : reqs) halo(rs, q.level, q.field, q.esize, q.wl, q.wr, s);
  }
  // partials[0 .. n) of every rank summed elementwise into gparts of every
  // rank (each element has one non-zero contributor, so the sum is exact)
  virtual void allreduce(std::vector<Rank*>& rs, int n, cudaStream_t s) = 0;
  virtual bool local() const = 0;
};

// Several ranks in this process, all on the same device and stream.
struct LocalComm : Comm {
  const double** d_parts = nullptr;
  double** d_outs = nullptr;
  int n = 0;
  explicit LocalComm(std::vector<Rank*>& rs) {
    n = static_cast<int>(rs.size());
    std::vector<const double*> p(n);
    std::vector<double*> o(n);
    for (int i = 0; i < n; ++i) {
      p[i] = rs[i]->partials;
      o[i] = rs[i]->gparts;
    }
    CK(cudaMalloc(&d_parts, sizeof(double*) * n));
    CK(cudaMalloc(&d_outs, sizeof(double*) * n));
    CK(cudaMemcpy(d_parts, p.data(), sizeof(double*) * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_outs, o.data(), sizeof(double*) * n, cudaMemcpyHostToDevice));
  }
  ~LocalComm() override {
    cudaFree(d_parts);
    cudaFree(d_outs);
  }
  bool local() const override { return true; }
  void halo(std::vector<Rank*>& rs, int level, const std::function<void*(Rank&)>& field, size_t esize, int wl,
            int wr, cudaStream_t s) override {
    for (size_t i = 0; i < rs.size(); ++i) {
      Rank& me = *rs[i];
      const Grid& g = me.lev[level].g;
      const size_t col = esize * g.P;
      char* mine = static_cast<char*>(field(me));
      if (i > 0 && wl > 0) {
        Rank& L = *rs[i - 1];
        const Grid& gl = L.lev[level].g;
        char* src = static_cast<char*>(field(L)) + (gl.ncol + kGX - wl) * esize * gl.P;
        CK(cudaMemcpyAsync(mine + (kGX - wl) * col, src, wl * col, cudaMemcpyDeviceToDevice, s));
      }
      if (i + 1 < rs.size() && wr > 0) {
        Rank& R = *rs[i + 1];
        char* src = static_cast<char*>(field(R)) + kGX * esize * R.lev[level].g.P;
        CK(cudaMemcpyAsync(mine + (kGX + g.ncol) * col, src, wr * col, cudaMemcpyDeviceToDevice, s));
      }
    }
  }
  void gather_columns(std::vector<Rank*>& rs, int level, const std::function<void*(Rank&)>& field, size_t esize,
                      long plane_stride, int planes, const std::vector<int>& X0, const std::vector<int>& ncol,
                      cudaStream_t s) override {
    for (size_t src = 0; src < rs.size(); ++src) {
      const long P = rs[src]->lev[level].g.P;
      for (size_t dst = 0; dst < rs.size(); ++dst) {
        if (dst == src) continue;
        for (int k = 0; k < planes; ++k) {
          const size_t off = (k * plane_stride + static_cast<long>(X0[src] + kGX) * P) * esize;
          CK(cudaMemcpyAsync(static_cast<char*>(field(*rs[dst])) + off, static_cast<char*>(field(*rs[src])) + off,
                             ncol[src] * P * esize, cudaMemcpyDeviceToDevice, s));
        }
      }
    }
  }
  void allreduce(std::vector<Rank*>&, int len, cudaStream_t s) override {
    k_sum_parts<<<(len + 255) / 256, 256, 0, s>>>(d_parts, n, d_outs, len);
    CKL();
  }
};

// One rank per process, NCCL over NVLink / NVSwitch.
struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  NcclComm(int nranks_, int rank_, const void* id) : rank(rank_), nranks(nranks_) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    NK(nccl().commInitRank(&comm, nranks, uid, rank));
  }
  ~NcclComm() override {
    if (comm) nccl().commDestroy(comm);
  }
  bool local() const override { return false; }
  void halo(std::vector<Rank*>& rs, int level, const std::function<void*(Rank&)>& field, size_t esize, int wl,
            int wr, cudaStream_t s) override {
    NK(nccl().groupStart());
    halo_ops(rs, level, field, esize, wl, wr, s);
    NK(nccl().groupEnd());
  }
  void halo_many(std::vector<Rank*>& rs, const std::vector<HaloReq>& reqs, cudaStream_t s) override {
    NK(nccl().groupStart());
    for (const HaloReq& q : reqs) halo_ops(rs, q.level, q.field, q.esize, q.wl, q.wr, s);
    NK(nccl().groupEnd());
  }
  // the sends and receives of one exchange (inside a group); both sides issue
  // them in the same order, which is how NCCL pairs several messages between
  // the same two ranks within a group
  void halo_ops(std::vector<Rank*>& rs, int level, const std::function<void*(Rank&)>& field, size_t esize, int wl,
                int wr, cudaStream_t s) {
    Rank& me = *rs[0];
    const Grid& g = me.lev[level].g;
    const size_t col = esize * g.P;
    char* mine = static_cast<char*>(field(me));
    if (rank > 0) {
      // my first wr columns to the left neighbour's right ghost; its last wl to my left ghost
      if (wr > 0) NK(nccl().send(mine + kGX * col, wr * col, ncclChar, rank - 1, comm, s));
      if (wl > 0) NK(nccl().recv(mine + (kGX - wl) * col, wl * col, ncclChar, rank - 1, comm, s));
    }
    if (rank + 1 < nranks) {
      if (wl > 0) NK(nccl().send(mine + (g.ncol + kGX - wl) * col, wl * col, ncclChar, rank + 1, comm, s));
      if (wr > 0) NK(nccl().recv(mine + (kGX + g.ncol) * col, wr * col, ncclChar, rank + 1, comm, s));
    }
  }
  void gather_columns(std::vector<Rank*>& rs, int level, const std::function<void*(Rank&)>& field, size_t esize,
                      long plane_stride, int planes, const std::vector<int>& X0, const std::vector<int>& ncol,
                      cudaStream_t s) override {
    Rank& me = *rs[0];
    const long P = me.lev[level].g.P;
    char* buf = static_cast<char*>(field(me));
    // The partition gives every rank the same column count but the last one
    // (which also holds column nx): one in-place all-gather of that common
    // count per plane, plus one broadcast of the last rank's extra columns.
    // Any other layout: one broadcast per rank and plane.
    const int cmin = ncol[0];
    bool uniform = nccl().allGather != nullptr && ncol[nranks - 1] >= cmin;
    for (int r = 0; r < nranks; ++r)
      uniform = uniform && X0[r] == X0[0] + r * cmin && (r == nranks - 1 || ncol[r] == cmin);
    NK(nccl().groupStart());
    for (int k = 0; k < planes; ++k) {
      char* p0 = buf + (k * plane_stride + static_cast<long>(X0[0] + kGX) * P) * esize;
      if (uniform) {
        const size_t cnt = static_cast<size_t>(cmin) * P * esize;
        NK(nccl().allGather(p0 + rank * cnt, p0, cnt, ncclChar, comm, s));
        const int extra = ncol[nranks - 1] - cmin;
        if (extra > 0) {
          char* pe = p0 + static_cast<size_t>(nranks) * cnt;
          NK(nccl().broadcast(pe, pe, static_cast<size_t>(extra) * P * esize, ncclChar, nranks - 1, comm, s));
        }
      } else {
        for (int src = 0; src < nranks; ++src) {
          char* p = buf + (k * plane_stride + static_cast<long>(X0[src] + kGX) * P) * esize;
          NK(nccl().broadcast(p, p, ncol[src] * P * esize, ncclChar, src, comm, s));
        }
      }
    }
    NK(nccl().groupEnd());
  }
  void allreduce(std::vector<Rank*>& rs, int len, cudaStream_t s) override {
    NK(nccl().allReduce(rs[0]->partials, rs[0]->gparts, len, ncclDouble, ncclSum, comm, s));
  }
};

}  // namespace tmgi

// --------------------------------------------------------------- handle -----

struct tmg_gpu_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  int nx = 0, ny = 0, nc = 0;
  int nranks = 1;  // global
  // the slab machinery (partials all-reduced, ghost exchanges, replicated
  // coarse levels) is on: several ranks, or an NCCL communicator of any size
  // (a one-rank NCCL handle runs every exchange through NCCL)
  bool distributed = false;
  int rep = 0;     // levels 0..rep are replicated on every rank
  std::vector<int> xpart;  // fine node-column partition, nranks + 1 entries
  std::vector<std::unique_ptr<Rank>> own;
  std::vector<Rank*> ranks;  // ranks driven by this process
  std::unique_ptr<Comm> comm;
  // several ranks in this process: one stream per rank, forked from and
  // joined back into `stream` around every pass (for_ranks)
  std::vector<cudaStream_t> rstreams;
  cudaEvent_t fork_ev = nullptr;
  std::vector<cudaEvent_t> join_ev;
  double nu = 0.3;
  double ke[64];
  bool have_problem = false, have_moduli = false, have_setup = false, have_solution = false;
  double omega = 0.6;
  // captured PCG iterations: graph[k] serves iterations with (it-1)&1 == k;
  // with the fused update (pre >= 2) iteration 1 has its own graph
  // (graph[2]) and graph[k] opens by finishing iteration it-1
  cudaGraphExec_t graph[3] = {nullptr, nullptr, nullptr};
  long graph_kernels[3] = {0, 0, 0};
  // kernels before the conditional stopping test (all of them without one)
  long graph_head_kernels[3] = {0, 0, 0};
  // device-side stopping test between the fused update and the rest of an
  // iteration (TMG_NO_COND_NODES=1 turns it off, for A/B timing)
  bool cond_nodes = true;
  // the whole PCG loop as one graph with a conditional WHILE node (fused
  // scheme, conditional nodes on); the host launches it once per solve
  // (TMG_NO_DEVICE_LOOP=1 keeps the per-iteration host loop)
  bool device_loop = true;
  // NCCL handles: conditional graph nodes (device-side stopping test and the
  // one-graph loop) with the collectives inside their bodies. Every rank
  // holds bitwise the same PCG scalars, so all take the same branches and
  // issue the same collectives; opt-in (TMG_NCCL_COND_NODES=1) because only a
  // one-rank communicator can be exercised on a one-GPU box
  bool nccl_cond = false;
  // banded coarsest Cholesky (TMG_DENSE_COARSE_FACTOR=1: the dense kernel)
  bool band_factor = true;
  cudaGraphExec_t loop = nullptr;
  long loop_first_kernels = 0, loop_head_kernels = 0, loop_rest_kernels = 0;
  int g_gamma = -1, g_pre = -1, g_post = -1;
  // omega the graphs were captured with: it is a by-value kernel argument
  // (fixed when the operators are built, solvers.cpp:471), so a setup with a
  // new omega re-captures
  double g_omega = -1.0;
  bool g_fused = false;
  // node columns per tile of the fine-level reductions (red_tiles)
  int red_tx = 64;
  // coarse levels at least this large use the two-stage kernels
  // (TMG_SMARCH_MIN_NODES overrides it, for tests on small meshes)
  long smarch_min_nodes = kSMinNodes;
  // coarse levels up to this many nodes run the V(2,2) halves as shared-memory
  // tiles instead of marching kernels (tmg_stile.cuh)
  long stile_max_nodes = kTileMaxNodes;
  // tile levels up to these sizes (nodes) take the 2- / 4-coarse-node tiles
  // instead of the 8-node ones (TMG_STILE_TC2_NODES / TMG_STILE_TC4_NODES)
  long stile_tc1_nodes = 0, stile_tc2_nodes = kTileTC2Nodes, stile_tc4_nodes = kTileTC4Nodes;
  // programmatic dependent launch of the V-cycle-bottom kernels (TMG_NO_PDL=1: plain launches)
  bool pdl = true;
  // two-stage coarse kernels with stage A and stage B on separate warps
  // (tmg_smarch2.cuh; TMG_SMARCH_LOCKSTEP=1 runs the lockstep k_smarch)
  bool smarch_split = true;
  // pipelined solves: the copy stream and its hand-off events (staged[k]:
  // slot k's inputs landed; consumed[k]: slot k copied into the resident
  // arrays; solved: the solution's staging copy is written; downloaded: it
  // reached the host)
  cudaStream_t cstream = nullptr;
  cudaEvent_t staged[2] = {nullptr, nullptr}, consumed[2] = {nullptr, nullptr};
  cudaEvent_t solved = nullptr, downloaded = nullptr;
  bool staged_ok[2] = {false, false};
  // instrumentation
  long launches = 0;
  bool capturing = false;
  long capture_kernels = 0;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t uev[8] = {};
  double last_setup_ms = 0.0, last_pcg_ms = 0.0;
  double last_oc_ms = 0.0;  // device time of the last OC exchange
  int last_oc_steps = 0;    // its bisection steps
  std::string err;
  int err_row = -1;

  bool multi() const { return distributed; }
  bool dist(int l) const { return distributed && l > rep; }
  void count(long k = 1) {
    if (capturing) capture_kernels += k;
    else launches += k;
  }
};

namespace {

using H = tmg_gpu_handle;

// ------------------------------------------------------------- geometry ----

// Node columns per tile of the fine-level reductions: the marching kernels'
// strip width for the whole fine level (strip_tx below, the same formula),
// rounded up to a power of two. It depends on the global mesh only, so every
// partition tiles the fine level identically.
// Strip width of the fine marching passes: the power of two in [1, 64]
// minimising waves x (a*tx + 3) column steps for a nominal 3 resident CTAs on
// each of 148 SMs (ties to the wider strip). On c1-c4 it is the width the
// passes used before (8-64); meshes of ~64^2 get 1-column strips, whose
// passes are 4 column steps long instead of 11.
// nominal resident CTAs per SM of the strip-width model (TMG_STRIP_SLOTS
// overrides it; read once per process, so every handle tiles alike)
long strip_slots_per_sm() {
  static const long v = [] {
    const char* e = std::getenv("TMG_STRIP_SLOTS");
    return e ? std::max(1L, std::atol(e)) : 3L;
  }();
  return v;
}
int pow2_strip(long rows_tiles, long cols, int a) {
  const long slots = strip_slots_per_sm() * 148;
  int best = 64;
  long best_cost = -1;
  for (int tx = 64; tx >= 1; tx /= 2) {
    const long ctas = rows_tiles * ((cols + tx - 1) / tx);
    const long cost = ((ctas + slots - 1) / slots) * (a * tx + 3);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = tx;
    }
  }
  // A grid that still takes two or more waves but would fit the device in
  // one at twice the strip width (four resident CTAs per SM, the fine passes'
  // measured occupancy) takes the single wave: its second wave's ring fill and
  // launch cost more than the longer strips on L2-resident meshes (c3 mesh
  // 1024^2: 8 -> 16 columns, -3 % per PCG iteration). Wider single-wave
  // strips (c2: 16 -> 64) measured slower. TMG_STRIP_ONE_WAVE=0 turns it off.
  static const bool one_wave = [] {
    const char* e = std::getenv("TMG_STRIP_ONE_WAVE");
    return !e || std::atoi(e) != 0;
  }();
  const long ctas = rows_tiles * ((cols + best - 1) / best);
  const long ctas2 = rows_tiles * ((cols + 2 * best - 1) / (2 * best));
  if (one_wave && best < 64 && ctas > 4L * 148 && ctas2 <= 4L * 148) best *= 2;
  return best;
}

int red_tx_of(int nx, int ny) { return pow2_strip((ny + 1L + kRedRows - 1) / kRedRows, nx + 1L, 1); }

// Fine node-column partition: boundaries multiples of 2^(nc - rep), so every
// distributed level has even slab boundaries, and of the reduction tile
// width, so no reduction tile straddles two ranks (both powers of two).
int partition_gran(int nx, int ny, int nc, int rep) {
  return std::max(1 << (nc - rep), red_tx_of(nx, ny));
}
std::vector<int> partition(int nx, int ny, int nc, int rep, int nranks) {
  std::vector<int> xp(nranks + 1, 0);
  const long gran = partition_gran(nx, ny, nc, rep);
  for (int r = 1; r < nranks; ++r) {
    const double target = static_cast<double>(r) * (nx + 1) / nranks;
    xp[r] = static_cast<int>(std::llround(target / gran) * gran);
  }
  xp[nranks] = nx + 1;
  return xp;
}

// highest replicated level: distribute level l while every rank owns >= 16
// node columns of it
int auto_rep(int nx, int nc, int nranks) {
  int rep = nc;
  for (int l = nc; l >= 1; --l) {
    const int cols = (nx >> (nc - l)) + 1;
    if (cols / nranks >= 16) rep = l - 1;
    else break;
  }
  return rep;
}

// owned node columns of rank r at level l (distributed-level geometry)
void slab_cols(const H* h, int r, int l, int& x0, int& n) {
  const int s = h->nc - l;
  const int nxl = h->nx >> s;
  x0 = h->xpart[r] >> s;
  const int x1 = (r + 1 == h->nranks) ? nxl + 1 : (h->xpart[r + 1] >> s);
  n = x1 - x0;
}

// A replicated level seen as the slab rank r's distributed parent level
// writes / reads: same pitch, base offset X0 columns.
Grid slab_view(const H* h, const Rank& R, int l, long& off) {
  int x0, n;
  slab_cols(h, R.index, l, x0, n);
  Grid g = R.lev[l].g;
  g.x0 = x0;
  g.ncol = n;
  off = static_cast<long>(x0) * g.P;
  return g;
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

// host vector in reference layout <-> owned columns of the level on a rank
void upload_nodes(cudaStream_t s, double2* d, const double* host, const Grid& g) {
  CK(cudaMemcpy2DAsync(d + g.idx(0, 0), sizeof(double2) * g.P, host + 2L * g.x0 * (g.ny + 1),
                       sizeof(double2) * (g.ny + 1), sizeof(double2) * (g.ny + 1), g.ncol, cudaMemcpyHostToDevice,
                       s));
}

void download_nodes(cudaStream_t s, double* host, const double2* d, const Grid& g) {
  CK(cudaMemcpy2DAsync(host + 2L * g.x0 * (g.ny + 1), sizeof(double2) * (g.ny + 1), d + g.idx(0, 0),
                       sizeof(double2) * g.P, sizeof(double2) * (g.ny + 1), g.ncol, cudaMemcpyDeviceToHost, s));
}

void check_level(H* h, int level) {
  if (level < 0 || level > h->nc) {
    fail(TMG_ERR_DIMENSION, "level " + std::to_string(level) + " outside [0, " + std::to_string(h->nc) + "]");
  }
}

void need_setup(H* h) {
  if (!h->have_setup) fail(TMG_ERR_DIMENSION, "multigrid operators not built (call tmg_gpu_set_moduli)");
}

void need_single(H* h, const char* what) {
  if (h->multi()) fail(TMG_ERR_CONFIG, std::string(what) + " is available on single-rank handles only");
}

void free_rank(Rank& R) {
  for (Level& L : R.lev) {
    cudaFree(L.u[0]);
    cudaFree(L.u[1]);
    cudaFree(L.res);
    cudaFree(L.S);
    if (&L != &R.lev.back()) cudaFree(L.f);
  }
  for (void* p : {static_cast<void*>(R.E), static_cast<void*>(R.M), static_cast<void*>(R.A0),
                  static_cast<void*>(R.LiT), static_cast<void*>(R.Ainv), static_cast<void*>(R.bad_row),
                  static_cast<void*>(R.x), static_cast<void*>(R.r), static_cast<void*>(R.r2), static_cast<void*>(R.ap),
                  static_cast<void*>(R.b), static_cast<void*>(R.x0), static_cast<void*>(R.pbuf[0]),
                  static_cast<void*>(R.pbuf[1]), static_cast<void*>(R.partials), static_cast<void*>(R.gparts),
                  static_cast<void*>(R.ticket),
                  static_cast<void*>(R.st), static_cast<void*>(R.scal), static_cast<void*>(R.dense),
                  static_cast<void*>(R.aux), static_cast<void*>(R.aux2), static_cast<void*>(R.ocbuf),
                  static_cast<void*>(R.Es[0]), static_cast<void*>(R.Es[1]), static_cast<void*>(R.bs[0]),
                  static_cast<void*>(R.bs[1]), static_cast<void*>(R.us)})
    cudaFree(p);
  if (R.hm) cudaFreeHost(R.hm);
  if (R.lrec) cudaFreeHost(R.lrec);
  if (R.rbk) cudaFreeHost(R.rbk);
  if (R.hist) cudaFreeHost(R.hist);
  if (R.scal_host) cudaFreeHost(R.scal_host);
}

void free_handle(H* h) {
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (cudaGraphExec_t gx : h->graph)
    if (gx) cudaGraphExecDestroy(gx);
  if (h->loop) cudaGraphExecDestroy(h->loop);
  h->comm.reset();
  for (Rank* R : h->ranks) free_rank(*R);
  for (cudaStream_t s : h->rstreams) cudaStreamDestroy(s);
  for (cudaEvent_t e : h->join_ev) cudaEventDestroy(e);
  if (h->fork_ev) cudaEventDestroy(h->fork_ev);
  for (cudaEvent_t e : h->ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : h->uev)
    if (e) cudaEventDestroy(e);
  if (h->cstream) {
    cudaStreamSynchronize(h->cstream);
    for (cudaEvent_t e : {h->staged[0], h->staged[1], h->consumed[0], h->consumed[1], h->solved, h->downloaded})
      if (e) cudaEventDestroy(e);
    cudaStreamDestroy(h->cstream);
  }
  if (h->stream) cudaStreamDestroy(h->stream);
}

// tile geometry of the fine-level reductions on a rank's slab g
RedTiles red_tiles(const H* h, const Grid& g) {
  RedTiles rt{};
  rt.tx = h->red_tx;
  rt.ctile0 = g.x0 / h->red_tx;
  const int ty = (h->ny + kRedRows) / kRedRows;  // ceil((ny + 1) / kRedRows)
  rt.nparts = ty * ((h->nx + 1 + h->red_tx - 1) / h->red_tx);
  return rt;
}

void alloc_rank(H* h, Rank& R) {
  cudaStream_t s = h->stream;
  R.nx = h->nx;
  R.ny = h->ny;
  R.nc = h->nc;
  R.lev.resize(h->nc + 1);
  for (int l = 0; l <= h->nc; ++l) {
    Level& L = R.lev[l];
    const int sh = h->nc - l;
    const int nxl = h->nx >> sh, nyl = h->ny >> sh;
    L.dist = h->dist(l);
    int x0 = 0, n = nxl + 1;
    if (L.dist) slab_cols(h, R.index, l, x0, n);
    L.g = make_grid(nxl, nyl, x0, n);
    L.ndof = 2L * (nxl + 1) * (nyl + 1);
    const size_t vb = sizeof(double2) * (L.g.size + kSlackNodes);
    for (double2** v : {&L.u[0], &L.u[1], &L.res}) {
      CK(cudaMalloc(v, vb));
      CK(cudaMemsetAsync(*v, 0, vb, s));
    }
    if (l < h->nc) {
      CK(cudaMalloc(&L.f, vb));
      CK(cudaMemsetAsync(L.f, 0, vb, s));
      const size_t sb = sizeof(double) * (kStencilPlanes * L.g.size + kSlackNodes);
      CK(cudaMalloc(&L.S, sb));
      CK(cudaMemsetAsync(L.S, 0, sb, s));
    }
  }
  Level& F = R.fine();
  const size_t vb = sizeof(double2) * (F.g.size + kSlackNodes);
  for (double2** v : {&R.x, &R.r, &R.r2, &R.pbuf[0], &R.pbuf[1], &R.ap, &R.b, &R.x0}) {
    CK(cudaMalloc(v, vb));
    CK(cudaMemsetAsync(*v, 0, vb, s));
  }
  F.f = R.r;  // the finest cycle smooths against the PCG residual
  CK(cudaMalloc(&R.E, sizeof(double) * (F.g.size + kSlackNodes)));
  CK(cudaMemsetAsync(R.E, 0, sizeof(double) * (F.g.size + kSlackNodes), s));
  CK(cudaMalloc(&R.M, F.g.size + kSlackNodes));
  CK(cudaMemsetAsync(R.M, 0, F.g.size + kSlackNodes, s));
  const Grid& g0 = R.lev[0].g;
  R.n0 = 2 * (g0.nx + 1) * (g0.ny + 1);
  const size_t n0sq = sizeof(double) * R.n0 * R.n0;
  // k_coarse_solve stages the right-hand side in shared memory (one limit for every handle)
  CK(cudaFuncSetAttribute(k_coarse_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          static_cast<int>(sizeof(double) * kCoarsestMaxDofs)));
  CK(cudaMalloc(&R.A0, n0sq));
  CK(cudaMalloc(&R.LiT, n0sq));
  CK(cudaMalloc(&R.Ainv, n0sq));
  CK(cudaMalloc(&R.bad_row, sizeof(int)));
  const dim3 ng = node_grid(F.g);
  // reduction partials: the global tile array (zero outside this rank's
  // tiles, which it never writes), or one per CTA of a node-grid launch
  const long nparts = std::max(static_cast<long>(ng.x) * ng.y, static_cast<long>(red_tiles(h, F.g).nparts));
  CK(cudaMalloc(&R.partials, sizeof(double) * nparts));
  CK(cudaMemsetAsync(R.partials, 0, sizeof(double) * nparts, s));
  if (h->multi()) {
    CK(cudaMalloc(&R.gparts, sizeof(double) * nparts));
    CK(cudaMemsetAsync(R.gparts, 0, sizeof(double) * nparts, s));
  }
  CK(cudaMalloc(&R.ticket, sizeof(unsigned)));
  CK(cudaMemsetAsync(R.ticket, 0, sizeof(unsigned), s));
  R.rticket = h->multi() ? nullptr : R.ticket;
  CK(cudaMalloc(&R.st, sizeof(PcgState)));
  CK(cudaMemsetAsync(R.st, 0, sizeof(PcgState), s));
  CK(cudaMalloc(&R.scal, 4 * sizeof(double)));
  CK(cudaMemsetAsync(R.scal, 0, 4 * sizeof(double), s));
  CK(cudaHostAlloc(&R.hm, sizeof(HostMirror), cudaHostAllocMapped));
  std::memset(R.hm, 0, sizeof(HostMirror));
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&R.hm_dev), R.hm, 0));
  CK(cudaHostAlloc(&R.scal_host, 4 * sizeof(double), cudaHostAllocDefault));
  CK(cudaHostAlloc(&R.rbk, sizeof(Readback), cudaHostAllocMapped));
  std::memset(R.rbk, 0, sizeof(Readback));
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&R.rbk_dev), R.rbk, 0));
  CK(cudaHostAlloc(&R.lrec, sizeof(LoopRecord), cudaHostAllocMapped));
  std::memset(R.lrec, 0, sizeof(LoopRecord));
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&R.lrec_dev), R.lrec, 0));
}

// ------------------------------------------------------------- exchanges ---

void halo_vec(H* h, int l, const std::function<double2*(Rank&)>& field, int wl = 1, int wr = 1) {
  if (!h->dist(l)) return;
  h->comm->halo(h->ranks, l, [&](Rank& R) -> void* { return field(R); }, sizeof(double2), wl, wr, h->stream);
}
// several vector exchanges at one point (level, field, wl, wr each): one
// NCCL group; levels that are not distributed are skipped
struct VecHalo {
  int level;
  std::function<double2*(Rank&)> field;
  int wl, wr;
};
void halo_vecs(H* h, const std::vector<VecHalo>& hs) {
  std::vector<Comm::HaloReq> reqs;
  for (const VecHalo& v : hs) {
    if (!h->dist(v.level)) continue;
    auto f = v.field;
    reqs.push_back({v.level, [f](Rank& R) -> void* { return f(R); }, sizeof(double2), v.wl, v.wr});
  }
  if (!reqs.empty()) h->comm->halo_many(h->ranks, reqs, h->stream);
}

// replicated level l: every rank's owned columns to all ranks
void gather_level(H* h, int l, const std::function<void*(Rank&)>& field, size_t esize, long plane_stride,
                  int planes) {
  std::vector<int> X0(h->nranks), n(h->nranks);
  for (int r = 0; r < h->nranks; ++r) slab_cols(h, r, l, X0[r], n[r]);
  h->comm->gather_columns(h->ranks, l, field, esize, plane_stride, planes, X0, n, h->stream);
}

// Per-rank work of one pass. With several ranks in this process (LocalComm)
// each rank's launches go on its own stream between a fork from and a join
// into the handle's stream, so the slabs run concurrently on the device as
// they would on N GPUs and the captured graphs hold N parallel branches; the
// exchanges (halos, all-reduce, gathers) stay on the handle's stream between
// the joins. One rank: a plain call.
template <class F>
void for_ranks(H* h, F&& fn) {
  if (h->rstreams.empty()) {
    for (Rank* R : h->ranks) fn(*R);
    return;
  }
  cudaStream_t main = h->stream;
  CK(cudaEventRecord(h->fork_ev, main));
  for (size_t i = 0; i < h->ranks.size(); ++i) {
    CK(cudaStreamWaitEvent(h->rstreams[i], h->fork_ev, 0));
    h->stream = h->rstreams[i];
    try {
      fn(*h->ranks[i]);
    } catch (...) {
      h->stream = main;
      throw;
    }
    h->stream = main;
    CK(cudaEventRecord(h->join_ev[i], h->rstreams[i]));
  }
  for (cudaEvent_t e : h->join_ev) CK(cudaStreamWaitEvent(main, e, 0));
}

// ---------------------------------------------------------- reductions ----

// Launch a reduction on every rank: single rank -> the kernel's last block
// applies `op`; several ranks -> the kernels only write their tiles'
// partials (rticket is null), the partial arrays are all-reduced and every
// rank finishes the same array in the same fixed order (k_finish), so the
// scalars are bitwise those of the single-rank solve.
void reduce(H* h, RedOp op, const std::function<void(Rank&, RedOp, double*)>& launch, bool want_out = false) {
  if (!h->multi()) {
    Rank& R = *h->ranks[0];
    launch(R, op, want_out ? R.scal : nullptr);
    return;
  }
  for_ranks(h, [&](Rank& R) { launch(R, op, nullptr); });
  const int n = red_tiles(h, h->ranks[0]->fine().g).nparts;
  h->comm->allreduce(h->ranks, n, h->stream);
  for (Rank* R : h->ranks) {
    k_finish<<<1, 128, 0, h->stream>>>(R->gparts, n, op, R->st, R->hm_dev, want_out ? R->scal : nullptr);
    CKL();
  }
  h->count(static_cast<long>(h->ranks.size()) + (h->comm->local() ? 1 : 0));
}

// ------------------------------------------------------------ launches ----

// Output columns per fine-level marching CTA: short strips (many waves of
// 3-5 resident CTAs per SM) balance best; measured on c4, one-wave long
// strips ran 10-25% slower for these kernels.
int strip_tx(long rows_tiles, long cols, int a = 1) { return pow2_strip(rows_tiles, cols, a); }

// Resident CTAs of one marching kernel on the whole device (occupancy x SMs;
// cached per kernel: every handle of a process runs on the same GPU type).
int device_slots(const void* fn, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<const void*, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(fn);
  if (it != cache.end()) return it->second;
  int dev = 0, sms = 0, per_sm = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem));
  const int slots = std::max(1, sms * per_sm);
  cache.emplace(fn, slots);
  return slots;
}

// Output columns per coarse-level (two-stage) marching CTA. A CTA marching tx columns streams
// a*tx + b ring entries (b: halo columns + pipeline fill). With `slots`
// resident CTAs the grid of rows_tiles x ceil(cols/tx) CTAs runs in w waves;
// pick the w and tx minimising w * (a*tx + b), so the last wave is never a
// few stragglers (a 5.02-wave grid costs 6 full waves).
int march_tx(long rows_tiles, long cols, int slots, int a, int b, bool even = false) {
  long best_tx = cols, best_cost = -1;
  for (long w = 1; w <= 512; ++w) {
    const long nct = std::min<long>(cols, w * slots / rows_tiles);
    if (nct < 1) continue;
    long tx = (cols + nct - 1) / nct;
    if (even) tx = (tx + 1) & ~1L;
    const long waves = (rows_tiles * ((cols + tx - 1) / tx) + slots - 1) / slots;
    const long cost = waves * (a * tx + b);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best_tx = tx;
    }
    if (nct == cols) break;
  }
  return static_cast<int>(std::max<long>(1, best_tx));
}

MarchArgs march_args(H* h, Rank& R, const double2* u) {
  MarchArgs a{};
  a.g = R.fine().g;
  a.u = u;
  a.E = R.E;
  a.M = R.M;
  a.omega = h->omega;
  a.partials = R.partials;
  a.ticket = R.rticket;
  a.rt = red_tiles(h, R.fine().g);
  a.rop = kRedNone;
  a.st = R.st;
  a.hm = R.hm_dev;
  return a;
}

// Grid + base offset of the coarse level l-1 as level l's kernels address it
Grid coarse_of(H* h, Rank& R, int l, long& off) {
  off = 0;
  if (h->dist(l) && !h->dist(l - 1)) return slab_view(h, R, l - 1, off);
  return R.lev[l - 1].g;
}

template <class Stage, bool RED>
void launch_march(H* h, MarchArgs a) {
  dim3 grid;
  const size_t sm = static_cast<size_t>(Stage::kSlot) * RingOf<Stage>::value;
  if constexpr (Stage::kRow0 == -1) {  // restriction: tiles of coarse rows / columns
    const long ty = (a.gc.ny + 1 + Stage::kOwned / 2 - 1) / (Stage::kOwned / 2);
    a.tx = strip_tx(ty, a.gc.ncol, 2);
    grid = dim3(ty, (a.gc.ncol + a.tx - 1) / a.tx);
  } else {
    const long ty = (a.g.ny + 1 + Stage::kOwned - 1) / Stage::kOwned;
    // reducing stages march the reduction tiles (global geometry)
    a.tx = RED ? h->red_tx : strip_tx(ty, a.g.ncol);
    grid = dim3(ty, (a.g.ncol + a.tx - 1) / a.tx);
  }
  k_march<Stage, RED><<<grid, kMarchThreads, sm, h->stream>>>(a);
  CKL();
  h->count();
}

template <class F>
void with_op(Rank& R, int l, F&& fn) {
  if (l == R.nc) fn(R.fine_op());
  else fn(R.stencil_op(l));
}

void apply_level(H* h, Rank& R, int l, const double2* x, double2* y) {
  const Level& L = R.lev[l];
  if (l == R.nc) {
    MarchArgs a = march_args(h, R, x);
    a.out0 = y;
    launch_march<StApply<false>, false>(h, a);
    return;
  }
  with_op(R, l, [&](auto op) {
    k_apply<decltype(op), false><<<node_grid(L.g), node_block(), 0, h->stream>>>(
        op, L.g, x, y, nullptr, nullptr, kRedNone, nullptr, nullptr, nullptr);
  });
  CKL();
  h->count();
}

// y = A x and x.y on every rank (reduction op `op` updates the PCG scalars)
void apply_dot_fine(H* h, const std::function<const double2*(Rank&)>& x,
                    const std::function<double2*(Rank&)>& y, RedOp op, bool want_out) {
  reduce(
      h, op,
      [&](Rank& R, RedOp rop, double* out) {
        MarchArgs a = march_args(h, R, x(R));
        a.out0 = y(R);
        a.rop = rop;
        a.red_out = out;
        launch_march<StApply<true>, true>(h, a);
      },
      want_out);
}

void sweep_level(H* h, Rank& R, int l, bool zero, const double2* xin, double2* xout, const double2* f) {
  const Level& L = R.lev[l];
  if (l == R.nc && !zero) {
    MarchArgs a = march_args(h, R, xin);
    a.f = f;
    a.out0 = xout;
    launch_march<StSweep<false>, false>(h, a);
    return;
  }
  with_op(R, l, [&](auto op) {
    if (zero)
      k_sweep<decltype(op), true><<<node_grid(L.g), node_block(), 0, h->stream>>>(op, L.g, xin, xout, f, h->omega);
    else
      k_sweep<decltype(op), false><<<node_grid(L.g), node_block(), 0, h->stream>>>(op, L.g, xin, xout, f, h->omega);
  });
  CKL();
  h->count();
}

void residual_level(H* h, Rank& R, int l, const double2* x, const double2* f, double2* r) {
  const Level& L = R.lev[l];
  if (l == R.nc) {
    MarchArgs a = march_args(h, R, x);
    a.f = f;
    a.out0 = r;
    launch_march<StResidual, false>(h, a);
    return;
  }
  with_op(R, l, [&](auto op) {
    k_residual<decltype(op)><<<node_grid(L.g), node_block(), 0, h->stream>>>(op, L.g, x, f, r);
  });
  CKL();
  h->count();
}

void restrict_level(H* h, Rank& R, int l, const double2* r, double2* fc) {
  long off;
  const Grid cg = coarse_of(h, R, l, off);
  k_restrict<<<node_grid(cg), node_block(), 0, h->stream>>>(cg, R.lev[l].g, r, fc + off);
  CKL();
  h->count();
}

void prolong_level(H* h, Rank& R, int l, const double2* uc, double2* x, bool add) {
  long off;
  const Grid cg = coarse_of(h, R, l, off);
  const Grid& fg = R.lev[l].g;
  if (add) k_prolong<true><<<node_grid(fg), node_block(), 0, h->stream>>>(fg, cg, uc + off, x);
  else k_prolong<false><<<node_grid(fg), node_block(), 0, h->stream>>>(fg, cg, uc + off, x);
  CKL();
  h->count();
}

// Launch of a V-cycle-bottom kernel (tile kernels, coarsest solve) with
// programmatic stream serialization: it starts while its predecessor runs,
// stages its invariant inputs, and waits (griddepcontrol.wait) before reading
// what the predecessor writes; each such kernel releases its own dependent
// only after that wait, so at most one kernel runs ahead. Single-rank
// handles only: slab handles interleave event joins (LocalComm) or NCCL
// collectives (multi-rank NCCL never ran here) with the bottom kernels.
template <class... P, class... A>
void launch_dep(H* h, void (*kernel)(P...), dim3 grid, dim3 block, size_t smem, A&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = h->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (h->pdl && !h->distributed) ? 1 : 0;
  CK(cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...));
}

void coarse_solve(H* h, Rank& R, const double2* f, double2* u) {
  const int warps = R.n0 / 2, per_block = kCoarseSolveThreads / 32;
  launch_dep(h, k_coarse_solve, dim3((warps + per_block - 1) / per_block), dim3(kCoarseSolveThreads),
             sizeof(double) * R.n0, static_cast<const double*>(R.Ainv), R.n0, R.lev[0].g, f, u);
  CKL();
  h->count();
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// link-time libcuda dependency)
PFN_cuTensorMapEncodeTiled tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) fail(TMG_ERR_CUDA, "cuTensorMapEncodeTiled not available");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(p);
  }();
  return fn;
}

// the stencil planes of a level as a (padded row, storage column, plane)
// tensor; one box = kSRows rows of one column, all planes (tmg_smarch.cuh)
CUtensorMap stencil_tensor_map(const double* S, const Grid& g) {
  CUtensorMap m;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(g.P), static_cast<cuuint64_t>(g.size / g.P),
                              static_cast<cuuint64_t>(kStencilPlanes)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(g.P) * 8, static_cast<cuuint64_t>(g.size) * 8};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(kSBoxRows), 1, static_cast<cuuint32_t>(kStencilPlanes)};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = tensor_map_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(S), dims,
                                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(TMG_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return m;
}

// two-stage marching kernels of a coarse (stencil) level: DOWN writes x2 into
// `out` and f_c into the coarse rhs; UP prolongs u_c onto x2 and smooths twice
template <bool UP>
void launch_smarch(H* h, Rank& R, int l, const double2* x2, const double2* uc, double2* out, double2* fc) {
  SMarchArgs a{};
  a.g = R.lev[l].g;
  long off;
  a.gc = coarse_of(h, R, l, off);
  a.S = R.lev[l].S;
  a.tmS = stencil_tensor_map(a.S, a.g);
  a.f = R.lev[l].f;
  a.x2 = x2;
  a.uc = uc ? uc + off : nullptr;
  a.out = out;
  a.fc = fc ? fc + off : nullptr;
  a.omega = h->omega;
  dim3 grid;
  size_t sm;
  if (!UP) {
    sm = static_cast<size_t>(kSSlotDown) * s_stages<false>();
    const int slots = h->smarch_split
                          ? device_slots(reinterpret_cast<const void*>(k_smarch2<false>), kS2Threads, sm)
                          : device_slots(reinterpret_cast<const void*>(k_smarch<false>), kSThreads, sm);
    const long ty = (a.gc.ny + 1 + (kSY - 4) / 2 - 1) / ((kSY - 4) / 2);
    a.tx = march_tx(ty, a.gc.ncol, slots, 2, 7);
    grid = dim3(ty, (a.gc.ncol + a.tx - 1) / a.tx);
  } else {
    sm = static_cast<size_t>(kSSlotUp) * s_stages<true>();
    const int slots = h->smarch_split
                          ? device_slots(reinterpret_cast<const void*>(k_smarch2<true>), kS2Threads, sm)
                          : device_slots(reinterpret_cast<const void*>(k_smarch<true>), kSThreads, sm);
    const long ty = (a.g.ny + 1 + (kSY - 2) - 1) / (kSY - 2);
    // even: CTA column ranges start on even columns
    a.tx = march_tx(ty, a.g.ncol, slots, 1, 7, true);
    grid = dim3(ty, (a.g.ncol + a.tx - 1) / a.tx);
  }
  if (!h->dist(l) && static_cast<long>(a.g.nx + 1) * (a.g.ny + 1) <= h->stile_max_nodes) {
    // small level: one shared-memory tile per CTA (tmg_stile.cuh)
    const long nodes = static_cast<long>(a.g.nx + 1) * (a.g.ny + 1);
    auto tile = [&](auto tc) {
      constexpr int TC = decltype(tc)::value;
      const dim3 tg = UP ? dim3((a.g.ny + 2 * TC) / (2 * TC), (a.g.ncol + 2 * TC - 1) / (2 * TC))
                         : dim3((a.gc.ny + TC) / TC, (a.gc.ncol + TC - 1) / TC);
      launch_dep(h, k_stile<UP, TC>, tg, dim3(t_threads<TC>()), t_smem<UP, TC>(), a);
    };
    if (nodes <= h->stile_tc1_nodes) tile(std::integral_constant<int, 1>{});
    else if (nodes <= h->stile_tc2_nodes) tile(std::integral_constant<int, 2>{});
    else if (nodes <= h->stile_tc4_nodes) tile(std::integral_constant<int, 4>{});
    else tile(std::integral_constant<int, 8>{});
  } else if (h->smarch_split) {
    k_smarch2<UP><<<grid, kS2Threads, sm, h->stream>>>(a);
  } else {
    k_smarch<UP><<<grid, kSThreads, sm, h->stream>>>(a);
  }
  CKL();
  h->count();
}

// One gamma-cycle at level l on every rank in lockstep (mg_cycle,
// solvers.cpp:483-514). `zero` means the iterate is logically zero on entry
// (the reference zeroes u_coarse before the first visit, solvers.cpp:501, and
// pcgmg starts from z = 0, solvers.cpp:524); its buffer is then never read. At
// the finest level the passes are the fused marching stages (tmg_march.cuh);
// with `zr_op` set the last post-sweep also reduces z.r for PCG. Returns
// whether that reduction was fused. Distributed levels exchange one ghost
// column (two before the fused restriction) before every pass that reads
// neighbours; the finest replicated level is assembled from the ranks' owned
// columns after the restriction.
bool enqueue_cycle(H* h, int l, bool zero, int gamma, int pre, int post, RedOp zr_op = kRedNone,
                   int upd_k = -1, const std::function<void()>& after_update = nullptr) {
  auto& rs = h->ranks;
  if (l == 0) {
    for_ranks(h, [&](Rank& R) { coarse_solve(h, R, R.lev[0].f, R.lev[0].u[R.lev[0].cur]); });
    return false;
  }
  const bool fine = (l == h->nc);
  const bool dist = h->dist(l);
  const bool cdist = h->dist(l - 1);
  auto cur = [&](Rank& R) { return R.lev[l].u[R.lev[l].cur]; };
  auto nxt = [&](Rank& R) { return R.lev[l].u[R.lev[l].cur ^ 1]; };
  auto flip = [&] {
    for (Rank* R : rs) R->lev[l].cur ^= 1;
  };
  int s = 0;
  if (fine && zero && pre >= 2 && upd_k >= 0) {
    // finish the previous PCG iteration (x += alpha p, r = r_old - alpha Ap,
    // r.r) inside the first smoothing pass; r_old = rbuf(k^1) and A p carry
    // their halos, the new r = rbuf(k) gets its halo for the next iteration
    reduce(h, kRedRr, [&](Rank& R, RedOp rop, double* out) {
      MarchArgs a = march_args(h, R, nullptr);
      a.f = R.rbuf(upd_k ^ 1);
      a.u2 = R.ap;
      a.uc = R.pbuf[upd_k];
      a.out2 = R.x;
      a.out1 = R.rbuf(upd_k);
      a.out0 = nxt(R);
      a.rop = rop;
      a.red_out = out;
      launch_march<StSweep01U, true>(h, a);
    });
    halo_vec(h, l, [&](Rank& R) { return R.rbuf(upd_k); });
    flip();
    s = 2;
    zero = false;
    if (after_update) after_update();
  } else if (fine && zero && pre >= 2) {
    // the finest f (the PCG residual) already carries its halo
    for_ranks(h, [&](Rank& Rk) {
      Rank* R = &Rk;
      MarchArgs a = march_args(h, *R, nullptr);
      a.f = R->lev[l].f;
      a.out0 = nxt(*R);
      launch_march<StSweep01, false>(h, a);
    });
    flip();
    s = 2;
    zero = false;
  }
  bool restricted = false;
  // the two-stage kernels pay off once a level streams more than it waits
  // (decided on the global level size, so every partition runs the same kernels)
  const bool big = (static_cast<long>(rs[0]->lev[l].g.nx) + 1) * (rs[0]->lev[l].g.ny + 1) >= h->smarch_min_nodes;
  if (!fine && big && zero && pre == 2) {
    // coarse level: both pre-sweeps, the residual and the restriction in one
    // pass over the stencil (tmg_smarch.cuh)
    halo_vec(h, l, [&](Rank& R) { return R.lev[l].f; }, 3, 2);
    for_ranks(h, [&](Rank& R) { launch_smarch<false>(h, R, l, nullptr, nullptr, nxt(R), R.lev[l - 1].f); });
    flip();
    s = 2;
    zero = false;
    restricted = true;
  }
  for (; s < pre; ++s) {
    if (!zero) halo_vec(h, l, cur);
    for_ranks(h, [&](Rank& R) { sweep_level(h, R, l, zero, cur(R), nxt(R), R.lev[l].f); });
    flip();
    zero = false;
  }
  if (restricted) {
  } else if (zero) {
    halo_vec(h, l, [&](Rank& R) { return R.lev[l].f; });
    for_ranks(h, [&](Rank& R) { restrict_level(h, R, l, R.lev[l].f, R.lev[l - 1].f); });
  } else if (fine) {
    halo_vec(h, l, cur, 2, 1);
    for_ranks(h, [&](Rank& Rk) {
      Rank* R = &Rk;
      MarchArgs a = march_args(h, *R, cur(*R));
      long coff;
      a.gc = coarse_of(h, *R, l, coff);
      a.f = R->lev[l].f;
      a.out0 = R->lev[l - 1].f + coff;
      launch_march<StResidRestrict, false>(h, a);
    });
  } else {
    halo_vec(h, l, cur);
    for_ranks(h, [&](Rank& R) { residual_level(h, R, l, cur(R), R.lev[l].f, R.lev[l].res); });
    halo_vec(h, l, [&](Rank& R) { return R.lev[l].res; });
    for_ranks(h, [&](Rank& R) { restrict_level(h, R, l, R.lev[l].res, R.lev[l - 1].f); });
  }
  if (dist && !cdist) gather_level(h, l - 1, [&](Rank& R) -> void* { return R.lev[l - 1].f; }, sizeof(double2), 0, 1);
  const int visits = fine ? 1 : gamma;
  for (int t = 0; t < visits; ++t) enqueue_cycle(h, l - 1, t == 0, gamma, pre, post);
  auto ccur = [&](Rank& R) { return R.lev[l - 1].u[R.lev[l - 1].cur]; };
  // the two-stage UP pass prolongates onto two ghost columns on the right:
  // column ncol+1 interpolates coarse columns ncol/2 and ncol/2 + 1
  int p = 0;
  if (!fine && big && !zero && post == 2) {
    // coarse level: prolongation + both post-sweeps in one pass; its three
    // inputs' ghosts (coarse correction, iterate, rhs) in one exchange
    halo_vecs(h, {{l - 1, ccur, 1, 2}, {l, cur, 2, 2}, {l, [&](Rank& R) { return R.lev[l].f; }, 3, 2}});
    for_ranks(h, [&](Rank& R) { launch_smarch<true>(h, R, l, cur(R), ccur(R), nxt(R), nullptr); });
    flip();
    p = post;
  } else if (fine && !zero && post >= 1) {
    if (cdist) halo_vec(h, l - 1, ccur, 1, 2);
    for_ranks(h, [&](Rank& Rk) {
      Rank* R = &Rk;
      MarchArgs a = march_args(h, *R, cur(*R));
      long coff;
      a.gc = coarse_of(h, *R, l, coff);
      a.uc = ccur(*R) + coff;
      a.f = R->lev[l].f;
      a.out0 = nxt(*R);
      launch_march<StProlongSweep, false>(h, a);
    });
    flip();
    p = 1;
  } else {
    if (cdist) halo_vec(h, l - 1, ccur, 1, 2);
    for_ranks(h, [&](Rank& R) { prolong_level(h, R, l, ccur(R), cur(R), !zero); });
  }
  bool fused = false;
  for (; p < post; ++p) {
    halo_vec(h, l, cur);
    const bool last = (p == post - 1);
    if (fine && last && zr_op != kRedNone) {
      reduce(h, zr_op, [&](Rank& R, RedOp rop, double* out) {
        MarchArgs a = march_args(h, R, cur(R));
        a.f = R.lev[l].f;
        a.out0 = nxt(R);
        a.rop = rop;
        a.red_out = out;
        launch_march<StSweep<true>, true>(h, a);
      });
      fused = true;
    } else {
      for_ranks(h, [&](Rank& R) { sweep_level(h, R, l, false, cur(R), nxt(R), R.lev[l].f); });
    }
    flip();
  }
  return fused;
}

int red_grid(long n2) {
  long b = (n2 + kRedThreads - 1) / kRedThreads;
  return static_cast<int>(b < kRedBlocks ? (b < 1 ? 1 : b) : kRedBlocks);
}

// launch grid of a fine-level reduction over a rank's slab: (row tiles,
// local column tiles)
dim3 red_launch_grid(const H* h, const Grid& g) {
  return dim3((g.ny + kRedRows) / kRedRows, (g.ncol + h->red_tx - 1) / h->red_tx);
}

// a.b over the owned columns of the finest level of every rank
void dot(H* h, const std::function<const double2*(Rank&)>& a, const std::function<const double2*(Rank&)>& b,
         RedOp op, bool want_out) {
  reduce(
      h, op,
      [&](Rank& R, RedOp rop, double* out) {
        const Grid& g = R.fine().g;
        k_dot<<<red_launch_grid(h, g), kRedRows, 0, h->stream>>>(a(R), b(R), g, red_tiles(h, g), R.partials,
                                                                 R.rticket, rop, R.st, R.hm_dev, out);
        CKL();
        h->count();
      },
      want_out);
}

// Buffer roles of a captured PCG iteration of direction-buffer parity k:
// every level's iterate starts in u[0]; iteration it smooths against
// r_{it-1}, which lives in rbuf((it-1)&1) under the fused update.
void set_iteration_roles(H* h, int k, bool fused_upd) {
  for (Rank* R : h->ranks) {
    for (Level& L : R->lev) L.cur = 0;
    R->fine().f = fused_upd ? R->rbuf(k) : R->r;
  }
}

// The kernels of one PCG iteration (pcg_solve loop body, solvers.cpp:359-391)
// on parity k, enqueued on the (capturing) stream. `split` runs right after
// the fused update pass that opens an iteration it >= 2.
void enqueue_iteration(H* h, int k, bool first, bool fused_upd, int gamma, int pre, int post,
                       const std::function<void()>& split) {
  const int nc = h->nc;
  // z = M^-1 r: one cycle from z = 0 (solvers.cpp:523-527), fused with z.r
  const bool fused = enqueue_cycle(h, nc, true, gamma, pre, post, kRedZr, (fused_upd && !first) ? k : -1, split);
  auto z = [&](Rank& R) { return R.fine().u[R.fine().cur]; };
  if (!fused) dot(h, z, [&](Rank& R) { return R.fine().f; }, kRedZr, false);
  // p = z + beta p; Ap; pAp; alpha (solvers.cpp:367-382)
  halo_vec(h, nc, z);
  reduce(h, kRedPap, [&](Rank& R, RedOp rop, double* out) {
    MarchArgs a = march_args(h, R, z(R));
    a.u2 = R.pbuf[k];
    a.out0 = R.pbuf[k ^ 1];
    a.out1 = R.ap;
    a.rop = rop;
    a.red_out = out;
    launch_march<StPupd, true>(h, a);
  });
  if (fused_upd) {
    // x and r are updated by the next iteration's first pass (or by
    // finish_update after the last one); it reads A p with halo (p and A p
    // in one exchange)
    halo_vecs(h, {{nc, [&](Rank& R) { return R.pbuf[k ^ 1]; }, 1, 1}, {nc, [&](Rank& R) { return R.ap; }, 1, 1}});
  } else {
    halo_vec(h, nc, [&](Rank& R) { return R.pbuf[k ^ 1]; });
    // x += alpha p; r -= alpha Ap; rr (solvers.cpp:383-386)
    reduce(h, kRedRr, [&](Rank& R, RedOp rop, double* out) {
      const Grid& g = R.fine().g;
      k_update_xr<<<red_launch_grid(h, g), kRedRows, 0, h->stream>>>(R.x, R.r, R.pbuf[k ^ 1], R.ap, g,
                                                                     red_tiles(h, g), R.partials, R.rticket, rop,
                                                                     R.st, R.hm_dev, out);
      CKL();
      h->count();
    });
    halo_vec(h, nc, [&](Rank& R) { return R.r; });
  }
}

// The graph being captured on the handle's stream.
cudaGraph_t capturing_graph(H* h) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t cg = nullptr;
  CK(cudaStreamGetCaptureInfo(h->stream, &cs, nullptr, &cg, nullptr, nullptr));
  return cg;
}

// Appends a conditional node on `hc` after everything captured so far, ends
// that capture and continues capturing into the node's body.
void capture_into_conditional(H* h, cudaGraphConditionalHandle hc, cudaGraphConditionalNodeType type) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t cg = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  CK(cudaStreamGetCaptureInfo(h->stream, &cs, nullptr, &cg, &deps, &ndeps));
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = hc;
  cp.conditional.type = type;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, cg, deps, ndeps, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  cudaGraph_t done = nullptr;
  CK(cudaStreamEndCapture(h->stream, &done));
  CK(cudaStreamBeginCaptureToGraph(h->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
}

// The whole PCG loop of the fused scheme as one graph:
//   iteration 1; tail
//   WHILE (loop) {
//     update(it-1) [StSweep01U]; head: IF (rest) { rest of iteration it (parity 1); tail:
//       IF (next) { update(it); head: IF (rest) { rest of iteration it+1 (parity 0); tail } } }
//   }
// k_loop_head records the residual history and applies the stopping test and
// the iteration cap; k_loop_tail stops on a breakdown (kernels in
// tmg_kernels.cuh). The kernels are those of the per-iteration graphs, so
// the results are bitwise the same; the host launches once and reads the
// LoopRecord.
void capture_loop(H* h, int gamma, int pre, int post) {
  Rank& R0 = *h->ranks[0];
  cudaGraph_t G = nullptr;
  CK(cudaGraphCreate(&G, 0));
  cudaGraphConditionalHandle hw;
  CK(cudaGraphConditionalHandleCreate(&hw, G, 0, cudaGraphCondAssignDefault));
  h->capturing = true;
  h->capture_kernels = 0;
  long head_k = 0, rest_k = 0, first_k = 0;
  try {
    CK(cudaStreamBeginCaptureToGraph(h->stream, G, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    set_iteration_roles(h, 0, true);
    enqueue_iteration(h, 0, true, true, gamma, pre, post, nullptr);
    k_loop_tail<<<1, 1, 0, h->stream>>>(hw, hw, R0.st, R0.lrec_dev);
    CKL();
    h->count();
    first_k = h->capture_kernels;
    capture_into_conditional(h, hw, cudaGraphCondTypeWhile);
    auto iteration = [&](int k, bool last) {
      set_iteration_roles(h, k, true);
      const long k0 = h->capture_kernels;
      auto split = [&] {
        cudaGraphConditionalHandle hr;
        CK(cudaGraphConditionalHandleCreate(&hr, capturing_graph(h), 0, cudaGraphCondAssignDefault));
        k_loop_head<<<1, 1, 0, h->stream>>>(hr, hw, R0.st, R0.lrec_dev);
        CKL();
        h->count();
        head_k = h->capture_kernels - k0;
        capture_into_conditional(h, hr, cudaGraphCondTypeIf);
      };
      enqueue_iteration(h, k, false, true, gamma, pre, post, split);
      cudaGraphConditionalHandle next = hw;
      if (!last) CK(cudaGraphConditionalHandleCreate(&next, capturing_graph(h), 0, cudaGraphCondAssignDefault));
      k_loop_tail<<<1, 1, 0, h->stream>>>(next, hw, R0.st, R0.lrec_dev);
      CKL();
      h->count();
      rest_k = h->capture_kernels - k0 - head_k;
      if (!last) capture_into_conditional(h, next, cudaGraphCondTypeIf);
    };
    iteration(1, false);  // it = 2, 4, ...: r_{it-1} in rbuf(1)
    iteration(0, true);   // it = 3, 5, ...
    cudaGraph_t body = nullptr;
    CK(cudaStreamEndCapture(h->stream, &body));
  } catch (...) {
    h->capturing = false;
    cudaGraph_t part = nullptr;
    cudaStreamEndCapture(h->stream, &part);
    cudaGraphDestroy(G);
    for (Rank* R : h->ranks) R->fine().f = R->r;
    throw;
  }
  h->capturing = false;
  for (Rank* R : h->ranks) R->fine().f = R->r;
  CK(cudaGraphInstantiate(&h->loop, G, 0));
  cudaGraphDestroy(G);
  h->loop_first_kernels = first_k;
  h->loop_head_kernels = head_k;
  h->loop_rest_kernels = rest_k;
}

// One PCG iteration (pcg_solve loop body, solvers.cpp:359-391) as a graph.
// Two graphs alternate the roles of the two direction buffers, because the
// fused p-update reads the old p around each node while writing the new one.
void capture_iteration(H* h, int gamma, int pre, int post) {
  if (h->graph[0] && h->g_gamma == gamma && h->g_pre == pre && h->g_post == post && h->g_omega == h->omega) return;
  for (auto& gx : h->graph) {
    if (gx) cudaGraphExecDestroy(gx);
    gx = nullptr;
  }
  if (h->loop) cudaGraphExecDestroy(h->loop);
  h->loop = nullptr;
  const int nc = h->nc;
  // fused update: the first fine pass is the two-sweep stage, which then
  // also finishes the previous iteration (StSweep01U)
  // (a one-level hierarchy has no smoothing pass: its cycle is the direct solve)
  const bool fused_upd = pre >= 2 && nc >= 1;
  // conditional nodes: not with NCCL collectives inside their bodies (that
  // transport cannot be exercised on a one-GPU box, so its graphs keep the
  // plain form)
  const bool cond_ok = fused_upd && h->cond_nodes && (!h->comm || h->comm->local() || h->nccl_cond);
  // graph slot g: 0/1 = iterations with (it-1)&1 == g (it >= 2 when fused),
  // 2 = iteration 1 of the fused scheme
  auto capture = [&](int g_slot) {
    const int k = g_slot & 1;
    const bool first = g_slot == 2;
    set_iteration_roles(h, k, fused_upd);
    cudaGraph_t g = nullptr;
    // iterations that open with the fused update get a device-side stopping
    // test: the rest of the iteration is the body of a conditional node
    const bool cond = cond_ok && !first;
    long head_kernels = -1;
    std::function<void()> split;
    if (cond) {
      CK(cudaGraphCreate(&g, 0));
      cudaGraphConditionalHandle hc;
      CK(cudaGraphConditionalHandleCreate(&hc, g, 0, cudaGraphCondAssignDefault));
      CK(cudaStreamBeginCaptureToGraph(h->stream, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
      split = [h, hc, &head_kernels] {
        // every rank holds the same r.r, so all take the same branch
        k_set_continue<<<1, 1, 0, h->stream>>>(hc, h->ranks[0]->st);
        CKL();
        h->count();
        head_kernels = h->capture_kernels;
        capture_into_conditional(h, hc, cudaGraphCondTypeIf);
      };
    } else {
      CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    }
    h->capturing = true;
    h->capture_kernels = 0;
    try {
      enqueue_iteration(h, k, first, fused_upd, gamma, pre, post, split);
    } catch (...) {
      h->capturing = false;
      cudaGraph_t part = nullptr;
      cudaStreamEndCapture(h->stream, &part);
      if (part && part != g) cudaGraphDestroy(part);
      if (g) cudaGraphDestroy(g);
      for (Rank* R : h->ranks) R->fine().f = R->r;
      throw;
    }
    h->capturing = false;
    if (cond) {
      cudaGraph_t body = nullptr;
      CK(cudaStreamEndCapture(h->stream, &body));  // the body belongs to g
      if (head_kernels < 0) fail(TMG_ERR_CUDA, "conditional iteration graph without its update pass");
    } else {
      CK(cudaStreamEndCapture(h->stream, &g));
    }
    CK(cudaGraphInstantiate(&h->graph[g_slot], g, 0));
    cudaGraphDestroy(g);
    h->graph_kernels[g_slot] = h->capture_kernels;
    h->graph_head_kernels[g_slot] = cond ? head_kernels : h->capture_kernels;
    for (Rank* R : h->ranks) R->fine().f = R->r;
  };
  capture(0);
  capture(1);
  if (fused_upd) capture(2);
  if (cond_ok && h->device_loop) capture_loop(h, gamma, pre, post);
  h->g_gamma = gamma;
  h->g_pre = pre;
  h->g_post = post;
  h->g_omega = h->omega;
  h->g_fused = fused_upd;
}

// The update of the last iteration when no further graph runs it (fused
// scheme at max_iter): x += alpha p_it, r_it = r_{it-1} - alpha A p_it, r.r.
void finish_update(H* h, int it) {
  const int k = (it - 1) & 1;
  reduce(h, kRedRr, [&](Rank& R, RedOp rop, double* out) {
    const Grid& g = R.fine().g;
    k_update_xr<<<red_launch_grid(h, g), kRedRows, 0, h->stream>>>(R.x, R.rbuf(k), R.pbuf[k ^ 1], R.ap, g,
                                                                   red_tiles(h, g), R.partials, R.rticket, rop,
                                                                   R.st, R.hm_dev, out);
    CKL();
    h->count();
  });
}

// Lower half-bandwidth (in dofs) of the coarsest matrix: 2 dofs per node,
// column-major node numbering, 9-point stencil (the lower neighbour farthest
// away is (x-1, y-1), ny + 2 nodes back).
int coarsest_band(const Grid& g0, int n) { return std::min(n - 1, 2 * (g0.ny + 2) + 1); }


// dense Cholesky of the coarsest matrix, in shared memory when it fits
void launch_cholesky(cudaStream_t s, double* A, int n, int* bad_row) {
  if (n <= kCholSmemMax) {
    const size_t sm = sizeof(double) * (n * n + n);
    CK(cudaFuncSetAttribute(k_cholesky<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
    k_cholesky<true><<<1, 1024, sm, s>>>(A, n, bad_row);
  } else {
    k_cholesky<false><<<1, 1024, 0, s>>>(A, n, bad_row);
  }
  CKL();
}

// ----------------------------------------------------------------- setup --

void setup(H* h, double omega) {
  NvtxRange nvtx("tmg.setup (Galerkin hierarchy + coarsest inverse)");
  if (!h->have_problem) fail(TMG_ERR_DIMENSION, "tmg_gpu_set_problem must precede setup");
  if (!h->have_moduli) fail(TMG_ERR_DIMENSION, "no element moduli uploaded");
  h->omega = omega;
  h->have_setup = false;
  // Galerkin hierarchy, finest to coarsest (solvers.cpp:474-478)
  for (int l = h->nc; l >= 1; --l) {
    for_ranks(h, [&](Rank& Rk) {
      Rank* R = &Rk;
      long off;
      const Grid cg = coarse_of(h, *R, l, off);
      dim3 blk(32, 4), grd((cg.ny + 1 + 31) / 32, (cg.ncol + 3) / 4);
      // the output pointer is offset by `off` nodes inside every plane; the
      // plane stride stays that of the stored level
      if (l == h->nc) {
        k_galerkin_cells<<<grd, blk, 0, h->stream>>>(R->fine_op(), R->lev[l].g, cg, R->lev[l - 1].S + off,
                                                     R->lev[l - 1].g.size);
      } else {
        with_op(*R, l, [&](auto op) {
          k_galerkin<decltype(op)><<<grd, blk, 0, h->stream>>>(op, R->lev[l].g, cg, R->lev[l - 1].S + off,
                                                               R->lev[l - 1].g.size);
        });
      }
      CKL();
      h->count();
    });
    if (h->dist(l - 1)) {
      // ghost columns of the new level's stencil (backward blocks, Galerkin
      // of the next level reads two columns to the left)
      for (int k = 0; k < kStencilPlanes; ++k)
        h->comm->halo(h->ranks, l - 1,
                      [&](Rank& R) -> void* { return R.lev[l - 1].S + static_cast<long>(k) * R.lev[l - 1].g.size; },
                      sizeof(double), kGX, 2, h->stream);
    } else if (h->dist(l)) {
      gather_level(h, l - 1, [&](Rank& R) -> void* { return R.lev[l - 1].S; }, sizeof(double),
                   h->ranks[0]->lev[l - 1].g.size, kStencilPlanes);
    }
  }
  // coarsest: dense matrix -> Cholesky -> explicit symmetric inverse (replicated)
  for (Rank* R : h->ranks) {
    const int n = R->n0;
    const Grid& g0 = R->lev[0].g;
    CK(cudaMemsetAsync(R->A0, 0, sizeof(double) * n * n, h->stream));
    with_op(*R, 0, [&](auto op) {
      k_dense_assemble<decltype(op)><<<dim3((g0.ny + 1 + 63) / 64, g0.nx + 1), 64, 0, h->stream>>>(op, g0, R->A0, n);
    });
    CKL();
    const int b = coarsest_band(g0, n);
    const size_t bsm = static_cast<size_t>(n) * (b + 2) * sizeof(double);
    if (n > kDenseFactorMaxDofs) {
      // large coarsest level: the band is factored in place in L2 (LiT's
      // first row is the scratch for the original diagonal)
      k_cholesky_band_g<<<1, kCholBandGThreads, sizeof(double) * b, h->stream>>>(R->A0, n, b, R->LiT, R->bad_row);
    } else if (h->band_factor && b <= 31 && bsm <= 200 * 1024) {
      CK(cudaFuncSetAttribute(k_cholesky_band, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bsm)));
      k_cholesky_band<<<1, kCholBandThreads, bsm, h->stream>>>(R->A0, n, b, R->bad_row);
    } else {
      launch_cholesky(h->stream, R->A0, n, R->bad_row);
    }
    CKL();
    h->count(2);
  }
  // the explicit inverse is queued behind the factor before the host reads
  // the pivot check (a failed factor's inverse is never used: setup throws)
  for (Rank* R : h->ranks) {
    const int n = R->n0;
    if (n > kDenseFactorMaxDofs) {
      const int b = coarsest_band(R->lev[0].g, n);
      int RW = 32;
      while (RW < b + 1) RW *= 2;
      const int wpb = 8;
      k_lower_inverse_band<<<(n + wpb - 1) / wpb, 32 * wpb, sizeof(double) * RW * wpb, h->stream>>>(R->A0, R->LiT, n,
                                                                                                     b, RW);
      CKL();
      const int nt = (n + kGramTile - 1) / kGramTile;
      k_gram_tiled<<<dim3(nt, nt), 256, 0, h->stream>>>(R->LiT, R->Ainv, n);
      CKL();
      h->count(2);
      continue;
    }
    const int wpb = 4;
    const size_t sm = sizeof(double) * n * wpb;
    CK(cudaFuncSetAttribute(k_lower_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
    k_lower_inverse<<<(n + wpb - 1) / wpb, 32 * wpb, sm, h->stream>>>(R->A0, R->LiT, n,
                                                                       coarsest_band(R->lev[0].g, n));
    CKL();
    k_gram<<<dim3((n + 127) / 128, n), 128, 0, h->stream>>>(R->LiT, R->Ainv, n);
    CKL();
    h->count(2);
  }
  for (Rank* R : h->ranks) {
    k_readback<<<1, 1, 0, h->stream>>>(R->bad_row, nullptr, nullptr, R->rbk_dev);
    CKL();
    h->count();
  }
  CK(cudaStreamSynchronize(h->stream));
  for (Rank* R : h->ranks) {
    const int bad = R->rbk->bad_row;
    if (bad >= 0) {
      fail(TMG_ERR_DEFINITENESS,
           "matrix is not positive definite: non-positive pivot at row " + std::to_string(bad), bad);
    }
  }
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

void solve_resident(H* h, bool use_x0, double tol, int max_iter, int gamma, int pre, int post, SolveOut& o) {
  NvtxRange nvtx("tmg.pcgmg_solve");
  need_setup(h);
  // SolverConfig::validate subset enforced by pcgmg_solve (solvers.cpp:518-521)
  if (pre != post) {
    fail(TMG_ERR_CONFIG, "pcgmg needs pre_sweeps == post_sweeps for a symmetric preconditioner");
  }
  if (gamma != 1 && gamma != 2) fail(TMG_ERR_CONFIG, "gamma must be 1 (V-cycle) or 2 (W-cycle)");
  if (pre < 0) fail(TMG_ERR_CONFIG, "smoothing sweep counts must be non-negative");
  const int nc = h->nc;
  capture_iteration(h, gamma, pre, post);
  const bool dloop = h->loop && max_iter >= 1;
  if (dloop) {
    // the device loop writes residual_history[1 .. iterations] here
    Rank& R0 = *h->ranks[0];
    if (R0.hist_cap < max_iter + 1) {
      if (R0.hist) CK(cudaFreeHost(R0.hist));
      R0.hist = nullptr;
      R0.hist_cap = 0;
      CK(cudaHostAlloc(&R0.hist, sizeof(double) * (max_iter + 1), cudaHostAllocMapped));
      CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&R0.hist_dev), R0.hist, 0));
      R0.hist_cap = max_iter + 1;
    }
  }
  CK(cudaEventRecord(h->ev[0], h->stream));
  auto bvec = [&](Rank& R) { return R.b; };
  // without x0, r = b bitwise, so b.b is also r.r (the plain value lands in scal)
  dot(h, bvec, bvec, kRedB, !use_x0);
  for (Rank* R : h->ranks) {
    k_pcg_begin<<<1, 1, 0, h->stream>>>(R->st, tol, max_iter, R->hist_dev);
    CKL();
    h->count();
    const Level& F = R->fine();
    const long n2 = F.g.size;
    CK(cudaMemsetAsync(R->pbuf[0], 0, sizeof(double2) * n2, h->stream));
    if (use_x0) CK(cudaMemcpyAsync(R->x, R->x0, sizeof(double2) * n2, cudaMemcpyDeviceToDevice, h->stream));
    else CK(cudaMemsetAsync(R->x, 0, sizeof(double2) * n2, h->stream));
  }
  if (use_x0) {
    halo_vec(h, nc, [&](Rank& R) { return R.x; });
    for (Rank* R : h->ranks) apply_level(h, *R, nc, R->x, R->fine().res);
  }
  for (Rank* R : h->ranks) {
    const Grid& g = R->fine().g;
    const long o = g.own_begin();
    k_sub<<<red_grid(g.own_count()), kRedThreads, 0, h->stream>>>(R->b + o, use_x0 ? R->fine().res + o : nullptr,
                                                                   R->r + o, g.own_count());
    CKL();
    h->count();
  }
  halo_vec(h, nc, [&](Rank& R) { return R.r; });
  auto rvec = [&](Rank& R) { return R.r; };
  if (use_x0) dot(h, rvec, rvec, kRedPlain, true);
  Rank& R0 = *h->ranks[0];
  k_readback<<<1, 1, 0, h->stream>>>(nullptr, R0.st, R0.scal, R0.rbk_dev);
  CKL();
  h->count();
  CK(cudaStreamSynchronize(h->stream));
  const double bnorm = R0.rbk->bnorm, rr0 = R0.rbk->scal0;
  o = SolveOut{};
  h->have_solution = true;
  // pcg_solve, solvers.cpp:336-357
  if (bnorm == 0.0) {
    for (Rank* R : h->ranks) CK(cudaMemsetAsync(R->x, 0, sizeof(double2) * R->fine().g.size, h->stream));
    o.converged = 1;
    o.hist.push_back(0.0);
  } else {
    double rel = std::sqrt(rr0) / bnorm;
    o.final_residual = rel;
    o.hist.push_back(rel);
    if (rel <= tol) {
      o.converged = 1;
    } else if (dloop) {
      // the whole loop on the device: one launch, one synchronisation
      LoopRecord* lr = R0.lrec;
      std::memset(lr, 0, sizeof(LoopRecord));
      CK(cudaGraphLaunch(h->loop, h->stream));
      CK(cudaStreamSynchronize(h->stream));
      LoopRecord rec;
      std::memcpy(&rec, lr, sizeof rec);  // written by the device before the synchronisation
      h->launches += h->loop_first_kernels + rec.heads * h->loop_head_kernels +
                     std::max(0, rec.rests - 1) * h->loop_rest_kernels;
      if (rec.status == 4) {
        char buf[200];
        std::snprintf(buf, sizeof buf, "preconditioner is not positive definite: z^T r = %f at iteration %d",
                      rec.zr, rec.err_it);
        fail(TMG_ERR_PRECONDITIONER, buf);
      }
      if (rec.status == 3) {
        char buf[200];
        std::snprintf(buf, sizeof buf, "PCG breakdown: p^T A p = %f at iteration %d", rec.pap, rec.err_it);
        fail(TMG_ERR_DEFINITENESS, buf);
      }
      o.hist.insert(o.hist.end(), R0.hist + 1, R0.hist + 1 + rec.iterations);
      o.iterations = rec.iterations;
      o.converged = rec.converged;
      o.final_residual = o.hist.back();
    } else {
      const bool fu = h->g_fused;
      const volatile HostMirror* m = R0.hm;
      auto record = [&](int done) {  // relres of iteration `done` (solvers.cpp:388-393)
        rel = m->relres;
        o.iterations = done;
        o.final_residual = rel;
        o.hist.push_back(rel);
        if (rel <= tol || rel == 0.0) {
          o.converged = 1;
          return true;
        }
        return false;
      };
      for (int it = 1; it <= max_iter; ++it) {
        const int gs = (fu && it == 1) ? 2 : (it - 1) & 1;
        CK(cudaGraphLaunch(h->graph[gs], h->stream));
        CK(cudaStreamSynchronize(h->stream));
        // fused: this graph opened by finishing iteration it-1; its residual
        // decides before anything iteration `it` computed speculatively (the
        // graph's conditional node already skipped that work on the device)
        if (fu && it >= 2 && record(it - 1)) {
          h->launches += h->graph_head_kernels[gs];
          break;
        }
        h->launches += h->graph_kernels[gs];
        const int status = m->status;
        if (status == 4) {
          char buf[200];
          std::snprintf(buf, sizeof buf, "preconditioner is not positive definite: z^T r = %f at iteration %d",
                        static_cast<double>(m->zr), it);
          fail(TMG_ERR_PRECONDITIONER, buf);
        }
        if (status == 3) {
          char buf[200];
          std::snprintf(buf, sizeof buf, "PCG breakdown: p^T A p = %f at iteration %d", static_cast<double>(m->pap),
                        it);
          fail(TMG_ERR_DEFINITENESS, buf);
        }
        if (fu) {
          if (it == max_iter) {
            finish_update(h, it);
            CK(cudaStreamSynchronize(h->stream));
            record(it);
          }
        } else if (record(it)) {
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
    if (!h->stream) fail(TMG_ERR_CUDA, h->err.empty() ? "handle has no device" : h->err);
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

// Host upload of the fine moduli of one rank: element columns
// [x0 - kGX, x0 + ncol + kGX) clipped to the mesh (ghost elements stay 0).
void upload_moduli_rank(H* h, Rank& R, const double* moduli, double* dst = nullptr, cudaStream_t s = nullptr) {
  const Grid& g = R.fine().g;
  const int e0 = std::max(0, g.x0 - kGX), e1 = std::min(g.nx, g.x0 + g.ncol + kGX);
  if (e1 > e0)
    CK(cudaMemcpy2DAsync((dst ? dst : R.E) + g.idx(e0 - g.x0, 0), sizeof(double) * g.P,
                         moduli + static_cast<long>(e0) * g.ny, sizeof(double) * g.ny, sizeof(double) * g.ny,
                         e1 - e0, cudaMemcpyHostToDevice, s ? s : h->stream));
}

int create_common(H* hp, int nx, int ny, int nc, int dpn, int device, int nranks, int rank, int nlocal,
                  const void* nccl_id, int rep) {
  // build_hierarchy validation (grid.cpp:55-80)
  auto cfg = [&](const std::string& m) {
    hp->err = m;
    return TMG_ERR_CONFIG;
  };
  if (nx < 1 || ny < 1)
    return cfg("grid must have at least one element per direction, got " + std::to_string(nx) + "x" +
               std::to_string(ny));
  if (nc < 0) return cfg("num_coarsenings must be non-negative");
  if (dpn != 2) return cfg("dofs_per_node must be 2: the GPU path solves the plane-elasticity system");
  if (nc > 24) return cfg("num_coarsenings too large");
  const int factor = 1 << nc;
  if (nx % factor != 0)
    return cfg("nx = " + std::to_string(nx) + " is not divisible by 2^" + std::to_string(nc) + " = " +
               std::to_string(factor));
  if (ny % factor != 0)
    return cfg("ny = " + std::to_string(ny) + " is not divisible by 2^" + std::to_string(nc) + " = " +
               std::to_string(factor));
  const int n0 = 2 * (nx / factor + 1) * (ny / factor + 1);
  if (n0 > kCoarsestMaxDofs) {
    return cfg("coarsest level has " + std::to_string(n0) + " dofs; the device coarse solve supports <= " +
               std::to_string(kCoarsestMaxDofs) + " (add coarsenings)");
  }
  // the large-coarsest factor is one CTA walking the band: keep its b^2 n / 2
  // updates around a second (129 x 65 or 65 x 129 coarsest nodes and smaller)
  if (n0 > kDenseFactorMaxDofs && 2 * (ny / factor + 2) + 1 > kLargeCoarsestMaxBand) {
    return cfg("coarsest level has " + std::to_string(n0) + " dofs in columns of " + std::to_string(ny / factor + 1) +
               " nodes; above " + std::to_string(kDenseFactorMaxDofs) + " dofs the device coarse solve supports columns"
               " of at most " + std::to_string((kLargeCoarsestMaxBand - 1) / 2 - 1) + " nodes (add coarsenings)");
  }
  if (nranks < 1 || rank < 0 || rank >= nranks) return cfg("invalid rank / nranks");
  hp->device = device;
  hp->nx = nx;
  hp->ny = ny;
  hp->nc = nc;
  hp->nranks = nranks;
  hp->red_tx = red_tx_of(nx, ny);
  hp->distributed = nranks > 1 || nccl_id != nullptr;
  hp->rep = !hp->distributed ? nc : (rep >= 0 ? std::min(rep, nc - 1) : auto_rep(nx, nc, nranks));
  if (hp->distributed) {
    if (nc < 1 || hp->rep >= nc) return cfg("a distributed solve needs at least the finest level distributed");
    hp->xpart = partition(nx, ny, nc, hp->rep, nranks);
    for (int r = 0; r < nranks; ++r)
      if (hp->xpart[r + 1] - hp->xpart[r] < 2 * partition_gran(nx, ny, nc, hp->rep))
        return cfg("mesh too small for " + std::to_string(nranks) + " slabs");
  } else {
    hp->xpart = {0, nx + 1};
  }
  hp->stream = nullptr;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) fail(TMG_ERR_CUDA, "CUDA device " + std::to_string(device) + " not present");
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) fail(TMG_ERR_CUDA, std::string("libtmg_gpu is built for sm_100a; device is ") + prop.name);
  CK(cudaSetDevice(device));
  CK(cudaFuncSetAttribute(k_smarch<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          static_cast<int>(kSSlotDown * s_stages<false>())));
  CK(cudaFuncSetAttribute(k_smarch<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          static_cast<int>(kSSlotUp * s_stages<true>())));
  CK(cudaFuncSetAttribute(k_smarch2<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          static_cast<int>(kSSlotDown * s_stages<false>())));
  CK(cudaFuncSetAttribute(k_smarch2<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          static_cast<int>(kSSlotUp * s_stages<true>())));
  CK(cudaFuncSetAttribute(k_stile<false, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, t_smem<false, 8>()));
  CK(cudaFuncSetAttribute(k_stile<true, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, t_smem<true, 8>()));
  CK(cudaFuncSetAttribute(k_stile<false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, t_smem<false, 4>()));
  CK(cudaFuncSetAttribute(k_stile<true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, t_smem<true, 4>()));
  CK(cudaFuncSetAttribute(k_stile<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, t_smem<false, 2>()));
  CK(cudaFuncSetAttribute(k_stile<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, t_smem<false, 1>()));
  CK(cudaFuncSetAttribute(k_stile<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, t_smem<true, 1>()));
  CK(cudaFuncSetAttribute(k_stile<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, t_smem<true, 2>()));
  CK(cudaFuncSetAttribute(k_march<StSweep01U, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          static_cast<int>(StSweep01U::kSlot * RingOf<StSweep01U>::value)));
  CK(cudaStreamCreateWithFlags(&hp->stream, cudaStreamNonBlocking));
  if (const char* v = std::getenv("TMG_SMARCH_MIN_NODES")) hp->smarch_min_nodes = std::atol(v);
  if (const char* v = std::getenv("TMG_STILE_MAX_NODES")) hp->stile_max_nodes = std::atol(v);
  if (const char* v = std::getenv("TMG_NO_PDL")) hp->pdl = std::atoi(v) == 0;
  if (const char* v = std::getenv("TMG_STILE_TC1_NODES")) hp->stile_tc1_nodes = std::atol(v);
  if (const char* v = std::getenv("TMG_STILE_TC2_NODES")) hp->stile_tc2_nodes = std::atol(v);
  if (const char* v = std::getenv("TMG_STILE_TC4_NODES")) hp->stile_tc4_nodes = std::atol(v);
  if (const char* v = std::getenv("TMG_NO_COND_NODES")) hp->cond_nodes = std::atoi(v) == 0;
  if (const char* v = std::getenv("TMG_NO_DEVICE_LOOP")) hp->device_loop = std::atoi(v) == 0;
  if (const char* v = std::getenv("TMG_DENSE_COARSE_FACTOR")) hp->band_factor = std::atoi(v) == 0;
  if (const char* v = std::getenv("TMG_NCCL_COND_NODES")) hp->nccl_cond = std::atoi(v) != 0;
  if (const char* v = std::getenv("TMG_SMARCH_LOCKSTEP")) hp->smarch_split = std::atoi(v) == 0;
  for (cudaEvent_t& e : hp->ev) CK(cudaEventCreate(&e));
  for (int i = 0; i < nlocal; ++i) {
    hp->own.push_back(std::make_unique<Rank>());
    Rank& R = *hp->own.back();
    R.index = (nlocal == 1) ? rank : i;
    hp->ranks.push_back(&R);
    alloc_rank(hp, R);
  }
  if (hp->distributed) {
    if (nlocal > 1) {
      hp->comm = std::make_unique<LocalComm>(hp->ranks);
      CK(cudaEventCreateWithFlags(&hp->fork_ev, cudaEventDisableTiming));
      for (int i = 0; i < nlocal; ++i) {
        cudaStream_t s;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        hp->rstreams.push_back(s);
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        hp->join_ev.push_back(e);
      }
    }
    else hp->comm = std::make_unique<NcclComm>(nranks, rank, nccl_id);
  }
  CK(cudaStreamSynchronize(hp->stream));
  return TMG_OK;
}

int create_handle(int nx, int ny, int nc, int dpn, int device, int nranks, int rank, int nlocal, const void* id,
                  int rep, tmg_gpu_handle** out) {
  if (!out) return TMG_ERR_DIMENSION;
  auto h = std::make_unique<tmg_gpu_handle>();
  h->device = device;
  int st = TMG_OK;
  try {
    st = create_common(h.get(), nx, ny, nc, dpn, device, nranks, rank, nlocal, id, rep);
  } catch (const TmgError& e) {
    st = finish(h.get(), e);
  }
  if (st != TMG_OK && h->stream) {
    // keep only the message: the caller may read it, then destroys the handle
    const std::string msg = h->err;
    free_handle(h.get());
    h = std::make_unique<tmg_gpu_handle>();
    h->device = device;
    h->err = msg;
  }
  *out = h.release();
  return st;
}

}  // namespace

// =================================================================== ABI ==

// Pipelined solves: the copy stream, its events and every rank's staging
// buffers (zero-filled once, so their ghost columns and padding stay zero).
void ensure_pipeline(H* h) {
  if (h->cstream) return;
  CK(cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking));
  for (cudaEvent_t* e : {&h->staged[0], &h->staged[1], &h->consumed[0], &h->consumed[1], &h->solved,
                         &h->downloaded})
    CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  for (Rank* R : h->ranks) {
    const Grid& g = R->fine().g;
    const size_t eb = sizeof(double) * (g.size + kSlackNodes), vb = sizeof(double2) * (g.size + kSlackNodes);
    for (int k = 0; k < 2; ++k) {
      CK(cudaMalloc(&R->Es[k], eb));
      CK(cudaMemsetAsync(R->Es[k], 0, eb, h->stream));
      CK(cudaMalloc(&R->bs[k], vb));
      CK(cudaMemsetAsync(R->bs[k], 0, vb, h->stream));
    }
    CK(cudaMalloc(&R->us, vb));
  }
  for (cudaEvent_t e : {h->consumed[0], h->consumed[1]}) CK(cudaEventRecord(e, h->stream));
  CK(cudaEventRecord(h->downloaded, h->cstream));
  CK(cudaStreamSynchronize(h->stream));
}

extern "C" {

int tmg_gpu_create(int nx, int ny, int num_coarsenings, int dofs_per_node, int device, tmg_gpu_handle** out) {
  return create_handle(nx, ny, num_coarsenings, dofs_per_node, device, 1, 0, 1, nullptr, -1, out);
}

int tmg_gpu_create_local_slabs(int nx, int ny, int num_coarsenings, int dofs_per_node, int device, int nslabs,
                               int replicated_level, tmg_gpu_handle** out) {
  return create_handle(nx, ny, num_coarsenings, dofs_per_node, device, nslabs, 0, nslabs, nullptr,
                       replicated_level, out);
}

int tmg_gpu_create_nccl(int nx, int ny, int num_coarsenings, int dofs_per_node, int device, int nranks, int rank,
                        const void* nccl_unique_id, int replicated_level, tmg_gpu_handle** out) {
  return create_handle(nx, ny, num_coarsenings, dofs_per_node, device, nranks, rank, 1, nccl_unique_id,
                       replicated_level, out);
}

int tmg_nccl_unique_id(void* out128) {
  try {
    ncclUniqueId id;
    NK(nccl().getUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
    return TMG_OK;
  } catch (const TmgError& e) {
    return e.code;
  }
}

int tmg_partition(int nx, int ny, int num_coarsenings, int nranks, int replicated_level, int* x0s, int* rep_out) {
  if (nranks < 1 || num_coarsenings < 0 || nx < 1 || ny < 1) return TMG_ERR_CONFIG;
  const int rep = nranks == 1 ? num_coarsenings  // (a single rank stores every level whole)
                              : (replicated_level >= 0 ? std::min(replicated_level, num_coarsenings - 1)
                                                       : auto_rep(nx, num_coarsenings, nranks));
  const std::vector<int> xp =
      nranks == 1 ? std::vector<int>{0, nx + 1} : partition(nx, ny, num_coarsenings, rep, nranks);
  std::memcpy(x0s, xp.data(), sizeof(int) * xp.size());
  if (rep_out) *rep_out = rep;
  return TMG_OK;
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
    const long ndof = 2L * (h->nx + 1) * (h->ny + 1);
    // BoundaryConditions::validate (fem.cpp:110-129)
    std::vector<int> cnt(ndof, 0);
    for (int k = 0; k < n_fixed; ++k) {
      const int d = fixed_dofs[k];
      if (d < 0 || d >= ndof)
        fail(TMG_ERR_CONFIG, "fixed dof " + std::to_string(d) + " outside [0, " + std::to_string(ndof) + ")");
      cnt[d]++;
    }
    for (Rank* R : h->ranks) {
      const Grid& g = R->fine().g;
      std::vector<uint8_t> mask(g.size, 0);
      for (int lx = -kGX; lx < g.ncol + kGX; ++lx) {
        const int x = g.x0 + lx;
        if (x < 0 || x > g.nx) continue;
        for (int y = 0; y <= g.ny; ++y) {
          const long node = static_cast<long>(x) * (g.ny + 1) + y;
          const int c0 = std::min(cnt[2 * node], 15), c1 = std::min(cnt[2 * node + 1], 15);
          mask[g.idx(lx, y)] = static_cast<uint8_t>(c0 | (c1 << 4));
        }
      }
      CK(cudaMemcpyAsync(R->M, mask.data(), g.size, cudaMemcpyHostToDevice, h->stream));
      CK(cudaStreamSynchronize(h->stream));
    }
    h->nu = nu;
    tmg_element_stiffness(1.0, nu, h->ke);
    CK(cudaMemcpyToSymbolAsync(c_k8, h->ke, 8 * sizeof(double), 0, cudaMemcpyHostToDevice, h->stream));  // row 0
    CK(cudaMemcpyToSymbolAsync(c_ke64, h->ke, 64 * sizeof(double), 0, cudaMemcpyHostToDevice, h->stream));
    // M_q = (1/4) P_q^T Ke P_q of the four element quadrants of a coarse cell
    // (k_galerkin_cells), from the exact Ke the device applies
    {
      double mq[4][64];
      auto w1 = [](int f, int cc) { return f == 2 * cc ? 1.0L : (f == 1 ? 0.5L : 0.0L); };
      const int cx[4] = {0, 1, 1, 0}, cy[4] = {0, 0, 1, 1};  // corner -> (x, y)
      for (int q = 0; q < 4; ++q) {
        const int qx = q & 1, qy = q >> 1;
        long double Pm[8][8] = {};  // fine dof (2k+d) <- coarse dof (2m+d)
        for (int k = 0; k < 4; ++k)
          for (int m = 0; m < 4; ++m) {
            const long double w = w1(qx + cx[k], cx[m]) * w1(qy + cy[k], cy[m]);
            for (int d = 0; d < 2; ++d) Pm[2 * k + d][2 * m + d] = w;
          }
        for (int a = 0; a < 8; ++a)
          for (int b = 0; b < 8; ++b) {
            long double acc = 0.0L;
            for (int r = 0; r < 8; ++r)
              for (int c = 0; c < 8; ++c) acc += Pm[r][a] * static_cast<long double>(h->ke[r * 8 + c]) * Pm[c][b];
            mq[q][a * 8 + b] = static_cast<double>(0.25L * acc);
          }
      }
      CK(cudaMemcpyToSymbolAsync(c_mq, mq, sizeof(mq), 0, cudaMemcpyHostToDevice, h->stream));
    }
    CK(cudaStreamSynchronize(h->stream));
    h->have_problem = true;
    h->have_setup = false;
  });
}

int tmg_gpu_upload_moduli(tmg_gpu_handle* h, const double* moduli, long n_elem) {
  return guarded(h, [&] {
    if (n_elem != static_cast<long>(h->nx) * h->ny)
      fail(TMG_ERR_DIMENSION, "element modulus count " + std::to_string(n_elem) + " does not match grid with " +
                                  std::to_string(static_cast<long>(h->nx) * h->ny) + " elements");
    for (Rank* R : h->ranks) upload_moduli_rank(h, *R, moduli);
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

int tmg_gpu_set_density(tmg_gpu_handle* h, const double* alpha, int nphases, const double* phase_moduli,
                        double penalty, double omega) {
  const int s = guarded(h, [&] {
    need_single(h, "tmg_gpu_set_density");
    Rank& R = *h->ranks[0];
    const Grid& g = R.fine().g;
    const long ne = static_cast<long>(g.nx) * g.ny;
    double* da = grow(R.aux, R.aux_cap, ne * nphases);
    double* dp = grow(R.aux2, R.aux2_cap, nphases);
    CK(cudaMemcpyAsync(da, alpha, sizeof(double) * ne * nphases, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(dp, phase_moduli, sizeof(double) * nphases, cudaMemcpyHostToDevice, h->stream));
    k_simp<<<dim3((g.ny + 127) / 128, g.nx), 128, 0, h->stream>>>(g, nphases, da, dp, penalty, R.E);
    CKL();
    h->count();
    h->have_moduli = true;
    h->have_setup = false;
  });
  if (s != TMG_OK) return s;
  return tmg_gpu_setup(h, omega);
}

int tmg_gpu_upload_rhs(tmg_gpu_handle* h, const double* b) {
  return guarded(h, [&] {
    for (Rank* R : h->ranks) upload_nodes(h->stream, R->b, b, R->fine().g);
  });
}

int tmg_gpu_upload_x0(tmg_gpu_handle* h, const double* x0) {
  return guarded(h, [&] {
    for (Rank* R : h->ranks) upload_nodes(h->stream, R->x0, x0, R->fine().g);
  });
}

int tmg_gpu_solution_to_x0(tmg_gpu_handle* h) {
  return guarded(h, [&] {
    for (Rank* R : h->ranks)
      CK(cudaMemcpyAsync(R->x0, R->x, sizeof(double2) * R->fine().g.size, cudaMemcpyDeviceToDevice, h->stream));
  });
}

int tmg_gpu_solve_resident(tmg_gpu_handle* h, int use_x0, double tol, int max_iter, int gamma, int pre_sweeps,
                           int post_sweeps, int* iterations, double* final_residual, int* converged,
                           double* seconds, double* history, int history_cap, int* history_len) {
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
  return guarded(h, [&] {
    for (Rank* R : h->ranks) download_nodes(h->stream, x_out, R->x, R->fine().g);
    CK(cudaStreamSynchronize(h->stream));
  });
}

int tmg_gpu_solve(tmg_gpu_handle* h, const double* b, const double* x0, double tol, int max_iter, int gamma,
                  int pre_sweeps, int post_sweeps, double* x_out, int* iterations, double* final_residual,
                  int* converged, double* seconds, double* history, int history_cap, int* history_len) {
  return guarded(h, [&] {
    need_setup(h);
    for (Rank* R : h->ranks) {
      upload_nodes(h->stream, R->b, b, R->fine().g);
      if (x0) upload_nodes(h->stream, R->x0, x0, R->fine().g);
    }
    SolveOut o;
    solve_resident(h, x0 != nullptr, tol, max_iter, gamma, pre_sweeps, post_sweeps, o);
    for (Rank* R : h->ranks) download_nodes(h->stream, x_out, R->x, R->fine().g);
    CK(cudaStreamSynchronize(h->stream));
    if (iterations) *iterations = o.iterations;
    if (final_residual) *final_residual = o.final_residual;
    if (converged) *converged = o.converged;
    if (seconds) *seconds = o.seconds;
    copy_out_hist(o, history, history_cap, history_len);
  });
}

int tmg_gpu_stage_inputs(tmg_gpu_handle* h, int slot, const double* moduli, long n_elem, const double* b) {
  return guarded(h, [&] {
    if (slot != 0 && slot != 1) fail(TMG_ERR_DIMENSION, "staging slot must be 0 or 1");
    if (n_elem != static_cast<long>(h->nx) * h->ny)
      fail(TMG_ERR_DIMENSION, "element modulus count " + std::to_string(n_elem) + " does not match grid with " +
                                  std::to_string(static_cast<long>(h->nx) * h->ny) + " elements");
    if (!h->have_problem) fail(TMG_ERR_CONFIG, "problem not set (call tmg_gpu_set_problem)");
    ensure_pipeline(h);
    // the slot's previous contents must have been copied into the resident arrays
    CK(cudaStreamWaitEvent(h->cstream, h->consumed[slot], 0));
    for (Rank* R : h->ranks) {
      upload_moduli_rank(h, *R, moduli, R->Es[slot], h->cstream);
      upload_nodes(h->cstream, R->bs[slot], b, R->fine().g);
    }
    CK(cudaEventRecord(h->staged[slot], h->cstream));
    h->staged_ok[slot] = true;
  });
}

int tmg_gpu_solve_staged(tmg_gpu_handle* h, int slot, double omega, double tol, int max_iter, int gamma,
                         int pre_sweeps, int post_sweeps, double* x_out, int* iterations, double* final_residual,
                         int* converged, double* seconds, double* history, int history_cap, int* history_len) {
  return guarded(h, [&] {
    if (slot != 0 && slot != 1) fail(TMG_ERR_DIMENSION, "staging slot must be 0 or 1");
    if (!h->cstream || !h->staged_ok[slot]) fail(TMG_ERR_CONFIG, "no inputs staged in this slot");
    h->staged_ok[slot] = false;
    // install the staged moduli and rhs (device copies after the staging copies land)
    CK(cudaStreamWaitEvent(h->stream, h->staged[slot], 0));
    for (Rank* R : h->ranks) {
      const Grid& g = R->fine().g;
      CK(cudaMemcpyAsync(R->E, R->Es[slot], sizeof(double) * (g.size + kSlackNodes), cudaMemcpyDeviceToDevice,
                         h->stream));
      CK(cudaMemcpyAsync(R->b, R->bs[slot], sizeof(double2) * (g.size + kSlackNodes), cudaMemcpyDeviceToDevice,
                         h->stream));
    }
    CK(cudaEventRecord(h->consumed[slot], h->stream));
    h->have_moduli = true;
    h->have_setup = false;
    CK(cudaEventRecord(h->ev[2], h->stream));
    setup(h, omega);
    CK(cudaEventRecord(h->ev[3], h->stream));
    SolveOut o;
    solve_resident(h, false, tol, max_iter, gamma, pre_sweeps, post_sweeps, o);
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev[2], h->ev[3]));
    h->last_setup_ms = ms;
    // the solution's staging copy (once the previous download has read it),
    // then its download on the copy stream, overlapping whatever the compute
    // stream runs next
    CK(cudaStreamWaitEvent(h->stream, h->downloaded, 0));
    for (Rank* R : h->ranks)
      CK(cudaMemcpyAsync(R->us, R->x, sizeof(double2) * R->fine().g.size, cudaMemcpyDeviceToDevice, h->stream));
    CK(cudaEventRecord(h->solved, h->stream));
    CK(cudaStreamWaitEvent(h->cstream, h->solved, 0));
    for (Rank* R : h->ranks) download_nodes(h->cstream, x_out, R->us, R->fine().g);
    CK(cudaEventRecord(h->downloaded, h->cstream));
    if (iterations) *iterations = o.iterations;
    if (final_residual) *final_residual = o.final_residual;
    if (converged) *converged = o.converged;
    if (seconds) *seconds = o.seconds;
    copy_out_hist(o, history, history_cap, history_len);
  });
}

int tmg_gpu_sync_outputs(tmg_gpu_handle* h) {
  return guarded(h, [&] {
    if (!h->cstream) return;
    // later work on the compute stream (and its events) orders after the downloads
    CK(cudaStreamWaitEvent(h->stream, h->downloaded, 0));
    CK(cudaEventSynchronize(h->downloaded));
  });
}

int tmg_gpu_compliance(tmg_gpu_handle* h, const double* u, double* out) {
  return guarded(h, [&] {
    if (!h->have_moduli || !h->have_problem) fail(TMG_ERR_DIMENSION, "operator not set");
    if (!u && !h->have_solution) fail(TMG_ERR_DIMENSION, "no resident solution");
    if (u)
      for (Rank* R : h->ranks) upload_nodes(h->stream, R->fine().res, u, R->fine().g);
    auto src = [&](Rank& R) -> double2* { return u ? R.fine().res : R.x; };
    halo_vec(h, h->nc, src);
    apply_dot_fine(h, src, [&](Rank& R) { return R.fine().u[1]; }, kRedPlain, true);
    Rank& R0 = *h->ranks[0];
    CK(cudaMemcpyAsync(R0.scal_host, R0.scal, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    *out = *R0.scal_host;
  });
}

int tmg_gpu_element_energies(tmg_gpu_handle* h, const double* u, double* out) {
  return guarded(h, [&] {
    need_single(h, "tmg_gpu_element_energies");
    if (!h->have_problem) fail(TMG_ERR_DIMENSION, "problem not set");
    Rank& R = *h->ranks[0];
    Level& F = R.fine();
    const Grid& g = F.g;
    const long ne = static_cast<long>(g.nx) * g.ny;
    const double2* src = R.x;
    if (u) {
      upload_nodes(h->stream, F.res, u, g);
      src = F.res;
    } else if (!h->have_solution) {
      fail(TMG_ERR_DIMENSION, "no resident solution");
    }
    double* d = grow(R.dense, R.dense_cap, ne);
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
    need_single(h, "tmg_gpu_sensitivities");
    if (!h->have_problem) fail(TMG_ERR_DIMENSION, "problem not set");
    Rank& R = *h->ranks[0];
    Level& F = R.fine();
    const Grid& g = F.g;
    const long ne = static_cast<long>(g.nx) * g.ny;
    const double2* src = R.x;
    if (u) {
      upload_nodes(h->stream, F.res, u, g);
      src = F.res;
    } else if (!h->have_solution) {
      fail(TMG_ERR_DIMENSION, "no resident solution");
    }
    double* en = grow(R.dense, R.dense_cap, ne * (nphases + 1));
    double* da = grow(R.aux, R.aux_cap, ne * nphases);
    double* dp = grow(R.aux2, R.aux2_cap, nphases);
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

int tmg_gpu_filter(tmg_gpu_handle* h, int nphases, const double* alpha, int phase, double radius, const double* raw,
                   double* out) {
  return guarded(h, [&] {
    need_single(h, "tmg_gpu_filter");
    Rank& R = *h->ranks[0];
    const Grid& g = R.fine().g;
    const long ne = static_cast<long>(g.nx) * g.ny;
    if (phase < 0 || phase >= nphases) fail(TMG_ERR_DIMENSION, "filter: phase out of range");
    if (radius <= 1.0) {  // only the self weight survives (mto.cpp:95)
      std::memcpy(out, raw, sizeof(double) * ne);
      return;
    }
    const int reach = static_cast<int>(std::ceil(radius)) - 1;
    double* da = grow(R.aux, R.aux_cap, ne * nphases);
    double* d = grow(R.dense, R.dense_cap, 2 * ne);
    CK(cudaMemcpyAsync(da, alpha, sizeof(double) * ne * nphases, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(d, raw, sizeof(double) * ne, cudaMemcpyHostToDevice, h->stream));
    k_filter<<<dim3((g.ny + 127) / 128, g.nx), 128, 0, h->stream>>>(g.nx, g.ny, nphases, phase, radius, reach, da, d,
                                                                     d + ne);
    CKL();
    h->count();
    CK(cudaMemcpyAsync(out, d + ne, sizeof(double) * ne, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  });
}

}  // extern "C"

namespace {

// Scratch of one OC exchange on rank 0: the per-element 32-byte records
// first (aligned at the allocation base), then maxima, partials, barrier and
// flags. Grown on demand; `extra` doubles after it are the caller's.
long oc_records(long ne) { return 4 * ne; }  // doubles: two 16-byte record streams

double* oc_scratch(Rank& R, long ne, long extra, int blocks) {
  return grow(R.ocbuf, R.ocbuf_cap, oc_records(ne) + 4L * blocks + 4 + extra);
}

int oc_blocks() {
  static int blocks = 0;
  if (!blocks) {
    int dev = 0, sms = 0, per_sm = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_oc_bisect, kOcThreads, 0));
    if (per_sm < 1) fail(TMG_ERR_CUDA, "k_oc_bisect cannot be resident");
    // TMG_OC_CTAS: fewer CTAs per SM than the residency limit (for A/B timing)
    if (const char* e = std::getenv("TMG_OC_CTAS")) per_sm = std::max(1, std::min(per_sm, std::atoi(e)));
    blocks = sms * per_sm;
  }
  return blocks;
}

// One OC exchange on device data (oc_update_pair, mto.cpp:142-227): alpha
// element-major, sens a/b and move per element, all on rank 0's device.
// Throws TMG_ERR_MULTIPLIER (alpha unchanged) like the reference.
void oc_pair_device(H* h, Rank& R, double* scratch, double* alpha, long ne, int np, double eps, int pa, int pb,
                    const double* sa, const double* sb, double target, const double* mv, double damping) {
  NvtxRange nvtx("tmg.oc_update_pair");
  const int blocks = oc_blocks();
  OcArgs a{};
  a.ne = ne;
  a.np = np;
  a.pa = pa;
  a.pb = pb;
  a.el0 = reinterpret_cast<double2*>(scratch);
  a.el1 = a.el0 + ne;
  a.pmax = scratch + oc_records(ne);
  a.part = a.pmax + 2L * blocks;
  a.bar = reinterpret_cast<unsigned*>(a.part + 2L * blocks);
  a.met = reinterpret_cast<int*>(a.bar + 2);
  a.alpha = alpha;
  a.sa = sa;
  a.sb = sb;
  a.mv = mv;
  a.eps = eps;
  a.target = target;
  a.damping = damping;
  CK(cudaMemsetAsync(a.bar, 0, 4 * sizeof(unsigned), h->stream));
  CK(cudaEventRecord(h->ev[2], h->stream));
  k_oc_prep<<<blocks, kOcThreads, 0, h->stream>>>(a);
  CKL();
  k_oc_gain<<<blocks, kOcThreads, 0, h->stream>>>(a, blocks);
  CKL();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(kOcThreads);
  cfg.stream = h->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // every CTA resident: the bisection crosses grid barriers
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k_oc_bisect, a, blocks));
  CK(cudaEventRecord(h->ev[3], h->stream));
  h->count(3);
  int* flags = reinterpret_cast<int*>(R.scal_host);
  CK(cudaMemcpyAsync(flags, a.met, 2 * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, h->ev[2], h->ev[3]));
  h->last_oc_ms = ms;
  h->last_oc_steps = flags[1];
  if (!flags[0]) {
    char buf[200];
    std::snprintf(buf, sizeof buf, "volume target %f for phase %d is unreachable under the current bounds", target,
                  pa + 1);
    fail(TMG_ERR_MULTIPLIER, buf);
  }
}

}  // namespace

extern "C" {

int tmg_gpu_oc_update_pair(tmg_gpu_handle* h, double* alpha, int nphases, double floor_eps, int phase_a,
                           int phase_b, const double* sens_a, const double* sens_b, double target,
                           const double* move, double damping) {
  return guarded(h, [&] {
    need_single(h, "tmg_gpu_oc_update_pair");
    if (phase_a == phase_b) fail(TMG_ERR_CONFIG, "oc_update_pair: phases must differ");
    if (phase_a < 0 || phase_b < 0 || phase_a >= nphases || phase_b >= nphases)
      fail(TMG_ERR_DIMENSION, "oc_update_pair: phase out of range");
    Rank& R = *h->ranks[0];
    const long ne = static_cast<long>(h->nx) * h->ny;
    // scratch, then the uploaded density, sens a/b and move
    const int blocks = oc_blocks();
    double* scratch = oc_scratch(R, ne, ne * nphases + 3 * ne, blocks);
    double* d_alpha = scratch + oc_records(ne) + 4L * blocks + 4;
    double* sa = d_alpha + ne * nphases;
    double* sb = sa + ne;
    double* mv = sb + ne;
    CK(cudaMemcpyAsync(d_alpha, alpha, sizeof(double) * ne * nphases, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(sa, sens_a, sizeof(double) * ne, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(sb, sens_b, sizeof(double) * ne, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(mv, move, sizeof(double) * ne, cudaMemcpyHostToDevice, h->stream));
    oc_pair_device(h, R, scratch, d_alpha, ne, nphases, floor_eps, phase_a, phase_b, sa, sb, target, mv, damping);
    CK(cudaMemcpy(alpha, d_alpha, sizeof(double) * ne * nphases, cudaMemcpyDeviceToHost));
  });
}

int tmg_gpu_optimize(tmg_gpu_handle* h, const tmg_optim_config* c, const double* rhs, double* density_out,
                     double* compliance_hist, double* change_hist, int* iters_hist, double* seconds_hist,
                     int* outer_iterations, long* total_solver_iterations, int* converged, double* seconds) {
  return guarded(h, [&] {
    using clk = std::chrono::steady_clock;
    const auto t_start = clk::now();
    need_single(h, "tmg_gpu_optimize");
    if (!h->have_problem) fail(TMG_ERR_DIMENSION, "tmg_gpu_set_problem must precede tmg_gpu_optimize");
    // OptimConfig::validate (mto.cpp:20-50), MaterialModel::validate
    // (density.cpp:10-27), SolverConfig::validate (solvers.cpp:70-87)
    const int np = c->nphases;
    if (np < 2) fail(TMG_ERR_CONFIG, "need at least two phases (one material plus void)");
    double sum = 0.0;
    for (int i = 0; i < np; ++i) {
      const double v = c->volume_fractions[i];
      if (!(v > 0.0 && v < 1.0))
        fail(TMG_ERR_CONFIG, "volume_fractions entries must lie in (0, 1), got " + std::to_string(v));
      sum += v;
    }
    if (std::abs(sum - 1.0) > 1e-12) fail(TMG_ERR_CONFIG, "volume_fractions must sum to 1, got " + std::to_string(sum));
    if (c->filter_radius < 0.0) fail(TMG_ERR_CONFIG, "filter_radius must be >= 0");
    if (!(c->filter_tol > 0.0)) fail(TMG_ERR_CONFIG, "filter_tol must be positive");
    if (!(c->tol > 0.0)) fail(TMG_ERR_CONFIG, "tol must be positive");
    if (c->inner_sweeps < 1) fail(TMG_ERR_CONFIG, "inner_sweeps must be >= 1");
    if (!(c->move_limit > 0.0 && c->move_limit <= 1.0)) fail(TMG_ERR_CONFIG, "move_limit must lie in (0, 1]");
    if (!(c->oc_damping > 0.0 && c->oc_damping <= 1.0)) fail(TMG_ERR_CONFIG, "oc_damping must lie in (0, 1]");
    if (c->max_outer < 1) fail(TMG_ERR_CONFIG, "max_outer must be >= 1");
    if (!(c->density_floor > 0.0 && c->density_floor < 0.5))
      fail(TMG_ERR_CONFIG, "density_floor must lie in (0, 0.5)");
    if (!(c->solver_tol > 0.0)) fail(TMG_ERR_CONFIG, "solver tol must be positive");
    if (c->solver_max_iter < 1) fail(TMG_ERR_CONFIG, "max_iter must be >= 1");
    if (!(c->omega > 0.0 && c->omega <= 1.0))
      fail(TMG_ERR_CONFIG, "omega must lie in (0, 1], got " + std::to_string(c->omega));
    if (c->gamma != 1 && c->gamma != 2) fail(TMG_ERR_CONFIG, "gamma must be 1 (V-cycle) or 2 (W-cycle)");
    if (c->pre_sweeps < 0 || c->post_sweeps < 0) fail(TMG_ERR_CONFIG, "smoothing sweep counts must be non-negative");
    if (c->pre_sweeps != c->post_sweeps)
      fail(TMG_ERR_CONFIG, "pcgmg needs pre_sweeps == post_sweeps for a symmetric preconditioner");
    for (int i = 0; i < np; ++i)
      if (!(c->phase_moduli[i] > 0.0))
        fail(TMG_ERR_CONFIG, "phase modulus " + std::to_string(i + 1) +
                                 " must be positive (void is a small positive number)");
    if (!(c->penalty >= 1.0)) fail(TMG_ERR_CONFIG, "penalty exponent must be >= 1, got " + std::to_string(c->penalty));

    Rank& R = *h->ranks[0];
    const Grid& g = R.fine().g;
    const long ne = static_cast<long>(g.nx) * g.ny, nv = ne * np;
    const int blocks = oc_blocks();
    // device state: density, the density before the OC sweep (and before each
    // inner sweep), last deltas, move limits, energies + raw and filtered
    // sensitivities, phase moduli and fractions, then the OC scratch
    double* scratch = oc_scratch(R, ne, 0, blocks);
    const long sz = 5 * nv + 2 * ne + nv + 2L * np + 2;
    double* base = grow(R.dense, R.dense_cap, sz);
    double* dens = base;
    double* before = dens + nv;
    double* pre = before + nv;
    double* last = pre + nv;
    double* filt = last + nv;
    double* move = filt + nv;
    double* en = move + ne;
    double* raw = en + ne;
    double* pm = raw + nv;
    double* fr = pm + np;
    auto* maxbits = reinterpret_cast<unsigned long long*>(fr + np);
    CK(cudaMemcpyAsync(pm, c->phase_moduli, sizeof(double) * np, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(fr, c->volume_fractions, sizeof(double) * np, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemsetAsync(last, 0, sizeof(double) * nv, h->stream));
    k_fill_uniform<<<1184, 256, 0, h->stream>>>(ne, np, fr, dens);
    CKL();
    std::vector<double> mv_host(static_cast<size_t>(ne), c->move_limit);
    CK(cudaMemcpyAsync(move, mv_host.data(), sizeof(double) * ne, cudaMemcpyHostToDevice, h->stream));
    for (Rank* Rk : h->ranks) upload_nodes(h->stream, Rk->b, rhs, Rk->fine().g);
    h->count();
    auto max_change = [&](const double* a, const double* b) {
      CK(cudaMemsetAsync(maxbits, 0, sizeof(unsigned long long), h->stream));
      k_max_abs_diff<<<1184, 256, 0, h->stream>>>(nv, a, b, maxbits);
      CKL();
      h->count();
      unsigned long long bits = 0;
      CK(cudaMemcpyAsync(R.scal_host, maxbits, sizeof(bits), cudaMemcpyDeviceToHost, h->stream));
      CK(cudaStreamSynchronize(h->stream));
      std::memcpy(&bits, R.scal_host, sizeof(bits));
      double v;
      std::memcpy(&v, &bits, sizeof(v));
      return v;
    };
    auto chk = [&](int st) {
      if (st != TMG_OK) fail(st, h->err, h->err_row);
    };
    *outer_iterations = 0;
    *total_solver_iterations = 0;
    *converged = 0;
    bool have_u = false;
    const int reach = static_cast<int>(std::ceil(c->filter_radius)) - 1;
    for (int outer = 1; outer <= c->max_outer; ++outer) {
      NvtxRange nvtx("tmg.optimize outer iteration");
      const auto t_iter = clk::now();
      // assemble_elasticity + build_multigrid_operators (mto.cpp:267-281)
      k_simp<<<dim3((g.ny + 127) / 128, g.nx), 128, 0, h->stream>>>(g, np, dens, pm, c->penalty, R.E);
      CKL();
      h->count();
      h->have_moduli = true;
      h->have_setup = false;
      setup(h, c->omega);
      // pcgmg_solve, warm-started from the previous u (mto.cpp:268-283)
      const bool warm = c->warm_start && have_u;
      if (warm)
        CK(cudaMemcpyAsync(R.x0, R.x, sizeof(double2) * g.size, cudaMemcpyDeviceToDevice, h->stream));
      SolveOut o;
      solve_resident(h, warm, c->solver_tol, c->solver_max_iter, c->gamma, c->pre_sweeps, c->post_sweeps, o);
      have_u = true;
      double comp = 0.0;
      chk(tmg_gpu_compliance(h, nullptr, &comp));
      compliance_hist[outer - 1] = comp;
      iters_hist[outer - 1] = o.iterations;
      *total_solver_iterations += o.iterations;
      // sensitivities and filtered sensitivities (mto.cpp:61-117, 300-310)
      k_element_energy<<<dim3((g.ny + 127) / 128, g.nx), 128, 0, h->stream>>>(g, R.x, en);
      CKL();
      k_sensitivity<<<1184, 256, 0, h->stream>>>(ne, np, dens, en, pm, c->penalty, raw);
      CKL();
      h->count(2);
      for (int i = 0; i < np; ++i) {
        if (c->filter_radius <= 1.0) {
          CK(cudaMemcpyAsync(filt + i * ne, raw + i * ne, sizeof(double) * ne, cudaMemcpyDeviceToDevice, h->stream));
        } else {
          k_filter<<<dim3((g.ny + 127) / 128, g.nx), 128, 0, h->stream>>>(g.nx, g.ny, np, i, c->filter_radius, reach,
                                                                           dens, raw + i * ne, filt + i * ne);
          CKL();
          h->count();
        }
      }
      // OC pair sweeps (mto.cpp:312-323)
      CK(cudaMemcpyAsync(before, dens, sizeof(double) * nv, cudaMemcpyDeviceToDevice, h->stream));
      for (int a = 0; a < np - 1; ++a)
        for (int b = a + 1; b < np; ++b)
          for (int sweep = 0; sweep < c->inner_sweeps; ++sweep) {
            if (c->inner_sweeps > 1)
              CK(cudaMemcpyAsync(pre, dens, sizeof(double) * nv, cudaMemcpyDeviceToDevice, h->stream));
            oc_pair_device(h, R, scratch, dens, ne, np, c->density_floor, a, b, filt + a * ne, filt + b * ne,
                           c->volume_fractions[a], move, c->oc_damping);
            // with one sweep the reference's stop test cannot change anything
            if (c->inner_sweeps == 1 || max_change(dens, pre) <= c->filter_tol) break;
          }
      // move limits and the convergence test (mto.cpp:325-350)
      k_move_adapt<<<1184, 256, 0, h->stream>>>(ne, np, dens, before, last, move, c->move_limit);
      CKL();
      h->count();
      const double change = max_change(dens, before);
      change_hist[outer - 1] = change;
      seconds_hist[outer - 1] = std::chrono::duration<double>(clk::now() - t_iter).count();
      *outer_iterations = outer;
      if (change <= c->tol) {
        *converged = 1;
        break;
      }
    }
    CK(cudaMemcpyAsync(density_out, dens, sizeof(double) * nv, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    *seconds = std::chrono::duration<double>(clk::now() - t_start).count();
  });
}

int tmg_gpu_oc_timings(tmg_gpu_handle* h, double* device_ms, int* steps) {
  if (!h) return TMG_ERR_DIMENSION;
  if (device_ms) *device_ms = h->last_oc_ms;
  if (steps) *steps = h->last_oc_steps;
  return TMG_OK;
}

int tmg_gpu_apply(tmg_gpu_handle* h, int level, const double* x, double* y) {
  return guarded(h, [&] {
    need_single(h, "tmg_gpu_apply");
    check_level(h, level);
    if (level < h->nc) need_setup(h);
    if (!h->have_moduli || !h->have_problem) fail(TMG_ERR_DIMENSION, "operator not set");
    Rank& R = *h->ranks[0];
    Level& L = R.lev[level];
    upload_nodes(h->stream, L.u[0], x, L.g);
    apply_level(h, R, level, L.u[0], L.res);
    download_nodes(h->stream, y, L.res, L.g);
    CK(cudaStreamSynchronize(h->stream));
  });
}

int tmg_gpu_level_values(tmg_gpu_handle* h, int level, const int* offsets, const int* cols, double* vals) {
  return guarded(h, [&] {
    need_single(h, "tmg_gpu_level_values");
    check_level(h, level);
    if (level < h->nc) need_setup(h);
    Rank& R = *h->ranks[0];
    const Level& L = R.lev[level];
    const long n = L.ndof;
    const long nnz = offsets[n];
    int* doff = reinterpret_cast<int*>(grow(R.aux, R.aux_cap, (n + 1 + nnz + 1) / 2 + 1));
    int* dcol = doff + n + 1;
    double* dv = grow(R.dense, R.dense_cap, nnz);
    CK(cudaMemcpyAsync(doff, offsets, sizeof(int) * (n + 1), cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(dcol, cols, sizeof(int) * nnz, cudaMemcpyHostToDevice, h->stream));
    with_op(R, level, [&](auto op) {
      k_level_values<decltype(op)><<<(n + 127) / 128, 128, 0, h->stream>>>(op, L.g, n, doff, dcol, dv);
    });
    CKL();
    h->count();
    CK(cudaMemcpyAsync(vals, dv, sizeof(double) * nnz, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  });
}

int tmg_gpu_vcycle(tmg_gpu_handle* h, const double* f, double* u, int gamma, int pre_sweeps, int post_sweeps) {
  return guarded(h, [&] {
    need_setup(h);
    const int nc = h->nc;
    // a zero start takes the zero-start passes, as inside pcgmg
    const long n = 2L * (h->nx + 1) * (h->ny + 1);
    const bool zero = std::all_of(u, u + n, [](double v) { return v == 0.0; });
    for (Rank* R : h->ranks) {
      for (Level& L : R->lev) L.cur = 0;
      upload_nodes(h->stream, R->r, f, R->fine().g);
      upload_nodes(h->stream, R->fine().u[0], u, R->fine().g);
    }
    halo_vec(h, nc, [&](Rank& R) { return R.r; });
    enqueue_cycle(h, nc, zero, gamma, pre_sweeps, post_sweeps);
    for (Rank* R : h->ranks) download_nodes(h->stream, u, R->fine().u[R->fine().cur], R->fine().g);
    CK(cudaStreamSynchronize(h->stream));
  });
}

int tmg_gpu_prolongate(tmg_gpu_handle* h, int level, const double* coarse, double* fine) {
  return guarded(h, [&] {
    need_single(h, "tmg_gpu_prolongate");
    check_level(h, level);
    if (level < 1) fail(TMG_ERR_DIMENSION, "prolongate: level " + std::to_string(level) + " has no coarser neighbor");
    Rank& R = *h->ranks[0];
    Level& F = R.lev[level];
    Level& C = R.lev[level - 1];
    upload_nodes(h->stream, C.u[0], coarse, C.g);
    prolong_level(h, R, level, C.u[0], F.res, false);
    download_nodes(h->stream, fine, F.res, F.g);
    CK(cudaStreamSynchronize(h->stream));
  });
}

int tmg_gpu_restrict(tmg_gpu_handle* h, int level, const double* fine, double* coarse) {
  return guarded(h, [&] {
    need_single(h, "tmg_gpu_restrict");
    check_level(h, level);
    if (level < 1) fail(TMG_ERR_DIMENSION, "restrict: level " + std::to_string(level) + " has no coarser neighbor");
    Rank& R = *h->ranks[0];
    Level& F = R.lev[level];
    Level& C = R.lev[level - 1];
    upload_nodes(h->stream, F.res, fine, F.g);
    restrict_level(h, R, level, F.res, C.res);
    download_nodes(h->stream, coarse, C.res, C.g);
    CK(cudaStreamSynchronize(h->stream));
  });
}

int tmg_gpu_smooth(tmg_gpu_handle* h, int level, const double* f, double* u, int sweeps) {
  return guarded(h, [&] {
    need_single(h, "tmg_gpu_smooth");
    check_level(h, level);
    if (level < h->nc) need_setup(h);
    if (!h->have_moduli || !h->have_problem) fail(TMG_ERR_DIMENSION, "operator not set");
    Rank& R = *h->ranks[0];
    Level& L = R.lev[level];
    upload_nodes(h->stream, L.f, f, L.g);
    upload_nodes(h->stream, L.u[0], u, L.g);
    L.cur = 0;
    for (int s = 0; s < sweeps; ++s) {
      sweep_level(h, R, level, false, L.u[L.cur], L.u[L.cur ^ 1], L.f);
      L.cur ^= 1;
    }
    download_nodes(h->stream, u, L.u[L.cur], L.g);
    CK(cudaStreamSynchronize(h->stream));
  });
}

void* tmg_gpu_stream(tmg_gpu_handle* h) { return h ? static_cast<void*>(h->stream) : nullptr; }

long tmg_gpu_launch_count(tmg_gpu_handle* h) { return h ? h->launches : 0; }

int tmg_gpu_time_kernel(tmg_gpu_handle* h, int which, int reps, double* avg_ms, double* bytes) {
  return guarded(h, [&] {
    if (!h->have_moduli || !h->have_problem) fail(TMG_ERR_DIMENSION, "operator not set");
    Rank& R = *h->ranks[0];
    Level& F = R.fine();
    const double nodes = static_cast<double>(F.g.ncol) * (F.g.ny + 1);
    if (which < 0 || which > 2) fail(TMG_ERR_DIMENSION, "time_kernel: which must be 0, 1 or 2");
    auto launch = [&] {
      if (which == 0) {
        apply_level(h, R, h->nc, R.pbuf[0], R.ap);
      } else if (which == 1) {
        sweep_level(h, R, h->nc, false, F.u[0], F.u[1], R.r);
      } else {
        // the fused PCG update + two sweeps as the solve runs it, on scratch
        // outputs (the iterate stays untouched) with a plain reduction
        MarchArgs a = march_args(h, R, nullptr);
        a.f = R.r;
        a.u2 = R.ap;
        a.uc = R.pbuf[0];
        a.out2 = F.res;
        a.out1 = R.r2;
        a.out0 = F.u[1];
        a.rop = kRedPlain;
        a.red_out = R.scal;
        launch_march<StSweep01U, true>(h, a);
      }
    };
    for (int w = 0; w < 3; ++w) launch();
    CK(cudaEventRecord(h->ev[2], h->stream));
    for (int k = 0; k < reps; ++k) launch();
    CK(cudaEventRecord(h->ev[3], h->stream));
    CK(cudaEventSynchronize(h->ev[3]));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev[2], h->ev[3]));
    *avg_ms = ms / reps;
    // algorithmic bytes per node: apply reads u 16 +
    // E 8 + mask 1, writes 16; the sweep additionally reads f 16; the fused
    // update + two sweeps reads r_old, A p, x, p (16 each), E 8, mask 1 and
    // writes r, x, x2 (16 each)
    *bytes = nodes * (which == 0 ? 41.0 : (which == 1 ? 57.0 : 121.0));
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

#include "tmg_poisson.cuh"
