// Internal state of an msp_handle (include/msp.h) and the launch helpers shared by the
// parts of libmsp's single translation unit (solver.cu includes the parts in order).
#pragma once

// MSP-GMRES SOLVE phase on B200 (sm_100a): device data, upload, orchestration of
// the hot-path kernels (kernels.cuh), CUDA-graph replay of Arnoldi steps, and the
// C-ABI of include/msp.h.  Paper: arXiv 2208.08594 (PAPER.md "P:n").
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <functional>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/msp.h"
#include "comm.h"
#include "setup.h"
#include "kernels.cuh"
#include "setup_kernels.cuh"
#include "bilu_meta.cuh"
#include <nvtx3/nvToolsExt.h>

using namespace mspk;

namespace {

thread_local std::string g_last_error;

struct CudaError {
  cudaError_t e;
  std::string where;
};

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess) throw CudaError{_e, std::string(#call) + " @" + std::to_string(__LINE__)}; \
  } while (0)

inline unsigned nblk(size_t n, int t) { return (unsigned)((n + t - 1) / t); }

// NVTX range named after the SURVEY §8(a) row it covers (host-side: visible in profiles of
// direct launches and of SETUP; graph replays show the graph launch)
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

// Launch with programmatic stream serialisation (PDL, see kernels.cuh) when enabled.
template <typename... KArgs, typename... Args>
void klaunch(cudaStream_t s, bool pdl, void (*k)(KArgs...), dim3 grid, dim3 block, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...));
}

constexpr int kRecStride = 2 * kMaxV + 4;   // doubles per Arnoldi step record (host)

struct DevLevel {
  int32_t n = 0, ncolor = 0, nslices = 0;
  std::vector<int32_t> color_row;    // host: row range per color (permuted)
  std::vector<int32_t> color_slice;  // host: slice range per color
  int32_t* slice_row = nullptr;
  int32_t* slice_off = nullptr;
  int32_t* col = nullptr;
  double* val = nullptr;
  double* diag = nullptr;
  int32_t* agg = nullptr;            // permuted row -> next-level row
  int32_t* pt_ptr = nullptr;         // next-level row -> members (permuted rows)
  int32_t* pt_idx = nullptr;
  int32_t* perm = nullptr;           // natural -> permuted
  int32_t* inv = nullptr;            // permuted -> natural
  double *b = nullptr, *x = nullptr, *r = nullptr;
  int64_t nnz_alloc = 0;
  int lpr = 1;                       // lanes per row (coarse levels)
  int idx = 0;                       // AMG level index
  int uniform_w = 0;                 // > 0: every slice has this width (offsets arithmetic)
  int tail = 1 << 30;                // first color handled by the single-CTA tail kernel
  int32_t *d_color_row = nullptr, *d_color_slice = nullptr, *row_start = nullptr, *row_width = nullptr;
  // distributed level (dist_levels, NEXT-3): ghosts of x after the owned rows -- matrix
  // ghosts (per-color halo xh) then parent ghosts (next-level rows the prolongation into
  // the level above reads, halo ph); ghosts of r after the owned rows: members of owned
  // next-level aggregates (halo mh, before the restriction)
  int32_t ngx = 0, ngp = 0, ngm = 0;
  msp::HaloPlan xh, ph, mh;
};

}  // namespace

struct msp_handle {
  msp::Params prm;
  msp_config cfg{};
  int device = 0;
  cudaStream_t s = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::string err;
  std::vector<std::pair<void*, size_t>> allocs;
  int64_t bytes = 0;

  int32_t n = 0, b = 0, nc = 0;
  size_t N = 0;
  int64_t nnzb = 0;
  std::vector<int32_t> order;        // position -> natural cell
  std::vector<int32_t> src_entry;    // permuted entry -> natural entry
  std::vector<int32_t> nat_rp, nat_ci;  // natural pattern of the setup matrix (reuse check)
  int32_t* d_src = nullptr;          // device copy of src_entry
  double* stage = nullptr;           // natural-order values staging (reuse path)
  // BSR (internal positions), shared pattern for A and the BILU factors
  int32_t *rp = nullptr, *ci = nullptr, *dg = nullptr, *d_order = nullptr;
  double *Aval = nullptr, *Fval = nullptr, *W = nullptr, *Pcol = nullptr;
  double *Dn = nullptr, *wfull = nullptr, *r1 = nullptr;  // B_N stage (stages = 3)
  int32_t* l0_of_cell = nullptr;
  int32_t* cell_of_l0 = nullptr;     // inverse map: level-0 row -> internal cell
  // ABMC blocks
  int32_t bilu_ncolor = 0, max_blk = 1;
  std::vector<int32_t> color_blk;    // host
  int32_t* blk_ptr = nullptr;
  int32_t* bcnt = nullptr;           // per cell: #external L | #intra U << 8
  int4* islot = nullptr;             // per cell: entry of (i, c0 + s) for the block's slots s (diag at its own)
  // AMG
  std::vector<DevLevel> lv;
  int32_t nL = 0, ldA = 0;
  int sell_tpb = 128;                        // CTA size of the LPR=1 (level-0) sweep kernels
  bool pdl = true;                   // programmatic dependent launch for every kernel
  bool coarse_diag = false;
  double *Ainv = nullptr, *cdiag = nullptr, *bL = nullptr, *xL = nullptr;
  // work vectors
  double *z = nullptr, *r = nullptr, *wp = nullptr, *xin = nullptr, *bin = nullptr, *u = nullptr;
  double *V = nullptr;
  int V_m = -1;
  double* Z = nullptr;               // z_j = B v_j of every step of a cycle (zbasis mode), m x N
  int zbasis = 1;                    // MSP_ZBASIS=0: the cycle end applies B to V y instead of Z y'
  double *part = nullptr, *dh1 = nullptr, *dh2 = nullptr, *hcol = nullptr, *hpin = nullptr;
  double* hrec = nullptr;            // pinned: step j's Hessenberg record at hrec + j * kRecStride
  cudaEvent_t ev_step[2] = {nullptr, nullptr};   // end of step j (parity j & 1)
  int spec_steps = 1;                // MSP_SPEC_STEPS=0: no step enqueued ahead of the host's Givens update
  double *gv = nullptr, *hgv = nullptr;        // device Givens state / its pinned host copy
  cudaGraphExec_t cycle_exec = nullptr;        // one restart cycle as ONE graph (conditional steps)
  int cycle_m = -1;
  std::vector<int64_t> cycle_kernels;          // kernels of step j inside the cycle graph
  bool cycle_graphs = false;                   // MSP_CYCLE_GRAPH=1: one graph per restart cycle (measured: no gain)
  double *dst = nullptr, *dsum = nullptr;     // DCGS2 state (2 parities x (kMaxV+2)) and sums
  unsigned* ticket = nullptr;
  double* io = nullptr;              // staging for host<->device and natural-order vectors
  // graphs
  std::vector<cudaGraphExec_t> graphs;
  int graphs_m = -1;
  int kernels_per_step = 0;
  int64_t nlaunch = 0;
  std::vector<int64_t> graph_kernels;
  double* flush = nullptr;           // 256 MB L2-flush scratch (msp_time_kernel)
  double* ftmp = nullptr;            // msp_bilu_set_factors scratch
  // a9 per-slot metadata (bilu_meta.cuh; 4x4 blocks, single GPU)
  int4 *bm_f = nullptr, *bm_b = nullptr, *bm_cf = nullptr, *bm_cb = nullptr, *bm_sl = nullptr;
  int a8_ell = 1;                    // MSP_A8_ELL=0: pcol_resid4_kernel on the BSR pressure columns
  int32_t pell_w = 0;                // ELL width of the pressure columns (0: no ELL copy)
  int32_t* pell_c = nullptr;
  double* pell_v = nullptr;
  int bilu_meta = 1;                 // MSP_BILU_META=0: bilu_block_kernel (the distributed path's kernel)
  bool setup_on_gpu = true;          // NEXT-2: S1 + Galerkin on the GPU (MSP_HOST_SETUP=1: host)
  cusolverDnHandle_t cs = nullptr;   // coarsest inverse (created once, reused by rebuilds)
  bool gpu_s1 = false;               // the last SETUP computed S1 on the GPU
  std::vector<double> W_nat, App_nat;  // S1 results of the last SETUP (natural order), for parity
  cudaStream_t caller = nullptr;     // the caller's stream (msp_setup / msp_set_stream)
  cudaEvent_t ev_in = nullptr;       // orders h->s after the caller's prior work
  bool valid = false;                // false after a failed (re)SETUP: compute calls rejected
  // distributed (z-slab) mode: owned cells [0, n), ghost cells after them
  std::unique_ptr<msp::Comm> comm;   // null: single GPU
  cudaStream_t s2 = nullptr;         // side stream of the overlapped halo (distributed)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int32_t *rows_in = nullptr, *rows_bd = nullptr;   // slab-interior / boundary rows (cell space)
  int n_rows_in = 0, n_rows_bd = 0;
  bool overlap_halo = true;          // MSP_DIST_OVERLAP=0: exchange, then the whole SpMV
  bool setup_rank0 = true;           // MSP_DIST_SETUP_ALL=1: every rank runs the host setup
  bool fuse_halo = true;             // MSP_DIST_FUSE_PACK=0: separate pack kernel per exchange
  int rank = 0, nranks = 1;
  int n_ghost = 0, n0_ghost = 0;     // cell-space / level-0 ghosts
  msp::HaloPlan cell_halo;           // segments = BILU block colors
  msp::HaloPlan l0_halo;             // segments = level-0 PGS-MC colors
  int dist_D = 0;                    // levels 0..dist_D partitioned (msp_config.dist_levels, clamped)
  int n_own_l1 = 0, l1_cmax = 0;     // owned rows of level dist_D+1 (replicated part), max over ranks
  int32_t *own_l1_pt = nullptr, *own_l1_idx = nullptr, *l1_scatter = nullptr;
  double *l1_send = nullptr, *l1_recv = nullptr, *lred = nullptr;
  std::vector<int32_t> owned_cells;  // natural ids of the owned cells, ascending
  std::vector<int32_t> owner_in;     // caller partition (kept for rebuilds)
  // stats
  msp_stats st{};
  std::vector<int32_t> level_n;
  std::vector<int64_t> level_nnz;
  std::vector<int32_t> level_colors;

  template <class T>
  T* dalloc(size_t count) {
    size_t bytes_ = std::max<size_t>(count, 1) * sizeof(T);
    void* p = nullptr;
    if (cfg.alloc) {
      // the caller's stream: the library's stream waits on it before touching the memory
      // and is synchronised before every free, so a caching allocator may hand the
      // blocks of a closed handle to the next one (keyed by the long-lived caller stream)
      p = cfg.alloc(bytes_, (void*)caller, cfg.alloc_ctx);
      if (!p) throw CudaError{cudaErrorMemoryAllocation, "alloc callback"};
    } else {
      CK(cudaMalloc(&p, bytes_));
    }
    allocs.push_back({p, bytes_});
    bytes += (int64_t)bytes_;
    return (T*)p;
  }
  template <class T>
  T* upload(const std::vector<T>& v) {
    T* p = dalloc<T>(v.size());
    if (!v.empty()) CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    return p;
  }
  void free_all() {
    if (s) cudaStreamSynchronize(s);
    for (auto g : graphs) if (g) cudaGraphExecDestroy(g);
    graphs.clear();
    graphs_m = -1;
    for (auto& a : allocs) {
      if (cfg.free_fn) cfg.free_fn(a.first, cfg.alloc_ctx);
      else cudaFree(a.first);
    }
    allocs.clear();
    bytes = 0;
    ftmp = nullptr;
    flush = nullptr;
    lv.clear();
    V = nullptr;
    V_m = -1;
    Z = nullptr;
    cell_halo = msp::HaloPlan();
    l0_halo = msp::HaloPlan();
    if (hpin) { cudaFreeHost(hpin); hpin = nullptr; }
    if (hrec) { cudaFreeHost(hrec); hrec = nullptr; }
    if (hgv) { cudaFreeHost(hgv); hgv = nullptr; }
    if (cycle_exec) { cudaGraphExecDestroy(cycle_exec); cycle_exec = nullptr; }
    cycle_m = -1;
    gv = nullptr;
  }
};
