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

namespace {

msp::Params params_of(const msp_config* c) {
  msp::Params p;
  if (!c) return p;
  p.coarsest_max_dof = c->coarsest_max_dof;
  p.max_levels = c->max_levels;
  p.pre_sweeps = c->pre_sweeps;
  p.post_sweeps = c->post_sweeps;
  p.pair_passes = c->pair_passes;
  p.decoupling = c->decoupling;
  p.bilu_order = c->bilu_order;
  p.stages = c->stages;
  p.orth = c->orth;
  p.use_graphs = c->use_graphs;
  p.use_coop = c->use_coop;
  p.smoother = c->smoother;
  p.gs_chunk = c->gs_chunk;
  p.coarse_mode = c->coarse_mode;
  p.bilu_local = c->bilu_local;
  p.dist_levels = c->dist_levels;
  return p;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Host-side bounds checks of every index structure before it is uploaded (the kernels
// index with these arrays unchecked; compute-sanitizer is not available on this pool).
// A violation is a setup bug: MSP_EINVAL with the structure's name.
void check_index(bool ok, const char* what) {
  if (!ok) throw std::pair<int, std::string>(MSP_EINVAL, std::string("internal index check failed: ") + what);
}
void check_range(const std::vector<int32_t>& v, int64_t lo, int64_t hi, const char* what) {
  for (int32_t x : v) check_index(x >= lo && x < hi, what);
}
void check_ptr(const std::vector<int32_t>& p, int64_t n, int64_t total, const char* what) {
  check_index((int64_t)p.size() == n + 1 && p[0] == 0 && p[n] == total, what);
  for (int64_t i = 0; i < n; ++i) check_index(p[i] <= p[i + 1], what);
}
void check_perm(const std::vector<int32_t>& v, const char* what) {
  std::vector<char> seen(v.size(), 0);
  for (int32_t x : v) {
    check_index(x >= 0 && (size_t)x < v.size() && !seen[x], what);
    seen[x] = 1;
  }
}

// Copy the ABI's BSR into a host BlockMat (validating it).
// view: host values are read in place during the call (SETUP entry points), not copied.
msp_status read_bsr(const msp_bsr* A, int nc, msp::BlockMat& M, std::string& err, bool view = false) {
  if (!A || A->n_cells <= 0 || A->n_cells > INT32_MAX || A->block != nc + 1 || nc < 0 || nc > 7 ||
      !A->row_ptr || !A->col_idx || !A->values) {
    err = "msp_bsr: invalid shape/pointers (block must equal nc+1, nc <= 7)";
    return MSP_EINVAL;
  }
  const int32_t n = (int32_t)A->n_cells;
  const int b = A->block;
  M.n = n;
  M.b = b;
  M.rp.resize(n + 1);
  if (A->device >= 0) {
    if (cudaMemcpy(M.rp.data(), A->row_ptr, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost) != cudaSuccess) {
      err = "msp_bsr: device copy of row_ptr failed";
      return MSP_ECUDA;
    }
  } else {
    std::memcpy(M.rp.data(), A->row_ptr, sizeof(int32_t) * (n + 1));
  }
  const int64_t nnzb = M.rp[n];
  if (M.rp[0] != 0 || nnzb <= 0) { err = "msp_bsr: bad row_ptr"; return MSP_EINVAL; }
  M.ci.resize(nnzb);
  const size_t nv = (size_t)nnzb * b * b;
  if (A->device >= 0) {
    if (cudaMemcpy(M.ci.data(), A->col_idx, sizeof(int32_t) * nnzb, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(M.v.owned(nv), A->values, sizeof(double) * nv, cudaMemcpyDeviceToHost) != cudaSuccess) {
      err = "msp_bsr: device copy failed";
      return MSP_ECUDA;
    }
  } else {
    std::memcpy(M.ci.data(), A->col_idx, sizeof(int32_t) * nnzb);
    if (view) M.v.view(A->values, nv);
    else std::memcpy(M.v.owned(nv), A->values, sizeof(double) * nv);
  }
  for (int32_t i = 0; i < n; ++i) {
    if (M.rp[i + 1] < M.rp[i]) { err = "msp_bsr: row_ptr decreasing at row " + std::to_string(i); return MSP_EINVAL; }
    bool diag = false;
    for (int32_t e = M.rp[i]; e < M.rp[i + 1]; ++e) {
      if (M.ci[e] < 0 || M.ci[e] >= n) { err = "msp_bsr: column out of range in row " + std::to_string(i); return MSP_EINVAL; }
      if (e > M.rp[i] && M.ci[e] <= M.ci[e - 1]) { err = "msp_bsr: unsorted/duplicate column in row " + std::to_string(i); return MSP_EINVAL; }
      if (M.ci[e] == i) diag = true;
    }
    if (!diag) { err = "msp_bsr: missing diagonal block in row " + std::to_string(i); return MSP_EINVAL; }
  }
  return MSP_OK;
}

// row-major b x b blocks -> column-major
// Build a SELL-32 device level from CSR rows that are already in their final (color-
// major) order; color[i] non-decreasing.  Columns may reference ghost rows >= n (their
// x values are received by halo exchanges); x is sized n_total = n + ghosts.
// lanes per row: 1 for stencil-width rows; 2 when a color alone has enough rows to fill
// the GPU (C3 level 1: 35k rows per color, 88 -> 74 us per V-cycle vs 4 lanes); else 4 / 8
// by the row width (latency-bound small levels).  Distributed levels take the choice of
// the whole level (same per-row summation grouping as one GPU).
int choose_lpr(int64_t nnz, int32_t n, int32_t ncolor) {
  const double avg = (double)nnz / std::max<int32_t>(n, 1);
  const double rows_per_color = (double)n / std::max(ncolor, 1);
  return (avg <= 8.0) ? 1 : (rows_per_color >= 16384.0 ? 2 : (avg <= 20.0 ? 4 : 8));
}

void upload_level_rows(msp_handle* h, DevLevel& L, int32_t n, int32_t n_total, const std::vector<int32_t>& rp,
                       const std::vector<int32_t>& ci, const std::vector<double>& v, int32_t ncolor,
                       const std::vector<int32_t>& color, int lpr_force = 0, int32_t n_r = -1) {
  L.n = n;
  L.ncolor = ncolor;
  std::vector<int32_t> cnt(ncolor + 1, 0);
  for (int32_t i = 0; i < n; ++i) cnt[color[i] + 1]++;
  for (int32_t c = 0; c < ncolor; ++c) cnt[c + 1] += cnt[c];
  L.color_row = cnt;
  std::vector<int32_t> slice_row, slice_off;
  L.color_slice.assign(ncolor + 1, 0);
  for (int32_t c = 0; c < ncolor; ++c) {
    for (int32_t r0 = cnt[c]; r0 < cnt[c + 1]; r0 += kSell) slice_row.push_back(r0);
    L.color_slice[c + 1] = (int32_t)slice_row.size();
  }
  L.nslices = (int32_t)slice_row.size();
  slice_row.push_back(n);
  slice_off.assign(L.nslices + 1, 0);
  std::vector<int32_t> sw(L.nslices, 0);
  int32_t wmax = 0;
  int64_t tot = 0;
#pragma omp parallel for schedule(static) reduction(max : wmax) reduction(+ : tot)
  for (int32_t s = 0; s < L.nslices; ++s) {
    int32_t r1 = std::min(slice_row[s] + kSell, slice_row[s + 1]);
    int32_t w = 0;
    for (int32_t p = slice_row[s]; p < r1; ++p) w = std::max(w, (int32_t)(rp[p + 1] - rp[p]) - 1);
    sw[s] = std::max(w, 0);
    wmax = std::max(wmax, sw[s]);
    tot += sw[s];
  }
  // narrow rows (one lane per row, <= 8 entries) with near-uniform slice widths: pad every
  // slice to the widest so that slice offsets and row ranges are arithmetic (the level-0
  // sweep kernel then needs no slice metadata loads); <= 5 % extra entries
  const double avg_row = (double)rp[n] / std::max<int32_t>(n, 1);
  const bool uniform = avg_row <= 8.0 && wmax > 0 && wmax <= 8 && (double)wmax * L.nslices <= 1.05 * (double)tot &&
                       true;
  for (int32_t s = 0; s < L.nslices; ++s) slice_off[s + 1] = slice_off[s] + (uniform ? wmax : sw[s]) * kSell;
  L.uniform_w = uniform ? wmax : 0;
  std::vector<int32_t> col(std::max<int32_t>(slice_off[L.nslices], 1));
  std::vector<double> val(col.size(), 0.0), diag(n, 0.0);
#pragma omp parallel for schedule(static)
  for (int32_t s = 0; s < L.nslices; ++s) {
    const int32_t w = (slice_off[s + 1] - slice_off[s]) / kSell;
    for (int32_t l = 0; l < kSell; ++l) {
      const int32_t p = slice_row[s] + l;
      const bool valid = p < slice_row[s + 1];
      int k = 0;
      if (valid) {
        for (int32_t e = rp[p]; e < rp[p + 1]; ++e) {
          if (ci[e] == p) { diag[p] = v[e]; continue; }
          col[slice_off[s] + k * kSell + l] = ci[e];
          val[slice_off[s] + k * kSell + l] = v[e];
          ++k;
        }
      }
      for (; k < w; ++k) {
        col[slice_off[s] + k * kSell + l] = valid ? p : slice_row[s];
        val[slice_off[s] + k * kSell + l] = 0.0;
      }
    }
  }
  L.nnz_alloc = slice_off[L.nslices];
  {
    L.lpr = lpr_force > 0 ? lpr_force : choose_lpr(rp[n], n, ncolor);
    if (const char* e = std::getenv("MSP_LPR")) L.lpr = std::atoi(e);
    {
      char key[32];
      std::snprintf(key, sizeof key, "MSP_LPR_L%d", L.idx);
      if (const char* e = std::getenv(key)) L.lpr = std::atoi(e);
    }
    int tail_rows = 0, t = ncolor;
    const int lim_env = std::getenv("MSP_TAIL_ROWS") ? std::atoi(std::getenv("MSP_TAIL_ROWS")) : 2048;
    const int lim_col = std::getenv("MSP_TAIL_COLOR") ? std::atoi(std::getenv("MSP_TAIL_COLOR")) : 1024;
    while (t > 1) {
      const int rows = cnt[t] - cnt[t - 1];
      if (rows * L.lpr > lim_col || tail_rows + rows * L.lpr > lim_env) break;
      tail_rows += rows * L.lpr;
      --t;
    }
    L.tail = (ncolor - t >= 2) ? t : (1 << 30);
  }
  {
    std::vector<int32_t> rs(n), rw(n);
#pragma omp parallel for schedule(static)
    for (int32_t s = 0; s < L.nslices; ++s)
      for (int32_t p = slice_row[s]; p < slice_row[s + 1]; ++p) {
        rs[p] = slice_off[s] + (p - slice_row[s]);
        rw[p] = (slice_off[s + 1] - slice_off[s]) / kSell;
      }
    L.row_start = h->upload(rs);
    L.row_width = h->upload(rw);
    L.d_color_row = h->upload(L.color_row);
    L.d_color_slice = h->upload(L.color_slice);
  }
  check_range(col, 0, n_total, "level SELL column");
  check_index(slice_off[L.nslices] == (int32_t)L.nnz_alloc || L.nslices == 0, "level SELL slice offsets");
  L.slice_row = h->upload(slice_row);
  L.slice_off = h->upload(slice_off);
  L.col = h->upload(col);
  L.val = h->upload(val);
  L.diag = h->upload(diag);
  L.b = h->dalloc<double>(n);
  L.x = h->dalloc<double>(n_total);
  L.r = h->dalloc<double>(n_r >= 0 ? n_r : n);
}

// Build a SELL-32 device level from a natural-order CSR + coloring (rows permuted by
// (color, natural index)).
void upload_level(msp_handle* h, DevLevel& L, const msp::SpMat& A, int32_t ncolor,
                  const std::vector<int32_t>& color, std::vector<int32_t>& perm_out) {
  const int32_t n = A.n;
  std::vector<int32_t> cnt(ncolor + 1, 0);
  for (int32_t i = 0; i < n; ++i) cnt[color[i] + 1]++;
  for (int32_t c = 0; c < ncolor; ++c) cnt[c + 1] += cnt[c];
  std::vector<int32_t> perm(n), inv(n), pcolor(n);
  {
    std::vector<int32_t> f(cnt.begin(), cnt.end() - 1);
    for (int32_t i = 0; i < n; ++i) { perm[i] = f[color[i]]++; inv[perm[i]] = i; }
  }
  std::vector<int32_t> rp(n + 1, 0), ci(A.ci.size());
  std::vector<double> v(A.ci.size());
  for (int32_t p = 0; p < n; ++p) {
    const int32_t i = inv[p];
    pcolor[p] = color[i];
    rp[p + 1] = rp[p] + (A.rp[i + 1] - A.rp[i]);
    int32_t q = rp[p];
    for (int32_t e = A.rp[i]; e < A.rp[i + 1]; ++e, ++q) { ci[q] = perm[A.ci[e]]; v[q] = A.v[e]; }
  }
  upload_level_rows(h, L, n, n, rp, ci, v, ncolor, pcolor);
  L.perm = h->upload(perm);
  L.inv = h->upload(inv);
  perm_out = perm;
}

struct SetupTimer {
  bool on = std::getenv("MSP_SETUP_VERBOSE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[msp setup] %-28s %8.3f s\n", what, std::chrono::duration<double>(n - t).count());
    t = n;
  }
};

// per-cell counts of external L / intra-block U entries (bilu_block_kernel), in global
// positions
std::vector<int32_t> block_counts(const msp::HostSetup& S, const std::vector<int32_t>& rp,
                                  const std::vector<int32_t>& ci, const std::vector<int32_t>& dg) {
  std::vector<int32_t> cnt(S.n, 0);
  for (size_t k = 0; k + 1 < S.blk_ptr.size(); ++k) {
    const int32_t c0 = S.blk_ptr[k], c1 = S.blk_ptr[k + 1];
    for (int32_t i = c0; i < c1; ++i) {
      int32_t next = 0, nint = 0;
      for (int32_t e = rp[i]; e < dg[i]; ++e) if (ci[e] < c0) ++next;
      for (int32_t e = dg[i] + 1; e < rp[i + 1]; ++e) if (ci[e] < c1) ++nint;
      if (next > 255 || nint > 255) throw std::pair<int, std::string>(MSP_EINVAL, "BILU: row too long for the block kernel");
      cnt[i] = next | (nint << 8);
    }
  }
  return cnt;
}

// Partitioned AMG level l >= 1 of rank `me` (dist_levels, host-only integer work): owned
// rows in the global row order, ghosts in receive order (peer-major, then global row
// order, which is color-major) and, per peer, the rows sent to it in the same order --
// matrix ghosts / x sends (the sweeps), parent ghosts / sends (the prolongation into
// level l-1) and member ghosts / sends of r (the restriction into level l+1).
struct LevelPlan {
  std::vector<int32_t> rows, gx, gp, gm;
  std::vector<std::vector<int32_t>> needx, needp, needm;
};
LevelPlan plan_level(const msp::HostSetup& S, const std::vector<std::vector<int32_t>>& perms,
                     const std::vector<std::vector<int32_t>>& own, int l, int me, int P) {
  const msp::SpMat& Al = S.lv[l].A;
  const int32_t nl = Al.n;
  const auto& ow = own[l];
  const auto& pl = perms[l];
  auto by_row = [&](int32_t x, int32_t y) { return pl[x] < pl[y]; };
  auto by_owner_row = [&](int32_t x, int32_t y) { return ow[x] != ow[y] ? ow[x] < ow[y] : pl[x] < pl[y]; };
  LevelPlan R;
  for (int32_t i = 0; i < nl; ++i) if (ow[i] == me) R.rows.push_back(i);
  std::sort(R.rows.begin(), R.rows.end(), by_row);
  R.needx.assign(P, {});
  R.needp.assign(P, {});
  R.needm.assign(P, {});
  {
    std::vector<uint8_t> mk(nl, 0);
    for (int32_t i = 0; i < nl; ++i) {
      const int t = ow[i];
      for (int32_t e = Al.rp[i]; e < Al.rp[i + 1]; ++e) {
        const int32_t d = Al.ci[e];
        const int o = ow[d];
        if (o == t) continue;
        if (o == me) R.needx[t].push_back(d);
        if (t == me && !mk[d]) { mk[d] = 1; R.gx.push_back(d); }
      }
    }
  }
  {
    const auto& aggp = S.lv[l - 1].agg;
    const auto& owp = own[l - 1];
    std::vector<uint8_t> mk(nl, 0);
    for (int32_t i = 0; i < S.lv[l - 1].A.n; ++i) {
      const int32_t I = aggp[i];
      const int t = owp[i], o = ow[I];
      if (o == t) continue;
      if (o == me) R.needp[t].push_back(I);
      if (t == me && !mk[I]) { mk[I] = 1; R.gp.push_back(I); }
    }
  }
  {
    const auto& aggn = S.lv[l].agg;
    const auto& own_n = own[l + 1];
    for (int32_t i = 0; i < nl; ++i) {
      const int t = own_n[aggn[i]], o = ow[i];
      if (o == t) continue;
      if (o == me) R.needm[t].push_back(i);
      if (t == me) R.gm.push_back(i);
    }
  }
  for (int q = 0; q < P; ++q)
    for (auto* v : {&R.needx[q], &R.needp[q], &R.needm[q]}) {
      std::sort(v->begin(), v->end(), by_row);
      v->erase(std::unique(v->begin(), v->end()), v->end());
    }
  std::sort(R.gx.begin(), R.gx.end(), by_owner_row);
  std::sort(R.gp.begin(), R.gp.end(), by_owner_row);
  std::sort(R.gm.begin(), R.gm.end(), by_owner_row);
  return R;
}

// owners of the rows of levels 0..upto: a level-(l+1) row (aggregate of level-l rows)
// lives on the owner of its lowest-index member
std::vector<std::vector<int32_t>> level_owners(const msp::HostSetup& S, const std::vector<int32_t>& own_cell,
                                               int upto) {
  std::vector<std::vector<int32_t>> own(upto + 1);
  own[0] = own_cell;
  for (int l = 0; l + 1 <= upto; ++l) {
    const auto& agg = S.lv[l].agg;
    own[l + 1].assign(S.lv[l].n_next, -1);
    for (int32_t i = S.lv[l].A.n - 1; i >= 0; --i) own[l + 1][agg[i]] = own[l][i];
  }
  return own;
}

// color-major permutation of a level (natural row -> global row), as upload_level
std::vector<int32_t> level_perm(const msp::HostLevel& Lv) {
  std::vector<int32_t> cnt(Lv.ncolor + 1, 0), perm(Lv.A.n);
  for (int32_t c : Lv.color) cnt[c + 1]++;
  for (int c = 0; c < Lv.ncolor; ++c) cnt[c + 1] += cnt[c];
  for (int32_t i = 0; i < Lv.A.n; ++i) perm[i] = cnt[Lv.color[i]]++;
  return perm;
}

void dist_localize(msp_handle* h, const msp::BlockMat& A, const msp::HostSetup& S, const std::vector<int32_t>& rp,
                   const std::vector<int32_t>& ci, const std::vector<int32_t>& dg, const std::vector<int32_t>& src,
                   const std::vector<double>& F, const std::vector<std::vector<int32_t>>& perms,
                   const double* dF = nullptr, const double* dAnat = nullptr);


// BILU block kernels: per cell i of aggregate block [c0, c1) (<= 4 cells), the entry index
// of (i, c0 + s) for every slot s of the block (-1: no coupling), with the diagonal entry
// in the cell's own slot, so the intra-block triangle needs no column search.
std::vector<int4> make_islot(int32_t n, const std::vector<int32_t>& rp, const std::vector<int32_t>& ci,
                             const std::vector<int32_t>& dg, const std::vector<int32_t>& blk_ptr) {
  std::vector<int4> sl(n, make_int4(-1, -1, -1, -1));
  for (size_t k = 0; k + 1 < blk_ptr.size(); ++k) {
    const int32_t c0 = blk_ptr[k], c1 = blk_ptr[k + 1];
    if (c1 - c0 > 4) continue;                          // (block kernels need <= 4 cells)
    for (int32_t i = c0; i < c1; ++i) {
      int v[4] = {-1, -1, -1, -1};
      v[i - c0] = dg[i];
      for (int32_t e = rp[i]; e < rp[i + 1]; ++e)
        if (ci[e] >= c0 && ci[e] < c1 && ci[e] != i) v[ci[e] - c0] = e;
      sl[i] = make_int4(v[0], v[1], v[2], v[3]);
    }
  }
  return sl;
}

// Device scratch for the GPU SETUP steps (freed on scope exit, stream-ordered).
// Large host -> device uploads of PAGEABLE caller buffers (the block values at SETUP and at
// msp_update): staged through a pinned ring in 32 MB chunks, the host copies of a chunk
// split over OpenMP threads while the previous chunks' DMAs run, instead of the driver's
// single-threaded pageable staging (~11 GB/s measured).  Pinned / small buffers: direct.
void h2d_large(cudaStream_t s, void* dst, const void* src, size_t bytes) {
  constexpr size_t kChunk = (size_t)32 << 20;
  constexpr int kSlots = 4;
  cudaPointerAttributes a;
  const bool pinned = cudaPointerGetAttributes(&a, src) == cudaSuccess && a.type != cudaMemoryTypeUnregistered;
  cudaGetLastError();
  if (bytes < 2 * kChunk || pinned) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return;
  }
  static std::mutex mu;
  static char* ring = nullptr;
  static cudaEvent_t ev[kSlots];
  static bool used[kSlots];
  std::lock_guard<std::mutex> lk(mu);
  if (!ring) {
    CK(cudaMallocHost(&ring, kChunk * kSlots));
    for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  const char* sp = static_cast<const char*>(src);
  char* dp = static_cast<char*>(dst);
  size_t i = 0;
  for (size_t off = 0; off < bytes; off += kChunk, ++i) {
    const int k = (int)(i % kSlots);
    const size_t len = std::min(kChunk, bytes - off);
    if (used[k]) CK(cudaEventSynchronize(ev[k]));
    char* slot = ring + (size_t)k * kChunk;
    constexpr size_t kPiece = (size_t)1 << 20;
    const int64_t np = (int64_t)((len + kPiece - 1) / kPiece);
#pragma omp parallel for schedule(static) num_threads(8)
    for (int64_t q = 0; q < np; ++q) {
      const size_t o = (size_t)q * kPiece;
      std::memcpy(slot + o, sp + off + o, std::min(kPiece, len - o));
    }
    CK(cudaMemcpyAsync(dp + off, slot, len, cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(ev[k], s));
    used[k] = true;
  }
}

// SETUP temporaries come from a library-private stream-ordered pool that keeps its memory
// across the synchronisations of one SETUP (release threshold = max; the default pool
// returns freed memory at every sync, and re-mapping GBs per Galerkin product cost up to
// 0.5 s); trimmed to zero when the SETUP ends (setup_pool_trim).
cudaMemPool_t setup_pool() {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = pools.find(dev);
  if (it != pools.end()) return it->second;
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.handleTypes = cudaMemHandleTypeNone;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool;
  CK(cudaMemPoolCreate(&pool, &props));
  uint64_t thr = UINT64_MAX;
  CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  pools[dev] = pool;
  return pool;
}
void setup_pool_trim(cudaStream_t s) {
  static const bool trim = !std::getenv("MSP_SETUP_POOL_TRIM") || std::atoi(std::getenv("MSP_SETUP_POOL_TRIM")) != 0;
  if (!trim) return;
  CK(cudaStreamSynchronize(s));
  CK(cudaMemPoolTrimTo(setup_pool(), 0));
}

struct DBuf {
  void* p = nullptr;
  cudaStream_t s;
  DBuf(size_t bytes, cudaStream_t st) : s(st) {
    CK(cudaMallocFromPoolAsync(&p, std::max<size_t>(bytes, 16), setup_pool(), s));
  }
  ~DBuf() { cudaFreeAsync(p, s); }
  template <class T> T* as() const { return static_cast<T*>(p); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
};
template <class T>
void h2d(cudaStream_t s, T* d, const std::vector<T>& v) {
  if (!v.empty()) CK(cudaMemcpyAsync(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, s));
}

// NEXT-2, S1 on the GPU (R4): block column sums (TI) or diagonal blocks (QI), the
// decoupling weights and A_PP = W^T A Pi_P, explicitly rounded in the host/oracle order
// (setup_kernels.cuh) -> bit-identical W and A_PP, returned to the host for the greedy
// steps (NPAIR, colorings) that follow.
std::unique_ptr<DBuf> gpu_setup_s1(cudaStream_t s, int decoupling, const msp::BlockMat& A, msp::HostSetup& S,
                                   DBuf** dApp_out = nullptr) {
  Nvtx nv("S1 weights + A_PP (GPU)");
  const int32_t n = A.n;
  const int b = A.b, bb = b * b;
  const int64_t nnzb = (int64_t)A.ci.size();
  std::unique_ptr<DBuf> dAp(new DBuf((size_t)nnzb * bb * sizeof(double), s));
  DBuf& dA = *dAp;
  DBuf dC((size_t)n * bb * sizeof(double), s), dW((size_t)n * b * sizeof(double), s);
  DBuf* dPp = new DBuf((size_t)nnzb * sizeof(double), s);
  std::unique_ptr<DBuf> dPown(dApp_out ? nullptr : dPp);
  if (dApp_out) *dApp_out = dPp;
  DBuf& dP = *dPp;
  DBuf dnz((size_t)nnzb, s);
  DBuf drp((size_t)(n + 1) * 4, s), dbad(4, s);
  h2d_large(s, dA.p, A.v.data(), sizeof(double) * A.v.size());
  h2d(s, drp.as<int32_t>(), A.rp);
  CK(cudaMemsetAsync(dbad.p, 0xff, 4, s));
  std::unique_ptr<DBuf> dcp, dce;
  if (decoupling == 2) {                        // CSC of the block pattern, rows ascending
    std::vector<int32_t> cp(n + 1, 0), ce(nnzb);
    for (int32_t c : A.ci) cp[c + 1]++;
    for (int32_t c = 0; c < n; ++c) cp[c + 1] += cp[c];
    std::vector<int32_t> f(cp.begin(), cp.end() - 1);
    for (int32_t p = 0; p < n; ++p)
      for (int32_t e = A.rp[p]; e < A.rp[p + 1]; ++e) ce[f[A.ci[e]]++] = e;
    dcp.reset(new DBuf((size_t)(n + 1) * 4, s));
    dce.reset(new DBuf((size_t)nnzb * 4, s));
    h2d(s, dcp->as<int32_t>(), cp);
    h2d(s, dce->as<int32_t>(), ce);
  } else if (decoupling == 1) {
    std::vector<int32_t> dg(n, -1);
    for (int32_t c = 0; c < n; ++c)
      for (int32_t e = A.rp[c]; e < A.rp[c + 1]; ++e) if (A.ci[e] == c) dg[c] = e;
    dcp.reset(new DBuf((size_t)n * 4, s));
    h2d(s, dcp->as<int32_t>(), dg);
  }
  const unsigned gC = nblk((size_t)n * bb, 256), gn = nblk(n, 128);
  switch (b) {
#define CASE(BV)                                                                                                  \
  case BV:                                                                                                        \
    if (decoupling == 2)                                                                                   \
      klaunch(s, false, colsum_kernel<BV>, gC, 256, n, (const int*)dcp->p, (const int*)dce->p, (const double*)dA.p, \
              dC.as<double>());                                                                                   \
    else if (decoupling == 1)                                                                              \
      klaunch(s, false, diagblock_kernel<BV>, gC, 256, n, (const int*)dcp->p, (const double*)dA.p, dC.as<double>()); \
    if (decoupling != 0) klaunch(s, false, weights_kernel<BV>, gn, 128, n, (const double*)dC.p, dW.as<double>(), \
                                        dbad.as<int>());                                                          \
    break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
  }
  S.W.assign((size_t)n * b, 0.0);
  if (decoupling == 0) {
    for (int32_t c = 0; c < n; ++c) S.W[(size_t)c * b] = 1.0;
    h2d(s, dW.as<double>(), S.W);
  }
  switch (b) {
#define CASE(BV) case BV: klaunch(s, false, app_kernel<BV>, gn, 128, n, (const int*)drp.p, (const double*)dW.p, \
                                  (const double*)dA.p, dP.as<double>()); \
                          klaunch(s, false, block_nonzero_kernel<BV>, nblk(nnzb, 256), 256, nnzb, (const double*)dA.p, \
                                  dnz.as<uint8_t>()); break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
  }
  S.block_nz.resize(nnzb);
  CK(cudaMemcpyAsync(S.block_nz.data(), dnz.p, nnzb, cudaMemcpyDeviceToHost, s));
  int bad = -1;
  S.App.n = n;
  S.App.rp = A.rp;
  S.App.ci = A.ci;
  S.App.v.resize(nnzb);
  CK(cudaMemcpyAsync(&bad, dbad.p, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(S.W.data(), dW.p, sizeof(double) * S.W.size(), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(S.App.v.data(), dP.p, sizeof(double) * nnzb, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (bad >= 0) throw std::pair<int, std::string>(MSP_ESINGULAR, "decoupling: singular N-N block at cell " + std::to_string(bad));
  return dAp;                                         // A's values on the device (natural order)
}

// Device-resident chain of the Galerkin products of one SETUP: the fine operand of the
// next product is the previous product's result (or A_PP from S1) already on the device,
// so only the aggregate map goes up and the coarse matrix (needed by the host NPAIR /
// colorings) comes down.  Buffers grow on demand and live for the SETUP.
struct RapChain {
  cudaStream_t s = nullptr;
  int32_t n = -1;                          // rows of the device-resident fine matrix (-1: none)
  int64_t nnz = -1;
  const double* host_v = nullptr;          // host buffer the device copy mirrors
  std::vector<std::unique_ptr<DBuf>> keep;
  int32_t *rp = nullptr, *ci = nullptr;
  double* v = nullptr;
};

// NEXT-2, S3 Galerkin product on the GPU (setup_kernels.cuh: pattern and values per
// coarse row in the specified summation order -> bit-identical to the host product).
// Returns nonzero (host fallback) when a coarse row has more than kRapMax candidates.
int gpu_rap(RapChain& ch, const msp::SpMat& A, const std::vector<int32_t>& agg, int32_t nagg, msp::SpMat& C) {
  cudaStream_t s = ch.s;
  const int32_t n = A.n;
  const int64_t nnz = (int64_t)A.ci.size();
  if (!(ch.n == n && ch.nnz == nnz && ch.host_v == A.v.data())) {     // fine matrix not resident
    ch.keep.clear();
    ch.keep.emplace_back(new DBuf((size_t)(n + 1) * 4, s));
    ch.keep.emplace_back(new DBuf((size_t)nnz * 4, s));
    ch.keep.emplace_back(new DBuf((size_t)nnz * 8, s));
    ch.rp = ch.keep[0]->as<int32_t>();
    ch.ci = ch.keep[1]->as<int32_t>();
    ch.v = ch.keep[2]->as<double>();
    h2d(s, ch.rp, A.rp);
    h2d(s, ch.ci, A.ci);
    h2d(s, ch.v, A.v);
  }
  std::vector<int32_t> mp(nagg + 1, 0), mi(n);
  for (int32_t i = 0; i < n; ++i) mp[agg[i] + 1]++;
  for (int32_t I = 0; I < nagg; ++I) mp[I + 1] += mp[I];
  {
    std::vector<int32_t> f(mp.begin(), mp.end() - 1);
    for (int32_t i = 0; i < n; ++i) mi[f[agg[i]]++] = i;
  }
  DBuf dagg((size_t)n * 4, s);
  DBuf dmp((size_t)(nagg + 1) * 4, s), dmi((size_t)n * 4, s), dcnt((size_t)(nagg + 1) * 4, s), dov(4, s);
  h2d(s, dagg.as<int32_t>(), agg);
  h2d(s, dmp.as<int32_t>(), mp);
  h2d(s, dmi.as<int32_t>(), mi);
  CK(cudaMemsetAsync(dov.p, 0, 4, s));
  const unsigned g = nblk(nagg, 128);
  klaunch(s, false, rap_count_kernel, g, 128, nagg, (const int*)dmp.p, (const int*)dmi.p, (const int*)ch.rp,
          (const int*)ch.ci, (const int*)dagg.p, dcnt.as<int>(), dov.as<int>());
  std::vector<int32_t> cnt(nagg);
  int ov = 0;
  CK(cudaMemcpyAsync(cnt.data(), dcnt.p, sizeof(int32_t) * nagg, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&ov, dov.p, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (ov) return 1;
  C.n = nagg;
  C.rp.assign(nagg + 1, 0);
  for (int32_t I = 0; I < nagg; ++I) C.rp[I + 1] = C.rp[I] + cnt[I];
  const int64_t cn = C.rp[nagg];
  std::unique_ptr<DBuf> dcrp(new DBuf((size_t)(nagg + 1) * 4, s)), dcci(new DBuf((size_t)cn * 4, s)),
      dcv(new DBuf((size_t)cn * 8, s));
  h2d(s, dcrp->as<int32_t>(), C.rp);
  klaunch(s, false, rap_fill_kernel, g, 128, nagg, (const int*)dmp.p, (const int*)dmi.p, (const int*)ch.rp,
          (const int*)ch.ci, (const double*)ch.v, (const int*)dagg.p, (const int*)dcrp->p, dcci->as<int>(),
          dcv->as<double>());
  C.ci.resize(cn);
  C.v.resize(cn);
  CK(cudaMemcpyAsync(C.ci.data(), dcci->p, sizeof(int32_t) * cn, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(C.v.data(), dcv->p, sizeof(double) * cn, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  // the product stays resident as the next fine operand (C is moved, its buffer kept)
  ch.keep.clear();
  ch.keep.push_back(std::move(dcrp));
  ch.keep.push_back(std::move(dcci));
  ch.keep.push_back(std::move(dcv));
  ch.rp = ch.keep[0]->as<int32_t>();
  ch.ci = ch.keep[1]->as<int32_t>();
  ch.v = ch.keep[2]->as<double>();
  ch.n = nagg;
  ch.nnz = cn;
  ch.host_v = C.v.data();
  return 0;
}

// ---- rank-0 SETUP of the distributed path: the result of S1-S4 (weights, A_PP, levels,
// colorings, aggregates, ABMC order) serialised on rank 0 and broadcast to the other ranks
// through the handle's Comm (NCCL broadcast / loopback copy), instead of every rank
// running the same host setup on the whole matrix.
struct SetupBlob {
  std::vector<char> b;
  size_t rd = 0;
  void put(const void* p, size_t n) { const char* c = (const char*)p; b.insert(b.end(), c, c + n); }
  void get(void* p, size_t n) {
    if (rd + n > b.size()) throw std::pair<int, std::string>(MSP_ECUDA, "setup broadcast: truncated");
    std::memcpy(p, b.data() + rd, n);
    rd += n;
  }
  template <class T> void vec(const std::vector<T>& v) { const uint64_t n = v.size(); put(&n, 8); put(v.data(), n * sizeof(T)); }
  template <class T> void vec(std::vector<T>& v, bool) { uint64_t n = 0; get(&n, 8); v.resize(n); get(v.data(), n * sizeof(T)); }
  template <class T> void val(const T& x) { put(&x, sizeof(T)); }
  template <class T> void val(T& x, bool) { get(&x, sizeof(T)); }
  void mat(const msp::SpMat& m) { val(m.n); vec(m.rp); vec(m.ci); vec(m.v); }
  void mat(msp::SpMat& m, bool) { val(m.n, true); vec(m.rp, true); vec(m.ci, true); vec(m.v, true); }
};

void pack_setup(const msp::HostSetup& S, SetupBlob& o) {
  o.val(S.n); o.vec(S.W); o.mat(S.App);
  const int32_t L = (int32_t)S.lv.size();
  o.val(L);
  for (const auto& l : S.lv) { o.mat(l.A); o.val(l.ncolor); o.vec(l.color); o.vec(l.agg); o.val(l.n_next); }
  o.mat(S.Ac); o.val(S.coarse_diag); o.vec(S.order); o.vec(S.pos); o.val(S.bilu_ncolor);
  o.vec(S.blk_ptr); o.vec(S.color_blk_ptr); o.vec(S.level1_agg);
}

void unpack_setup(SetupBlob& o, msp::HostSetup& S) {
  o.val(S.n, true); o.vec(S.W, true); o.mat(S.App, true);
  int32_t L = 0;
  o.val(L, true);
  S.lv.resize(L);
  for (auto& l : S.lv) { o.mat(l.A, true); o.val(l.ncolor, true); o.vec(l.color, true); o.vec(l.agg, true); o.val(l.n_next, true); }
  o.mat(S.Ac, true); o.val(S.coarse_diag, true); o.vec(S.order, true); o.vec(S.pos, true); o.val(S.bilu_ncolor, true);
  o.vec(S.blk_ptr, true); o.vec(S.color_blk_ptr, true); o.vec(S.level1_agg, true);
}

// Collective: rank 0 broadcasts {status, bytes} and then the blob (as doubles).
void bcast_setup(msp_handle* h, int& status, std::string& err, SetupBlob& blob) {
  cudaStream_t s = h->s;
  DBuf hdr(16, s);
  double hv[2] = {(double)status, (double)blob.b.size()};
  if (h->rank == 0) CK(cudaMemcpyAsync(hdr.p, hv, 16, cudaMemcpyHostToDevice, s));
  h->comm->broadcast(s, hdr.as<double>(), 2, 0);
  CK(cudaMemcpyAsync(hv, hdr.p, 16, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  status = (int)hv[0];
  if (status) {
    if (h->rank != 0) err = "setup failed on rank 0 (status " + std::to_string(status) + ")";
    return;
  }
  const size_t bytes = (size_t)hv[1], nd = (bytes + 7) / 8;
  DBuf dev(nd * 8, s);
  if (h->rank == 0) {
    blob.b.resize(nd * 8, 0);
    CK(cudaMemcpyAsync(dev.p, blob.b.data(), nd * 8, cudaMemcpyHostToDevice, s));
  }
  h->comm->broadcast(s, dev.as<double>(), (int)nd, 0);
  if (h->rank != 0) {
    blob.b.resize(nd * 8);
    CK(cudaMemcpyAsync(blob.b.data(), dev.p, nd * 8, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  blob.b.resize(bytes);
  blob.rd = 0;
}

// Global BILU(0) factorization on the GPU (distributed handles): every rank factorizes the
// whole matrix per block color exactly as the single-GPU setup does (bit-identical
// factors), then dist_localize keeps its rows.  Returns the factors, row-major blocks in
// the global permuted entry order.
std::unique_ptr<DBuf> gpu_bilu_global(msp_handle* h, const msp::BlockMat& A, const msp::HostSetup& S,
                                      const std::vector<int32_t>& rp, const std::vector<int32_t>& ci,
                                      const std::vector<int32_t>& dg, const std::vector<int32_t>& src, const DBuf& dAnat,
                                      const std::vector<int32_t>& masked) {
  Nvtx nv("S4 BILU(0) factorization (GPU, global)");
  cudaStream_t s = h->s;
  const int b = A.b, bb = b * b;
  const size_t ne = ci.size();
  std::unique_ptr<DBuf> F(new DBuf(ne * bb * sizeof(double), s));
  DBuf drp(rp.size() * 4, s), dci(ne * 4, s), ddg(dg.size() * 4, s), dsrc(ne * 4, s), dbp(S.blk_ptr.size() * 4, s),
      dbad(4, s);
  h2d(s, drp.as<int32_t>(), rp);
  h2d(s, dci.as<int32_t>(), ci);
  h2d(s, ddg.as<int32_t>(), dg);
  h2d(s, dsrc.as<int32_t>(), src);
  h2d(s, dbp.as<int32_t>(), S.blk_ptr);
  CK(cudaMemsetAsync(dbad.p, 0xff, 4, s));
  std::unique_ptr<DBuf> dmask;                        // rank-local BILU: couplings across owners
  if (!masked.empty()) {
    dmask.reset(new DBuf(masked.size() * 4, s));
    h2d(s, dmask->as<int32_t>(), masked);
  }
  switch (b) {
#define CASE(BV) case BV: \
    klaunch(s, false, gather_blocks_kernel<BV>, nblk(ne * bb, 256), 256, (int64_t)ne, (const int*)dsrc.p, \
            (const double*)dAnat.p, F->as<double>()); \
    if (dmask) klaunch(s, false, zero_blocks_kernel, nblk(masked.size() * bb, 256), 256, (int64_t)masked.size(), bb, \
                       (const int*)dmask->p, F->as<double>()); \
    for (int col = 0; col + 1 < (int)S.color_blk_ptr.size(); ++col) { \
      const int k0 = S.color_blk_ptr[col], k1 = S.color_blk_ptr[col + 1]; \
      if (k1 > k0) klaunch(s, false, bilu_factor_kernel<BV>, nblk(k1 - k0, 64), 64, k0, k1, (const int*)dbp.p, \
                           (const int*)drp.p, (const int*)dci.p, (const int*)ddg.p, F->as<double>(), dbad.as<int>()); \
    } \
    break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
  }
  int bad = -1;
  CK(cudaMemcpyAsync(&bad, dbad.p, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (bad >= 0) throw std::pair<int, std::string>(MSP_ESINGULAR, "BILU: singular pivot block at cell " + std::to_string(S.order[bad]));
  return F;
}

// a8, 4x4 blocks: ELL copy of the pressure columns (width = the longest row, <= kEllMax),
// refreshed with the values (setup, msp_update)
void fill_pell(msp_handle* h) {
  if (!h->pell_w) return;
  klaunch(h->s, false, pcol_ell_fill_kernel, nblk(h->n, 256), 256, (int)h->n, (int)h->pell_w, (const int*)h->rp,
          (const int*)h->ci, (const double*)h->Pcol, h->pell_c, h->pell_v);
}
void setup_pell(msp_handle* h, const std::vector<int32_t>& rp) {
  h->pell_w = 0;
  if (h->b != 4 || !h->a8_ell || h->n == 0) return;
  int w = 0;
  for (size_t i = 0; i + 1 < rp.size(); ++i) w = std::max(w, rp[i + 1] - rp[i]);
  if (w == 0 || w > kEllMax) return;
  h->pell_w = w;
  h->pell_c = h->dalloc<int32_t>((size_t)w * h->n);
  h->pell_v = h->dalloc<double>((size_t)w * h->n * 4);
  fill_pell(h);
}

void do_setup(msp_handle* h, const msp::BlockMat& A) {
  auto t0 = std::chrono::steady_clock::now();
  SetupTimer T;
  msp::HostSetup S;
  std::string err;
  Nvtx nv_setup("S1-S4 SETUP");
  int rc = 0;
  h->gpu_s1 = false;
  msp::Params prm = h->prm;
  std::unique_ptr<DBuf> dAvals;           // A's values on the device (S1 upload, reused for the stage)
  RapChain chain;
  chain.s = h->s;
  // distributed: only rank 0 runs S1-S4, the others receive the result (MSP_DIST_SETUP_ALL=1:
  // every rank runs it)
  const bool rank0_setup = h->comm && h->nranks > 1 && h->setup_rank0;
  const bool run_here = !rank0_setup || h->rank == 0;
  if (rank0_setup && h->rank != 0 && h->setup_on_gpu) {
    dAvals.reset(new DBuf(A.v.size() * sizeof(double), h->s));
    h2d_large(h->s, dAvals->p, A.v.data(), sizeof(double) * A.v.size());
  }
  if (h->setup_on_gpu && run_here) {     // NEXT-2: S1 and the Galerkin products on the GPU
    DBuf* dApp = nullptr;
    dAvals = gpu_setup_s1(h->s, h->prm.decoupling, A, S, &dApp);
    chain.keep.emplace_back(dApp);          // A_PP resident as the first fine operand
    chain.v = dApp->as<double>();
    chain.keep.emplace_back(new DBuf((size_t)(A.n + 1) * 4, h->s));
    chain.keep.emplace_back(new DBuf(A.ci.size() * 4, h->s));
    chain.rp = chain.keep[1]->as<int32_t>();
    chain.ci = chain.keep[2]->as<int32_t>();
    h2d(h->s, chain.rp, A.rp);
    h2d(h->s, chain.ci, A.ci);
    chain.n = A.n;
    chain.nnz = (int64_t)A.ci.size();
    chain.host_v = nullptr;                  // set below: the host copy the hierarchy starts from
    h->gpu_s1 = true;
    prm.s1_given = true;
    prm.rap = [&chain](const msp::SpMat& Af, const std::vector<int32_t>& agg, int32_t na, msp::SpMat& C) {
      if (chain.host_v == nullptr && Af.n == chain.n && (int64_t)Af.ci.size() == chain.nnz) chain.host_v = Af.v.data();
      return gpu_rap(chain, Af, agg, na, C);
    };
  }
  T.mark("S1 weights + A_PP (GPU)");
  if (run_here) {
    Nvtx nv("S2-S4 host: NPAIR, colorings, ABMC order (Galerkin on the GPU)");
    try {
      rc = msp::run_host_setup(A, prm, S, err);
    } catch (const std::pair<int, std::string>& e) {
      if (!rank0_setup) throw;
      rc = e.first;
      err = e.second;
    } catch (const CudaError& e) {        // rank 0 must still reach the broadcast
      if (!rank0_setup) throw;
      rc = MSP_ECUDA;
      err = std::string("CUDA: ") + cudaGetErrorString(e.e) + " in " + e.where;
    }
  }
  if (rank0_setup) {
    Nvtx nv("S1-S4 result broadcast from rank 0");
    SetupBlob blob;
    if (h->rank == 0 && rc == 0) pack_setup(S, blob);
    bcast_setup(h, rc, err, blob);
    if (rc == 0 && h->rank != 0) {
      unpack_setup(blob, S);
      S.prm = prm;
      S.A = &A;
    }
    T.mark("setup broadcast");
  }
  if (rc) throw std::pair<int, std::string>(rc, err);
  std::vector<int32_t> rp, ci, dg, src;
  std::vector<double> F;
  T.mark("host setup S2-S4");
  h->W_nat = S.W;
  h->App_nat = S.App.v;
  // BILU(0): on the GPU after the upload (single GPU), on the host for the distributed
  // setup (every rank factorizes the global matrix) or when MSP_HOST_BILU=1
  const bool host_bilu_env = std::getenv("MSP_HOST_BILU") && std::atoi(std::getenv("MSP_HOST_BILU"));
  // distributed handles factorize the GLOBAL matrix on the GPU too (every rank holds A's
  // values on its device after S1) and keep their rows; host factorization only without
  // the GPU setup steps
  const bool gpu_bilu = !host_bilu_env && (!h->comm || dAvals);
  rc = gpu_bilu ? msp::permuted_pattern(S, A, rp, ci, dg, src, err)
                : msp::bilu_factor_permuted(S, A, rp, ci, dg, src, F, err);
  if (rc) throw std::pair<int, std::string>(rc == 1 ? MSP_EINVAL : MSP_ESINGULAR, err);
  T.mark(gpu_bilu ? "BILU pattern (host)" : "BILU factorization (host)");

  h->free_all();
  h->valid = false;                  // until this SETUP completes (see msp_status docs)
  const int32_t n = A.n;
  const int b = A.b, bb = b * b;
  h->n = n;
  h->b = b;
  h->nc = b - 1;
  h->N = (size_t)n * b;
  h->nnzb = (int64_t)A.ci.size();
  h->order = S.order;
  h->src_entry = src;
  h->nat_rp = A.rp;
  h->nat_ci = A.ci;
  h->bilu_ncolor = S.bilu_ncolor;
  h->max_blk = 1;
  for (size_t k = 0; k + 1 < S.blk_ptr.size(); ++k) h->max_blk = std::max(h->max_blk, S.blk_ptr[k + 1] - S.blk_ptr[k]);
  h->n_ghost = 0;
  h->n0_ghost = 0;
  const int L = (int)S.lv.size();
  // AMG levels: natural-order permutations of every level (the upload of level 0 is
  // rank-local in distributed mode, levels >= 1 are replicated)
  h->level_n.clear();
  h->level_nnz.clear();
  h->level_colors.clear();
  h->lv.resize(L);
  std::vector<std::vector<int32_t>> perms(L);
  h->dist_D = h->comm ? std::max(0, std::min(h->prm.dist_levels, L - 1)) : 0;
  for (int l = 0; l < L; ++l) {
    h->lv[l].idx = l;
    if (!h->comm || l > h->dist_D) upload_level(h, h->lv[l], S.lv[l].A, S.lv[l].ncolor, S.lv[l].color, perms[l]);
    else {
      // permutation only (the partitioned levels are uploaded by dist_localize)
      const auto& col = S.lv[l].color;
      const int32_t nl = S.lv[l].A.n;
      std::vector<int32_t> cnt(S.lv[l].ncolor + 1, 0);
      for (int32_t c : col) cnt[c + 1]++;
      for (int c = 0; c < S.lv[l].ncolor; ++c) cnt[c + 1] += cnt[c];
      perms[l].resize(nl);
      for (int32_t i = 0; i < nl; ++i) perms[l][i] = cnt[col[i]]++;
    }
    h->level_n.push_back(S.lv[l].A.n);
    h->level_nnz.push_back(S.lv[l].A.nnz());
    h->level_colors.push_back(S.lv[l].ncolor);
  }
  h->nL = S.Ac.n;
  h->coarse_diag = S.coarse_diag;
  h->level_n.push_back(S.Ac.n);
  h->level_nnz.push_back(S.Ac.nnz());
  h->level_colors.push_back(0);
  for (int l = (h->comm ? h->dist_D + 1 : 0); l < L; ++l) {   // replicated levels
    DevLevel& D = h->lv[l];
    const auto& agg = S.lv[l].agg;
    const int32_t nn = S.lv[l].n_next;
    std::vector<int32_t> ap(D.n), inv(D.n);
    for (int32_t i = 0; i < D.n; ++i) inv[perms[l][i]] = i;
    for (int32_t p = 0; p < D.n; ++p) {
      const int32_t I = agg[inv[p]];
      ap[p] = (l + 1 < L) ? perms[l + 1][I] : I;
    }
    std::vector<int32_t> pp(nn + 1, 0), pi(D.n);
    for (int32_t p = 0; p < D.n; ++p) pp[ap[p] + 1]++;
    for (int32_t I = 0; I < nn; ++I) pp[I + 1] += pp[I];
    {
      std::vector<int32_t> f(pp.begin(), pp.end() - 1);
      for (int32_t p = 0; p < D.n; ++p) pi[f[ap[p]]++] = p;
    }
    check_range(ap, 0, nn, "aggregate map");
    check_ptr(pp, nn, D.n, "restriction pointers");
    check_perm(pi, "restriction members");
    D.agg = h->upload(ap);
    D.pt_ptr = h->upload(pp);
    D.pt_idx = h->upload(pi);
  }
  if (h->comm) {
    std::unique_ptr<DBuf> Fglob;
    std::vector<int32_t> masked;
    if (h->prm.bilu_local) {
      // rank-local BILU (NEXT-3 option): ILU(0) of the matrix with every coupling between
      // cells of different owners removed (block Jacobi across slabs) -- no halo exchange
      // in the substitutions, a preconditioner that depends on the partition
      const int nb = (int)S.blk_ptr.size() - 1;
      std::vector<int32_t> opos(A.n);
      for (int k = 0; k < nb; ++k) {
        int32_t lowest = INT32_MAX;
        for (int32_t p = S.blk_ptr[k]; p < S.blk_ptr[k + 1]; ++p) lowest = std::min(lowest, S.order[p]);
        for (int32_t p = S.blk_ptr[k]; p < S.blk_ptr[k + 1]; ++p) opos[p] = h->owner_in[lowest];
      }
      for (int32_t p = 0; p < A.n; ++p)
        for (int32_t e = rp[p]; e < rp[p + 1]; ++e)
          if (opos[p] != opos[ci[e]]) masked.push_back(e);
    }
    if (gpu_bilu) Fglob = gpu_bilu_global(h, A, S, rp, ci, dg, src, *dAvals, masked);
    else if (!masked.empty()) throw std::pair<int, std::string>(MSP_EINVAL, "bilu_local needs the GPU setup path");
    dist_localize(h, A, S, rp, ci, dg, src, F, perms, Fglob ? Fglob->as<double>() : nullptr,
                  dAvals ? dAvals->as<double>() : nullptr);
  } else {
  // BSR pattern + values (column-major blocks)
  check_ptr(rp, n, (int64_t)ci.size(), "BSR row pointers");
  check_range(ci, 0, n, "BSR columns");
  check_perm(src, "BSR entry permutation");
  for (int32_t i = 0; i < n; ++i) check_index(dg[i] >= rp[i] && dg[i] < rp[i + 1] && ci[dg[i]] == i, "BSR diagonal");
  check_perm(S.order, "ABMC cell order");
  check_ptr(S.blk_ptr, (int64_t)S.blk_ptr.size() - 1, n, "ABMC block pointers");
  h->rp = h->upload(rp);
  h->ci = h->upload(ci);
  h->d_src = h->upload(src);
  h->stage = nullptr;
  h->dg = h->upload(dg);
  h->d_order = h->upload(S.order);
  {
    // raw row-major values through the ASMSP staging buffer, laid out on the device:
    // A (caller's natural order) -> permuted column-major blocks + pressure columns (the
    // msp_update refresh kernel); F = BILU factors, computed on the GPU per block color
    // from the permuted row-major A (or uploaded from the host factorization), then
    // transposed to column-major
    const size_t nv = ci.size() * (size_t)bb;
    h->stage = h->dalloc<double>(std::max(nv, A.v.size()));
    h->Fval = h->dalloc<double>(nv);
    h->Aval = h->dalloc<double>(nv);
    h->Pcol = h->dalloc<double>(ci.size() * (size_t)b);
    if (T.on) {
      CK(cudaStreamSynchronize(h->s));
      T.mark("  A/F buffers allocated");
    }
    if (dAvals) CK(cudaMemcpyAsync(h->stage, dAvals->p, sizeof(double) * A.v.size(), cudaMemcpyDeviceToDevice, h->s));
    else h2d_large(h->s, h->stage, A.v.data(), sizeof(double) * A.v.size());
    int* dbad = nullptr;
    if (gpu_bilu) {
      dbad = h->dalloc<int>(1);
      CK(cudaMemsetAsync(dbad, 0xff, sizeof(int), h->s));               // -1
    }
    switch (b) {
#define CASE(BV) case BV: \
      klaunch(h->s, false, refresh_values_kernel<BV>, nblk(nv, 256), 256, (int64_t)ci.size(), (const int*)h->d_src, \
              (const double*)h->stage, h->Aval, h->Pcol); \
      if (gpu_bilu) { \
        klaunch(h->s, false, gather_blocks_kernel<BV>, nblk(nv, 256), 256, (int64_t)ci.size(), (const int*)h->d_src, \
                (const double*)h->stage, h->Fval); \
        const int32_t* bp = h->upload(S.blk_ptr); \
        for (int col = 0; col + 1 < (int)S.color_blk_ptr.size(); ++col) { \
          const int k0 = S.color_blk_ptr[col], k1 = S.color_blk_ptr[col + 1]; \
          if (k1 > k0) klaunch(h->s, false, bilu_factor_kernel<BV>, nblk(k1 - k0, 64), 64, k0, k1, bp, \
                               (const int*)h->rp, (const int*)h->ci, (const int*)h->dg, h->Fval, dbad); \
        } \
      } else { \
        CK(cudaMemcpyAsync(h->Fval, F.data(), sizeof(double) * nv, cudaMemcpyHostToDevice, h->s)); \
      } \
      klaunch(h->s, false, transpose_blocks_kernel<BV>, nblk(nv, 256), 256, (int64_t)ci.size(), \
              (const double*)h->Fval, h->stage); \
      std::swap(h->Fval, h->stage); \
      break;
      CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
    }
    CK(cudaStreamSynchronize(h->s));
    T.mark("  values + BILU factors (GPU)");
    if (gpu_bilu) {
      int bad = -1;
      CK(cudaMemcpy(&bad, dbad, sizeof(int), cudaMemcpyDeviceToHost));
      if (bad >= 0)
        throw std::pair<int, std::string>(MSP_ESINGULAR, "BILU: singular pivot block at cell " + std::to_string(S.order[bad]));
    }
  }
  setup_pell(h, rp);
  T.mark("A/F/Pcol transpose+upload");
  if (h->prm.stages == 3) {
    const int nc = b - 1;
    std::vector<double> Dn((size_t)n * nc * nc), D(nc * nc), Di(nc * nc);
    for (int32_t p = 0; p < n; ++p) {
      const int32_t c = S.order[p];
      int32_t ed = -1;
      for (int32_t e = A.rp[c]; e < A.rp[c + 1]; ++e) if (A.ci[e] == c) ed = e;
      for (int i = 0; i < nc; ++i)
        for (int k = 0; k < nc; ++k) D[i * nc + k] = A.v[(size_t)ed * bb + (1 + i) * b + 1 + k];
      if (!msp::invert_block(nc, D.data(), Di.data()))
        throw std::pair<int, std::string>(MSP_ESINGULAR, "BGS: singular N-N block at cell " + std::to_string(c));
      for (int i = 0; i < nc; ++i)
        for (int k = 0; k < nc; ++k) Dn[(size_t)p * nc * nc + k * nc + i] = Di[i * nc + k];   // column-major
    }
    h->Dn = h->upload(Dn);
    h->wfull = h->dalloc<double>((size_t)n * b);
    h->r1 = h->dalloc<double>((size_t)n * b);
    if (h->max_blk > 4) throw std::pair<int, std::string>(MSP_EINVAL, "stages=3 needs aggregate blocks of <= 4 cells");
  }
  {
    std::vector<double> Wi((size_t)n * b);
    for (int32_t p = 0; p < n; ++p)
      std::memcpy(&Wi[(size_t)p * b], &S.W[(size_t)S.order[p] * b], sizeof(double) * b);
    h->W = h->upload(Wi);
  }
  // ABMC blocks
  h->bilu_ncolor = S.bilu_ncolor;
  h->color_blk = S.color_blk_ptr;
  h->blk_ptr = h->upload(S.blk_ptr);
  h->max_blk = 1;
  for (size_t k = 0; k + 1 < S.blk_ptr.size(); ++k) h->max_blk = std::max(h->max_blk, S.blk_ptr[k + 1] - S.blk_ptr[k]);
  {
    std::vector<int32_t> cnt(n, 0);
    for (size_t k = 0; k + 1 < S.blk_ptr.size(); ++k) {
      const int32_t c0 = S.blk_ptr[k], c1 = S.blk_ptr[k + 1];
      for (int32_t i = c0; i < c1; ++i) {
        int32_t next = 0, nint = 0;
        for (int32_t e = rp[i]; e < dg[i]; ++e) if (ci[e] < c0) ++next;
        for (int32_t e = dg[i] + 1; e < rp[i + 1]; ++e) if (ci[e] < c1) ++nint;
        if (next > 255 || nint > 255) throw std::pair<int, std::string>(MSP_EINVAL, "BILU: row too long for the block kernel");
        cnt[i] = next | (nint << 8);
      }
    }
    h->bcnt = h->upload(cnt);
    h->islot = h->upload(make_islot(n, rp, ci, dg, S.blk_ptr));
    h->bm_f = nullptr;
    if (h->bilu_meta && b >= 4 && h->max_blk <= 4) {
      // per (block, cell slot) metadata of bilu_meta4_kernel
      const int mx = h->max_blk <= 1 ? 1 : (h->max_blk <= 2 ? 2 : 4);
      const size_t nbk = S.blk_ptr.size() - 1;
      std::vector<int4> mf(nbk * mx, make_int4(-1, 0, 0, 0)), mb(nbk * mx, make_int4(-1, 0, 0, 0)),
          cf(nbk * mx, make_int4(0, 0, 0, 0)), cb(nbk * mx, make_int4(0, 0, 0, 0)),
          sl(nbk * mx, make_int4(-1, -1, -1, -1));
      const std::vector<int4> isl = make_islot(n, rp, ci, dg, S.blk_ptr);
      for (size_t k = 0; k < nbk; ++k) {
        const int32_t c0 = S.blk_ptr[k], c1 = S.blk_ptr[k + 1];
        for (int32_t i = c0; i < c1; ++i) {
          const size_t sidx = k * mx + (i - c0);
          int32_t next = 0, nint = 0;
          for (int32_t e = rp[i]; e < dg[i]; ++e) if (ci[e] < c0) ++next;
          for (int32_t e = dg[i] + 1; e < rp[i + 1]; ++e) if (ci[e] < c1) ++nint;
          const int32_t ei = dg[i] + 1 + nint;
          mf[sidx] = make_int4(i, rp[i], rp[i] + next, 0);
          mb[sidx] = make_int4(i, dg[i], ei, rp[i + 1]);
          int a[4] = {0, 0, 0, 0}, bq[4] = {0, 0, 0, 0};
          for (int u = 0; u < 4 && u < next; ++u) a[u] = ci[rp[i] + u];
          for (int u = 0; u < 4 && ei + u < rp[i + 1]; ++u) bq[u] = ci[ei + u];
          cf[sidx] = make_int4(a[0], a[1], a[2], a[3]);
          cb[sidx] = make_int4(bq[0], bq[1], bq[2], bq[3]);
          sl[sidx] = isl[i];
        }
      }
      h->bm_f = h->upload(mf);
      h->bm_b = h->upload(mb);
      h->bm_cf = h->upload(cf);
      h->bm_cb = h->upload(cb);
      h->bm_sl = h->upload(sl);
    }
  }
    {
      std::vector<int32_t> l0(n);
      for (int32_t p = 0; p < n; ++p) l0[p] = (L > 0) ? perms[0][S.order[p]] : S.order[p];
      h->l0_of_cell = h->upload(l0);
      std::vector<int32_t> inv(n);
      for (int32_t p = 0; p < n; ++p) inv[l0[p]] = p;
      h->cell_of_l0 = h->upload(inv);
    }
  }
  T.mark("levels upload");
  // coarsest
  h->bL = h->dalloc<double>(h->nL);
  h->xL = h->dalloc<double>(h->nL);
  if (h->coarse_diag) {
    std::vector<double> d(h->nL, 0.0);
    for (int32_t i = 0; i < h->nL; ++i)
      for (int32_t e = S.Ac.rp[i]; e < S.Ac.rp[i + 1]; ++e)
        if (S.Ac.ci[e] == i) d[i] = S.Ac.v[e];
    h->cdiag = h->upload(d);
  } else {
    const int32_t m = h->nL;
    // dense A_L and the identity right-hand side assembled on the device (no 2 x m^2 host
    // uploads); inverse by LU (getrf) + m solves (getrs); the cuSOLVER handle is created
    // once per msp_handle and reused by every rebuild
    double* dA = h->dalloc<double>((size_t)m * m);           // row-major A == column-major A^T
    h->ldA = (m + 31) / 32 * 32;             // 256-byte aligned rows for the vector loads
    h->Ainv = h->dalloc<double>((size_t)m * h->ldA);
    {
      const int32_t* crp = h->upload(S.Ac.rp);
      const int32_t* cci = h->upload(S.Ac.ci);
      const double* cv = h->upload(S.Ac.v);
      CK(cudaMemsetAsync(dA, 0, sizeof(double) * (size_t)m * m, h->s));
      CK(cudaMemsetAsync(h->Ainv, 0, sizeof(double) * (size_t)m * h->ldA, h->s));
      klaunch(h->s, false, dense_identity_kernel, nblk(m, 128), 128, m, h->ldA, crp, cci, cv, dA, h->Ainv);
    }
    if (!h->cs) {
      if (cusolverDnCreate(&h->cs) != CUSOLVER_STATUS_SUCCESS) { h->cs = nullptr; throw CudaError{cudaErrorUnknown, "cusolverDnCreate"}; }
    }
    cusolverDnHandle_t cs = h->cs;
    cusolverDnSetStream(cs, h->s);
    int lwork = 0;
    cusolverDnDgetrf_bufferSize(cs, m, m, dA, m, &lwork);
    double* work = h->dalloc<double>(lwork);
    int* ipiv = h->dalloc<int>(m);
    int* info = h->dalloc<int>(1);
    cusolverStatus_t s1 = cusolverDnDgetrf(cs, m, m, dA, m, work, ipiv, info);
    int hinfo = 0;
    CK(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, h->s));
    CK(cudaStreamSynchronize(h->s));
    if (s1 != CUSOLVER_STATUS_SUCCESS || hinfo != 0)
      throw std::pair<int, std::string>(MSP_ESINGULAR, "coarsest: singular dense matrix (getrf info " + std::to_string(hinfo) + ")");
    // (A^T) X = I  =>  X = A^-T column-major  ==  A^-1 row-major
    cusolverStatus_t s2 = cusolverDnDgetrs(cs, CUBLAS_OP_N, m, m, dA, m, ipiv, h->Ainv, h->ldA, info);
    CK(cudaStreamSynchronize(h->s));
    if (s2 != CUSOLVER_STATUS_SUCCESS) throw CudaError{cudaErrorUnknown, "cusolverDnDgetrs"};
  }
  T.mark("coarsest inverse");
  setup_pool_trim(h->s);
  T.mark("setup pool trim");
  // work vectors (cell-space vectors read through ghost columns carry ghost slots)
  const size_t Ng = (size_t)(h->n + h->n_ghost) * h->b;
  h->z = h->dalloc<double>(Ng);
  h->r = h->dalloc<double>(Ng);
  CK(cudaMemsetAsync(h->r, 0, sizeof(double) * Ng, h->s));   // ghost slots finite (rank-local BILU reads 0 x them)
  h->u = h->dalloc<double>(h->N);
  h->xin = h->dalloc<double>(Ng);
  h->bin = h->dalloc<double>(h->N);
  h->io = h->dalloc<double>(h->N);
  h->wp = h->dalloc<double>(h->n + h->n_ghost);
  h->lred = h->dalloc<double>(kMaxV);
  h->part = h->dalloc<double>((size_t)kRedBlocks * kMaxV);
  h->dh1 = h->dalloc<double>(kMaxV);
  h->dh2 = h->dalloc<double>(kMaxV);
  h->hcol = h->dalloc<double>(4 * kMaxV);
  h->dst = h->dalloc<double>(2 * (kMaxV + 2));
  h->dsum = h->dalloc<double>(kMaxV + 2);
  h->ticket = h->dalloc<unsigned>(4);
  CK(cudaMemsetAsync(h->ticket, 0, 4 * sizeof(unsigned), h->s));
  CK(cudaMallocHost(&h->hpin, sizeof(double) * kMaxV * 4));
  CK(cudaMallocHost(&h->hrec, sizeof(double) * kMaxV * kRecStride));
  for (auto& e : h->ev_step)
    if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CK(cudaMallocHost(&h->hgv, sizeof(double) * kGvSize));
  h->gv = h->dalloc<double>(kGvSize);
  CK(cudaStreamSynchronize(h->s));
  auto t1 = std::chrono::steady_clock::now();
  const double secs = std::chrono::duration<double>(t1 - t0).count();
  h->st.setup_calls++;
  h->st.setup_seconds += secs;
  h->st.last_setup_seconds = secs;
  h->st.levels = L;
  h->st.n_coarsest = h->nL;
  h->st.bilu_colors = h->bilu_ncolor;
  h->valid = true;
}

// ---------------------------------------------------------------------------
// Distributed setup.  Every rank runs the same (deterministic) global
// host setup, so colorings, aggregates, orderings and factors are those of 1 GPU; it
// then keeps its owned rows.  Cell ownership follows the caller's partition (z-slabs),
// with every ABMC block (= level-1 aggregate) assigned whole to the owner of its
// lowest-index cell, so BILU blocks and level-1 aggregates are never split.
//  cell space : owned cells in global ABMC position order, then ghosts grouped by
//               (owner, block color, position) -> one contiguous receive per color;
//  level 0    : owned rows in global level-0 order (color-major), then ghosts grouped
//               by (owner, level-0 color, global row);
//  levels >= 1 and the coarsest are replicated; the level-1 right-hand side is
//  assembled by an allgather of every rank's owned aggregates.
// ---------------------------------------------------------------------------
static void build_halo(msp_handle* h, msp::HaloPlan& P, int nseg, int nranks, int me,
                       const std::vector<std::vector<std::vector<int32_t>>>& sendl,   // [peer][seg] owned local idx
                       const std::vector<std::vector<int32_t>>& recv_cnt,            // [peer][seg]
                       int n_own = -1) {
  P = msp::HaloPlan();
  P.nseg = nseg;
  std::vector<int32_t> idx;
  int ghost = 0;
  for (int q = 0; q < nranks; ++q) {
    if (q == me) continue;
    int ns = 0, nr = 0;
    for (int sg = 0; sg < nseg; ++sg) { ns += (int)sendl[q][sg].size(); nr += recv_cnt[q][sg]; }
    if (ns == 0 && nr == 0) continue;
    P.peers.push_back(q);
    P.send_base.push_back((int)idx.size());
    P.recv_base.push_back(ghost);
    std::vector<int> so(nseg + 1, 0), ro(nseg + 1, 0);
    for (int sg = 0; sg < nseg; ++sg) {
      so[sg + 1] = so[sg] + (int)sendl[q][sg].size();
      ro[sg + 1] = ro[sg] + recv_cnt[q][sg];
      idx.insert(idx.end(), sendl[q][sg].begin(), sendl[q][sg].end());
    }
    ghost += nr;
    P.send_off.push_back(so);
    P.recv_off.push_back(ro);
  }
  P.nsend = (int)idx.size();
  P.nghost = ghost;
  P.d_send_idx = h->upload(idx);
  P.d_sendbuf = h->dalloc<double>((size_t)std::max(P.nsend, 1) * 8);
  if (n_own >= 0) {                               // send positions per owned entry (<= 2)
    std::vector<int2> sl(std::max(n_own, 1), make_int2(-1, -1));
    bool ok = true;
    for (int k = 0; k < (int)idx.size() && ok; ++k) {
      int2& e = sl[idx[k]];
      if (e.x < 0) e.x = k;
      else if (e.y < 0) e.y = k;
      else ok = false;
    }
    P.d_slots = ok ? h->upload(sl) : nullptr;
  }
}

// Host-side plan of the cell space for rank `me` (pure integer work, no GPU).
struct CellPlan {
  std::vector<int32_t> own_pos, color_pos;   // effective owner / block color of every position
  std::vector<int32_t> posown, loc;          // owned positions (local order), position -> local
  std::vector<int32_t> ghosts, lcol;         // ghost positions (receive order), position -> local col
  std::vector<std::vector<std::vector<int32_t>>> sendl;   // [peer][color] owned local indices
  std::vector<std::vector<int32_t>> rcnt;                 // [peer][color] ghost counts
};

CellPlan compute_cell_plan(const msp::HostSetup& S, const std::vector<int32_t>& rp, const std::vector<int32_t>& ci,
                           const std::vector<int32_t>& owner_in, int P, int me) {
  const int32_t n = S.n;
  CellPlan C;
  C.own_pos.assign(n, 0);
  C.color_pos.assign(n, 0);
  const int nb = (int)S.blk_ptr.size() - 1;
  std::vector<int32_t> bcolor(nb);
  for (int c = 0; c < S.bilu_ncolor; ++c)
    for (int k = S.color_blk_ptr[c]; k < S.color_blk_ptr[c + 1]; ++k) bcolor[k] = c;
  for (int k = 0; k < nb; ++k) {
    int32_t lowest = INT32_MAX;
    for (int32_t p = S.blk_ptr[k]; p < S.blk_ptr[k + 1]; ++p) lowest = std::min(lowest, S.order[p]);
    const int32_t o = owner_in[lowest];
    for (int32_t p = S.blk_ptr[k]; p < S.blk_ptr[k + 1]; ++p) { C.own_pos[p] = o; C.color_pos[p] = bcolor[k]; }
  }
  C.loc.assign(n, -1);
  for (int32_t p = 0; p < n; ++p)
    if (C.own_pos[p] == me) { C.loc[p] = (int32_t)C.posown.size(); C.posown.push_back(p); }
  std::vector<std::vector<int32_t>> need(P);
  {
    std::vector<int32_t> mark(n, -1);
    for (int32_t p = 0; p < n; ++p) {
      const int t = C.own_pos[p];
      for (int32_t e = rp[p]; e < rp[p + 1]; ++e) {
        const int32_t qpos = ci[e];
        const int o = C.own_pos[qpos];
        if (o == t) continue;
        if (o == me) need[t].push_back(qpos);
        if (t == me && mark[qpos] < 0) { mark[qpos] = 1; C.ghosts.push_back(qpos); }
      }
    }
    for (int q = 0; q < P; ++q) {
      auto& v = need[q];
      std::sort(v.begin(), v.end());
      v.erase(std::unique(v.begin(), v.end()), v.end());
      std::sort(v.begin(), v.end(), [&](int32_t x, int32_t y) {
        return C.color_pos[x] != C.color_pos[y] ? C.color_pos[x] < C.color_pos[y] : x < y;
      });
    }
    std::sort(C.ghosts.begin(), C.ghosts.end(), [&](int32_t x, int32_t y) {
      if (C.own_pos[x] != C.own_pos[y]) return C.own_pos[x] < C.own_pos[y];
      if (C.color_pos[x] != C.color_pos[y]) return C.color_pos[x] < C.color_pos[y];
      return x < y;
    });
  }
  const int32_t no = (int32_t)C.posown.size(), ng = (int32_t)C.ghosts.size();
  C.lcol.assign(n, -1);
  for (int32_t l = 0; l < no; ++l) C.lcol[C.posown[l]] = l;
  for (int32_t k = 0; k < ng; ++k) C.lcol[C.ghosts[k]] = no + k;
  C.sendl.assign(P, std::vector<std::vector<int32_t>>(S.bilu_ncolor));
  C.rcnt.assign(P, std::vector<int32_t>(S.bilu_ncolor, 0));
  for (int q = 0; q < P; ++q)
    for (int32_t pos : need[q]) C.sendl[q][C.color_pos[pos]].push_back(C.loc[pos]);
  for (int32_t g : C.ghosts) C.rcnt[C.own_pos[g]][C.color_pos[g]]++;
  return C;
}

void dist_localize(msp_handle* h, const msp::BlockMat& A, const msp::HostSetup& S, const std::vector<int32_t>& rp,
                   const std::vector<int32_t>& ci, const std::vector<int32_t>& dg, const std::vector<int32_t>& src,
                   const std::vector<double>& F, const std::vector<std::vector<int32_t>>& perms,
                   const double* dF, const double* dAnat) {
  const int32_t n = A.n;
  const int b = A.b, bb = b * b;
  const int P = h->nranks, me = h->rank;
  const int L = (int)S.lv.size();
  if (L < 1) throw std::pair<int, std::string>(MSP_EINVAL, "distributed mode needs >= 1 AMG smoothing level (n > coarsest_max_dof)");
  // ---------------- cell space
  CellPlan C = compute_cell_plan(S, rp, ci, h->owner_in, P, me);
  const std::vector<int32_t>& own_pos = C.own_pos;
  const std::vector<int32_t>& posown = C.posown;
  const std::vector<int32_t>& lcol = C.lcol;
  std::vector<int32_t> own_cell(n);
  for (int32_t p = 0; p < n; ++p) own_cell[S.order[p]] = own_pos[p];
  const int32_t no = (int32_t)posown.size();
  const int32_t ng = (int32_t)C.ghosts.size();
  build_halo(h, h->cell_halo, S.bilu_ncolor, P, me, C.sendl, C.rcnt, (int)C.posown.size());
  // local BSR rows (entries keep the global position order: L | diag | U)
  std::vector<int32_t> lrp(no + 1, 0), lci, ldg(no), lsrc;
  std::vector<double> lF, lA, lPc, lW((size_t)no * b);
  const std::vector<int32_t> gcnt = block_counts(S, rp, ci, dg);
  std::vector<int32_t> lcnt(no);
  for (int32_t l = 0; l < no; ++l) {
    const int32_t p = posown[l];
    for (int32_t e = rp[p]; e < rp[p + 1]; ++e) {
      if (e == dg[p]) ldg[l] = (int32_t)lci.size();
      lci.push_back(lcol[ci[e]]);
      lsrc.push_back(src[e]);
    }
    lrp[l + 1] = (int32_t)lci.size();
    lcnt[l] = gcnt[p];
    std::memcpy(&lW[(size_t)l * b], &S.W[(size_t)S.order[p] * b], sizeof(double) * b);
  }
  const size_t ne = lci.size();
  std::vector<int32_t> lent;                      // global (permuted) entry of every local entry
  if (dF) {
    lent.reserve(ne);
    for (int32_t l = 0; l < no; ++l)
      for (int32_t e = rp[posown[l]]; e < rp[posown[l] + 1]; ++e) lent.push_back(e);
  } else {
  lF.resize(ne * bb);
  lA.resize(ne * bb);
  lPc.resize(ne * b);
  }
  if (!dF) {
    size_t q = 0;
    for (int32_t l = 0; l < no; ++l) {
      const int32_t p = posown[l];
      for (int32_t e = rp[p]; e < rp[p + 1]; ++e, ++q) {
        for (int r = 0; r < b; ++r)
          for (int c = 0; c < b; ++c) {
            lF[q * bb + c * b + r] = F[(size_t)e * bb + r * b + c];                  // column-major
            lA[q * bb + c * b + r] = A.v[(size_t)src[e] * bb + r * b + c];
          }
        for (int r = 0; r < b; ++r) lPc[q * b + r] = A.v[(size_t)src[e] * bb + r * b];
      }
    }
  }
  // owned blocks
  std::vector<int32_t> lblk(1, 0), lcolor_blk(S.bilu_ncolor + 1, 0);
  for (int c = 0; c < S.bilu_ncolor; ++c) {
    for (int k = S.color_blk_ptr[c]; k < S.color_blk_ptr[c + 1]; ++k) {
      if (own_pos[S.blk_ptr[k]] != me) continue;
      lblk.push_back(lblk.back() + (S.blk_ptr[k + 1] - S.blk_ptr[k]));
    }
    lcolor_blk[c + 1] = (int32_t)lblk.size() - 1;
  }
  // natural order of the owned cells (the caller's b/x layout on this rank)
  h->owned_cells.clear();
  for (int32_t c = 0; c < n; ++c) if (own_cell[c] == me) h->owned_cells.push_back(c);
  std::vector<int32_t> natloc(n, -1), lorder(no);
  for (size_t k = 0; k < h->owned_cells.size(); ++k) natloc[h->owned_cells[k]] = (int32_t)k;
  for (int32_t l = 0; l < no; ++l) lorder[l] = natloc[S.order[posown[l]]];
  // upload cell space
  h->n = no;
  h->N = (size_t)no * b;
  h->n_ghost = ng;
  h->rp = h->upload(lrp);
  h->ci = h->upload(lci);
  h->dg = h->upload(ldg);
  h->d_src = h->upload(lsrc);
  h->src_entry = lsrc;
  h->stage = nullptr;
  h->d_order = h->upload(lorder);
  h->order = lorder;
  if (dF) {
    // factors and values laid out on the device from the global GPU factorization and A's
    // natural values (no host copies of the local blocks)
    h->Fval = h->dalloc<double>(ne * bb);
    h->Aval = h->dalloc<double>(ne * bb);
    h->Pcol = h->dalloc<double>(ne * b);
    double* tmp = h->dalloc<double>(ne * bb);
    const int32_t* d_lent = h->upload(lent);
    switch (b) {
#define CASE(BV) case BV: \
      klaunch(h->s, false, gather_blocks_kernel<BV>, nblk(ne * bb, 256), 256, (int64_t)ne, d_lent, dF, tmp); \
      klaunch(h->s, false, transpose_blocks_kernel<BV>, nblk(ne * bb, 256), 256, (int64_t)ne, (const double*)tmp, h->Fval); \
      klaunch(h->s, false, refresh_values_kernel<BV>, nblk(ne * bb, 256), 256, (int64_t)ne, (const int*)h->d_src, dAnat, \
              h->Aval, h->Pcol); \
      break;
      CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
    }
    CK(cudaStreamSynchronize(h->s));
  } else {
    h->Fval = h->upload(lF);
    h->Aval = h->upload(lA);
    h->Pcol = h->upload(lPc);
  }
  setup_pell(h, lrp);
  h->W = h->upload(lW);
  h->color_blk = lcolor_blk;
  h->blk_ptr = h->upload(lblk);
  h->bcnt = h->upload(lcnt);
  h->islot = h->upload(make_islot(no, lrp, lci, ldg, lblk));
  h->nnzb = (int64_t)ne;
  {
    std::vector<int32_t> rin, rbd;                // rows without / with a ghost column
    for (int32_t l = 0; l < no; ++l) {
      bool gh = false;
      for (int32_t e = lrp[l]; e < lrp[l + 1]; ++e) gh = gh || lci[e] >= no;
      (gh ? rbd : rin).push_back(l);
    }
    h->n_rows_in = (int)rin.size();
    h->n_rows_bd = (int)rbd.size();
    h->rows_in = h->upload(rin);
    h->rows_bd = h->upload(rbd);
  }
  // ---------------- level 0
  const msp::SpMat& A0 = S.lv[0].A;               // natural level-0 numbering = cells
  const auto& col0 = S.lv[0].color;
  const int g0 = S.lv[0].ncolor;
  std::vector<int32_t> rows0;                     // owned natural cells by global level-0 row
  for (int32_t c = 0; c < n; ++c) if (own_cell[c] == me) rows0.push_back(c);
  std::sort(rows0.begin(), rows0.end(), [&](int32_t x, int32_t y) { return perms[0][x] < perms[0][y]; });
  std::vector<int32_t> l0loc(n, -1), gh0;
  for (size_t k = 0; k < rows0.size(); ++k) l0loc[rows0[k]] = (int32_t)k;
  std::vector<std::vector<int32_t>> need0(P);
  {
    std::vector<int32_t> mark(n, -1);
    for (int32_t c = 0; c < n; ++c) {
      const int t = own_cell[c];
      for (int32_t e = A0.rp[c]; e < A0.rp[c + 1]; ++e) {
        const int32_t d = A0.ci[e];
        const int o = own_cell[d];
        if (o == t) continue;
        if (o == me) need0[t].push_back(d);
        if (t == me && mark[d] < 0) { mark[d] = 1; gh0.push_back(d); }
      }
    }
    for (int q = 0; q < P; ++q) {
      auto& v = need0[q];
      std::sort(v.begin(), v.end(), [&](int32_t x, int32_t y) { return perms[0][x] < perms[0][y]; });
      v.erase(std::unique(v.begin(), v.end()), v.end());
    }
    std::sort(gh0.begin(), gh0.end(), [&](int32_t x, int32_t y) {
      if (own_cell[x] != own_cell[y]) return own_cell[x] < own_cell[y];
      return perms[0][x] < perms[0][y];                // color-major inside a peer
    });
  }
  const int32_t no0 = (int32_t)rows0.size(), ng0 = (int32_t)gh0.size();
  std::vector<int32_t> l0col(n, -1);
  for (int32_t k = 0; k < no0; ++k) l0col[rows0[k]] = k;
  for (int32_t k = 0; k < ng0; ++k) l0col[gh0[k]] = no0 + k;
  {
    std::vector<std::vector<std::vector<int32_t>>> sendl(P, std::vector<std::vector<int32_t>>(g0));
    std::vector<std::vector<int32_t>> rcnt(P, std::vector<int32_t>(g0, 0));
    for (int q = 0; q < P; ++q)
      for (int32_t d : need0[q]) sendl[q][col0[d]].push_back(l0loc[d]);
    for (int32_t d : gh0) rcnt[own_cell[d]][col0[d]]++;
    build_halo(h, h->l0_halo, g0, P, me, sendl, rcnt, no0);
  }
  {
    std::vector<int32_t> r0(no0 + 1, 0), c0v, rc0(no0);
    std::vector<double> v0;
    for (int32_t k = 0; k < no0; ++k) {
      const int32_t c = rows0[k];
      // same entry order as upload_level: natural column order of the row
      for (int32_t e = A0.rp[c]; e < A0.rp[c + 1]; ++e) { c0v.push_back(l0col[A0.ci[e]]); v0.push_back(A0.v[e]); }
      r0[k + 1] = (int32_t)c0v.size();
      rc0[k] = col0[c];
    }
    upload_level_rows(h, h->lv[0], no0, no0 + ng0, r0, c0v, v0, g0, rc0);
    h->n0_ghost = ng0;
  }
  // ---------------- levels 1..D partitioned (dist_levels, NEXT-3) and the hand-over to the
  // replicated part (levels > D and the coarsest; ROOT: rank 0 only)
  {
    const int D = h->dist_D;
    // owner of every row of levels 0..D+1: a level-(l+1) row (aggregate of level-l rows)
    // lives on the owner of its lowest-index member (level 1: whole aggregates per rank)
    std::vector<std::vector<int32_t>> own(D + 2);
    own[0] = own_cell;
    for (int l = 0; l <= D; ++l) {
      const auto& agg = S.lv[l].agg;
      own[l + 1].assign(S.lv[l].n_next, -1);
      for (int32_t i = S.lv[l].A.n - 1; i >= 0; --i) own[l + 1][agg[i]] = own[l][i];
    }
    // global row index of level l (the single-GPU color-major order; coarsest: natural)
    auto rowidx = [&](int l, int32_t i) { return (l < L) ? perms[l][i] : i; };
    struct LocLev {
      std::vector<int32_t> rows;             // owned rows (natural), global row order
      std::vector<int32_t> xloc, ploc, rloc; // natural -> local x (owned | matrix ghost),
                                             // x (owned | parent ghost), r (owned | member ghost)
      int32_t no = 0;
    };
    std::vector<LocLev> LL(D + 1);
    LL[0].rows = rows0;
    LL[0].no = no0;
    LL[0].rloc.assign(n, -1);
    for (int32_t k = 0; k < no0; ++k) LL[0].rloc[rows0[k]] = k;
    for (int l = 1; l <= D; ++l) {
      const msp::SpMat& Al = S.lv[l].A;
      const auto& col = S.lv[l].color;
      const int g = S.lv[l].ncolor;
      const int32_t nl = Al.n;
      const auto& ow = own[l];
      LocLev& Q = LL[l];
      LevelPlan LP = plan_level(S, perms, own, l, me, P);
      Q.rows = LP.rows;
      Q.no = (int32_t)Q.rows.size();
      std::vector<int32_t> lo(nl, -1);
      for (int32_t k = 0; k < Q.no; ++k) lo[Q.rows[k]] = k;
      const auto &gx = LP.gx, &gp = LP.gp, &gm = LP.gm;
      const auto &needx = LP.needx, &needp = LP.needp, &needm = LP.needm;
      const int32_t ngx = (int32_t)gx.size(), ngp = (int32_t)gp.size(), ngm = (int32_t)gm.size();
      Q.xloc = lo;
      Q.ploc = lo;
      Q.rloc = lo;
      for (int32_t k = 0; k < ngx; ++k) Q.xloc[gx[k]] = Q.no + k;
      for (int32_t k = 0; k < ngp; ++k) Q.ploc[gp[k]] = Q.no + ngx + k;
      for (int32_t k = 0; k < ngm; ++k) Q.rloc[gm[k]] = Q.no + k;
      // local rows (entries in the row's natural column order, as upload_level)
      std::vector<int32_t> r(Q.no + 1, 0), c, rc(Q.no);
      std::vector<double> v;
      for (int32_t k = 0; k < Q.no; ++k) {
        const int32_t i = Q.rows[k];
        for (int32_t e = Al.rp[i]; e < Al.rp[i + 1]; ++e) { c.push_back(Q.xloc[Al.ci[e]]); v.push_back(Al.v[e]); }
        r[k + 1] = (int32_t)c.size();
        rc[k] = col[i];
      }
      DevLevel& DL = h->lv[l];
      upload_level_rows(h, DL, Q.no, Q.no + ngx + ngp, r, c, v, g, rc, choose_lpr(Al.nnz(), nl, g), Q.no + ngm);
      DL.ngx = ngx;
      DL.ngp = ngp;
      DL.ngm = ngm;
      {
        std::vector<std::vector<std::vector<int32_t>>> sendl(P, std::vector<std::vector<int32_t>>(g));
        std::vector<std::vector<int32_t>> rcnt(P, std::vector<int32_t>(g, 0));
        for (int q = 0; q < P; ++q)
          for (int32_t d : needx[q]) sendl[q][col[d]].push_back(lo[d]);
        for (int32_t d : gx) rcnt[ow[d]][col[d]]++;
        build_halo(h, DL.xh, g, P, me, sendl, rcnt);
      }
      auto one_seg = [&](msp::HaloPlan& plan, const std::vector<std::vector<int32_t>>& need,
                         const std::vector<int32_t>& ghosts) {
        std::vector<std::vector<std::vector<int32_t>>> sendl(P, std::vector<std::vector<int32_t>>(1));
        std::vector<std::vector<int32_t>> rcnt(P, std::vector<int32_t>(1, 0));
        for (int q = 0; q < P; ++q)
          for (int32_t d : need[q]) sendl[q][0].push_back(lo[d]);
        for (int32_t d : ghosts) rcnt[ow[d]][0]++;
        build_halo(h, plan, 1, P, me, sendl, rcnt);
      };
      one_seg(DL.ph, needp, gp);
      one_seg(DL.mh, needm, gm);
    }
    // restriction lists (level l -> l+1, members in the single-GPU summation order:
    // ascending global level-l row) and prolongation maps of every partitioned level
    for (int l = 0; l <= D; ++l) {
      const auto& agg = S.lv[l].agg;
      const int32_t nl = S.lv[l].A.n, nn = S.lv[l].n_next;
      const bool next_dist = l + 1 <= D;
      std::vector<std::vector<int32_t>> owned_next(P);   // every rank's owned level-(l+1) rows, target order
      if (next_dist) owned_next[me] = LL[l + 1].rows;
      else {
        for (int32_t I = 0; I < nn; ++I) owned_next[own[l + 1][I]].push_back(I);
        for (int q = 0; q < P; ++q)
          std::sort(owned_next[q].begin(), owned_next[q].end(),
                    [&](int32_t x, int32_t y) { return rowidx(l + 1, x) < rowidx(l + 1, y); });
      }
      const std::vector<int32_t>& tgt = owned_next[me];
      const int32_t nt = (int32_t)tgt.size();
      std::vector<int32_t> slot(nn, -1);
      for (int32_t k = 0; k < nt; ++k) slot[tgt[k]] = k;
      std::vector<int32_t> inv(nl);
      for (int32_t i = 0; i < nl; ++i) inv[perms[l][i]] = i;
      std::vector<int32_t> pp(nt + 1, 0), pi;
      for (int32_t i = 0; i < nl; ++i) if (slot[agg[i]] >= 0) pp[slot[agg[i]] + 1]++;
      for (int32_t k = 0; k < nt; ++k) pp[k + 1] += pp[k];
      pi.assign(pp[nt], -1);
      {
        std::vector<int32_t> f(pp.begin(), pp.end() - 1);
        for (int32_t p = 0; p < nl; ++p) {                 // ascending global level-l row
          const int32_t i = inv[p];
          const int32_t k = slot[agg[i]];
          if (k < 0) continue;
          const int32_t li = LL[l].rloc[i];
          check_index(li >= 0, "restriction member without a local slot");
          pi[f[k]++] = li;
        }
      }
      // prolongation map of my level-l rows
      std::vector<int32_t> ap(LL[l].no);
      for (int32_t k = 0; k < LL[l].no; ++k) {
        const int32_t I = agg[LL[l].rows[k]];
        ap[k] = next_dist ? LL[l + 1].ploc[I] : rowidx(l + 1, I);
        check_index(ap[k] >= 0, "prolongation source without a local slot");
      }
      h->lv[l].agg = h->upload(ap);
      if (next_dist) {
        h->lv[l].pt_ptr = h->upload(pp);
        h->lv[l].pt_idx = h->upload(pi);
      } else {                                             // hand-over to the replicated part
        int cmax = 1;
        for (int q = 0; q < P; ++q) cmax = std::max(cmax, (int)owned_next[q].size());
        std::vector<int32_t> scat((size_t)P * cmax, -1);
        for (int q = 0; q < P; ++q)
          for (size_t k = 0; k < owned_next[q].size(); ++k) scat[(size_t)q * cmax + k] = rowidx(l + 1, owned_next[q][k]);
        h->n_own_l1 = nt;
        h->l1_cmax = cmax;
        h->own_l1_pt = h->upload(pp);
        h->own_l1_idx = h->upload(pi);
        h->l1_scatter = h->upload(scat);
        h->l1_send = h->dalloc<double>(cmax);
        h->l1_recv = h->dalloc<double>((size_t)P * cmax);
        CK(cudaMemsetAsync(h->l1_send, 0, sizeof(double) * cmax, h->s));
      }
    }
  }
  // cell <-> level-0 maps of the owned cells
  {
    std::vector<int32_t> l0(no), inv(no0);
    for (int32_t l = 0; l < no; ++l) l0[l] = l0loc[S.order[posown[l]]];
    for (int32_t l = 0; l < no; ++l) inv[l0[l]] = l;
    h->l0_of_cell = h->upload(l0);
    h->cell_of_l0 = h->upload(inv);
  }
  CK(cudaStreamSynchronize(h->s));
}

// ----------------------------------------------------------------- launches

template <int B>
void launch_spmv_t(cudaStream_t s, bool pdl, int mode, int n, const int* rp, const int* ci, const double* val,
                   const double* x, const double* g, double* y) {
  constexpr int TS = (B <= 4) ? 4 : 8;
  const unsigned grid = nblk((size_t)n * TS, 256);
  if (B == 4 && mode != 2) {
    const int* none = nullptr;
    if (mode == 0) klaunch(s, pdl, bsr_spmv4c_kernel<0>, grid, 256, n, rp, ci, val, x, g, y, none);
    else klaunch(s, pdl, bsr_spmv4c_kernel<1>, grid, 256, n, rp, ci, val, x, g, y, none);
    return;
  }
  if constexpr (B >= 5) {
    if (mode != 2) {
      if (mode == 0) klaunch(s, pdl, bsr_spmv8c_kernel<B, 0>, grid, 256, n, rp, ci, val, x, g, y);
      else klaunch(s, pdl, bsr_spmv8c_kernel<B, 1>, grid, 256, n, rp, ci, val, x, g, y);
      return;
    }
  }
  if (mode == 0) klaunch(s, pdl, bsr_spmv_kernel<B, 0>, grid, 256, n, rp, ci, val, x, g, y);
  else if (mode == 1) klaunch(s, pdl, bsr_spmv_kernel<B, 1>, grid, 256, n, rp, ci, val, x, g, y);
  else klaunch(s, pdl, bsr_spmv_kernel<B, 2>, grid, 256, n, rp, ci, val, x, g, y);
}

void launch_spmv(msp_handle* h, int mode, const double* x, const double* g, double* y) {
  ++h->nlaunch;
  const double* val = (mode == 2) ? h->Pcol : h->Aval;
  if (mode == 2 && h->pell_w) {
    klaunch(h->s, h->pdl, pcol_resid_ell4_kernel, nblk(h->n, 256), 256, (int)h->n, (int)h->n, (int)h->pell_w,
            (const int*)h->pell_c, (const double*)h->pell_v, x, g, y, (const int*)nullptr);
    return;
  }
  if (mode == 2 && h->b == 4) {
    klaunch(h->s, h->pdl, pcol_resid4_kernel, nblk((size_t)h->n * 4, 256), 256, h->n, h->rp, h->ci, val, x, g, y,
            (const int*)nullptr);
    return;
  }
  switch (h->b) {
#define CASE(BV) case BV: launch_spmv_t<BV>(h->s, h->pdl, mode, h->n, h->rp, h->ci, val, x, g, y); break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
  }
}

// Distributed mode, 4x4 blocks: y = A x (mode 0) or r = g - A[:,P] x_p (mode 2) with the z
// halo of x overlapped: the exchange runs on a side stream (fork/join by events; NCCL calls
// are captured into the step graph like the kernels) while the slab-interior rows (no
// ghost column) are computed, then the boundary rows.
void spmv_overlapped(msp_handle* h, int mode, double* x, int width, const double* g, double* y) {
  CK(cudaEventRecord(h->ev_fork, h->s));
  CK(cudaStreamWaitEvent(h->s2, h->ev_fork, 0));
  h->comm->halo(h->s2, h->cell_halo, x, h->n, width, -1);
  CK(cudaEventRecord(h->ev_join, h->s2));
  auto part = [&](const int32_t* rows, int nr) {
    if (nr <= 0) return;
    ++h->nlaunch;
    if (mode == 2 && h->pell_w)
      klaunch(h->s, h->pdl, pcol_resid_ell4_kernel, nblk(nr, 256), 256, nr, (int)h->n, (int)h->pell_w,
              (const int*)h->pell_c, (const double*)h->pell_v, (const double*)x, g, y, (const int*)rows);
    else if (mode == 2)
      klaunch(h->s, h->pdl, pcol_resid4_kernel, nblk((size_t)nr * 4, 256), 256, nr, (const int*)h->rp,
              (const int*)h->ci, (const double*)h->Pcol, (const double*)x, g, y, (const int*)rows);
    else
      klaunch(h->s, h->pdl, bsr_spmv4c_kernel<0>, nblk((size_t)nr * 4, 256), 256, nr, (const int*)h->rp,
              (const int*)h->ci, (const double*)h->Aval, (const double*)x, g, y, (const int*)rows);
  };
  part(h->rows_in, h->n_rows_in);
  CK(cudaStreamWaitEvent(h->s, h->ev_join, 0));
  part(h->rows_bd, h->n_rows_bd);
}
bool overlap_ok(const msp_handle* h) { return h->comm && h->b == 4 && h->s2 && h->overlap_halo; }

// halo exchanges of the distributed mode (no-ops on a single GPU)
void exch_cell(msp_handle* h, double* v, int width, int seg, bool packed = false) {
  if (h->comm) h->comm->halo(h->s, h->cell_halo, v, h->n, width, seg, packed);
}
void exch_l0(msp_handle* h, double* x, int seg, bool packed = false) {
  if (h->comm) h->comm->halo(h->s, h->l0_halo, x, h->lv[0].n, 1, seg, packed);
}

// half: 0 both substitutions (the MSP apply), 1 forward only (v: r -> y), 2 backward only
// (v: y -> x, z = x + wp) -- the halves exist for the per-kernel parity tests
template <int B, int MAXC, bool WF = false>
void launch_bilu_block(msp_handle* h, double* v, const double* wp, double* z, int half = 0) {
  constexpr int TM = MAXC * ((B <= 4) ? 4 : 8);
  const int g = h->bilu_ncolor;
  const bool fused_pack = h->comm && h->cell_halo.d_slots && h->fuse_halo && !h->prm.bilu_local && !half;
  auto run = [&](int c, int kind) {
    const int b0 = h->color_blk[c], b1 = h->color_blk[c + 1];
    if (b1 <= b0) return;
    const unsigned grid = nblk((size_t)(b1 - b0) * TM, 128);
    ++h->nlaunch;
    if constexpr (B >= 5 && !WF) {
      if (h->bm_f && !h->comm) {             // per-slot metadata, 8-lane groups
        auto kf = kind == 0 ? bilu_meta8_kernel<B, MAXC, true, false>
                            : (kind == 1 ? bilu_meta8_kernel<B, MAXC, false, true> : bilu_meta8_kernel<B, MAXC, true, true>);
        klaunch(h->s, h->pdl, kf, grid, 128, b0, b1, (const int4*)h->bm_f, (const int4*)h->bm_cf, (const int4*)h->bm_b,
                (const int4*)h->bm_cb, (const int4*)h->bm_sl, (const int*)h->ci, (const double*)h->Fval, v, wp, z);
        return;
      }
    }
    if constexpr (B == 4 && !WF) {
      if (h->bm_f && !h->comm) {             // per-slot metadata: shorter dependent load chain
        if (kind == 0)
          klaunch(h->s, h->pdl, bilu_meta4_kernel<MAXC, true, false>, grid, 128, b0, b1, (const int4*)h->bm_f,
                  (const int4*)h->bm_cf, (const int4*)h->bm_b, (const int4*)h->bm_cb, (const int4*)h->bm_sl,
                  (const int*)h->ci, (const double*)h->Fval, v, wp, z);
        else if (kind == 1)
          klaunch(h->s, h->pdl, bilu_meta4_kernel<MAXC, false, true>, grid, 128, b0, b1, (const int4*)h->bm_f,
                  (const int4*)h->bm_cf, (const int4*)h->bm_b, (const int4*)h->bm_cb, (const int4*)h->bm_sl,
                  (const int*)h->ci, (const double*)h->Fval, v, wp, z);
        else
          klaunch(h->s, h->pdl, bilu_meta4_kernel<MAXC, true, true>, grid, 128, b0, b1, (const int4*)h->bm_f,
                  (const int4*)h->bm_cf, (const int4*)h->bm_b, (const int4*)h->bm_cb, (const int4*)h->bm_sl,
                  (const int*)h->ci, (const double*)h->Fval, v, wp, z);
        return;
      }
    }
    // distributed: the kernel packs the halo of its color phase itself (v only: the BILU
    // vector whose ghosts the next phases read)
    const int2* sl = fused_pack ? (const int2*)h->cell_halo.d_slots : nullptr;
    double* sb = fused_pack ? h->cell_halo.d_sendbuf : nullptr;
    if (kind == 0)
      klaunch(h->s, h->pdl, bilu_block_kernel<B, MAXC, true, false, WF>, grid, 128, b0, b1, h->blk_ptr, h->rp, h->ci, h->dg, h->bcnt, (const int4*)h->islot, h->Fval, v, wp, z, sl, sb);
    else if (kind == 1)
      klaunch(h->s, h->pdl, bilu_block_kernel<B, MAXC, false, true, WF>, grid, 128, b0, b1, h->blk_ptr, h->rp, h->ci, h->dg, h->bcnt, (const int4*)h->islot, h->Fval, v, wp, z, sl, sb);
    else
      klaunch(h->s, h->pdl, bilu_block_kernel<B, MAXC, true, true, WF>, grid, 128, b0, b1, h->blk_ptr, h->rp, h->ci, h->dg, h->bcnt, (const int4*)h->islot, h->Fval, v, wp, z, sl, sb);
  };
  if (half == 1) {
    for (int c = 0; c < g; ++c) run(c, 0);
    return;
  }
  if (half == 2) {
    for (int c = g - 1; c >= 0; --c) run(c, 1);
    return;
  }
  // distributed: after each color phase, the ghost copies of that color's cells are
  // refreshed (y after the forward phase, x after the backward phase)
  // rank-local BILU: the factor blocks of couplings to other ranks are zero, ghost slots of v
  // are never read with a nonzero factor -> no exchange
  const bool ex = !h->prm.bilu_local;
  for (int c = 0; c < g - 1; ++c) { run(c, 0); if (ex) exch_cell(h, v, B, c, fused_pack); }
  run(g - 1, 2);
  if (g > 1 && ex) exch_cell(h, v, B, g - 1, fused_pack);
  for (int c = g - 2; c >= 0; --c) { run(c, 1); if (c > 0 && ex) exch_cell(h, v, B, c, fused_pack); }
}

template <int B>
void launch_bilu_t(msp_handle* h, double* v, const double* wp, double* z, bool wfull = false, int half = 0) {
  if (half) {
    if (h->max_blk > 4) throw std::pair<int, std::string>(MSP_EINVAL, "BILU halves need blocks of <= 4 cells");
    if (h->max_blk <= 1) launch_bilu_block<B, 1>(h, v, wp, z, half);
    else if (h->max_blk <= 2) launch_bilu_block<B, 2>(h, v, wp, z, half);
    else launch_bilu_block<B, 4>(h, v, wp, z, half);
    return;
  }
  if (wfull) {                                         // z = w (full vector) + R r
    if (h->max_blk <= 1) launch_bilu_block<B, 1, true>(h, v, wp, z);
    else if (h->max_blk <= 2) launch_bilu_block<B, 2, true>(h, v, wp, z);
    else launch_bilu_block<B, 4, true>(h, v, wp, z);
    return;
  }
  if (h->max_blk <= 4) {
    if (h->max_blk <= 1) launch_bilu_block<B, 1>(h, v, wp, z);
    else if (h->max_blk <= 2) launch_bilu_block<B, 2>(h, v, wp, z);
    else launch_bilu_block<B, 4>(h, v, wp, z);
    return;
  }
  // aggregate blocks of more than 4 cells (pair_passes >= 3): one team per block
  constexpr int TS = (B <= 4) ? 4 : 8;
  const int g = h->bilu_ncolor;
  auto run = [&](int c, int kind) {
    const int b0 = h->color_blk[c], b1 = h->color_blk[c + 1];
    if (b1 <= b0) return;
    const unsigned grid = nblk((size_t)(b1 - b0) * TS, 128);
    ++h->nlaunch;
    if (kind == 0)
      klaunch(h->s, h->pdl, bilu_color_kernel<B, true, false>, grid, 128, b0, b1, h->blk_ptr, h->rp, h->ci, h->dg, h->Fval, v, wp, z);
    else if (kind == 1)
      klaunch(h->s, h->pdl, bilu_color_kernel<B, false, true>, grid, 128, b0, b1, h->blk_ptr, h->rp, h->ci, h->dg, h->Fval, v, wp, z);
    else
      klaunch(h->s, h->pdl, bilu_color_kernel<B, true, true>, grid, 128, b0, b1, h->blk_ptr, h->rp, h->ci, h->dg, h->Fval, v, wp, z);
  };
  for (int c = 0; c < g - 1; ++c) run(c, 0);
  run(g - 1, 2);
  for (int c = g - 2; c >= 0; --c) run(c, 1);
}

void launch_bilu(msp_handle* h, double* v, const double* wp, double* z, bool wfull = false, int half = 0) {
  switch (h->b) {
#define CASE(BV) case BV: launch_bilu_t<BV>(h, v, wp, z, wfull, half); break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
  }
}

// a3 (+ the fused zero-guess first color of level 0 when it has a PGS-MC level)
void launch_restrict_pressure(msp_handle* h, const double* g, double* rp0, bool fuse_init, HaloPack pk = HaloPack{}) {
  const unsigned grid = nblk(h->n, 256);
  double* x0 = nullptr;
  const double* d0 = nullptr;
  int c1 = 0;
  if (fuse_init && !h->lv.empty() && h->prm.pre_sweeps > 0) {
    x0 = h->lv[0].x;
    d0 = h->lv[0].diag;
    c1 = h->lv[0].color_row[1];
  }
  switch (h->b) {
#define CASE(BV) case BV: klaunch(h->s, h->pdl, restrict_pressure_kernel<BV>, grid, 256, h->n, h->W, g, h->cell_of_l0, rp0, x0, d0, c1, pk); break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
  }
  ++h->nlaunch;
}

void coarsest_solve(msp_handle* h) {
  ++h->nlaunch;
  if (h->coarse_diag)
    klaunch(h->s, h->pdl, diag_solve_kernel, nblk(h->nL, 256), 256, h->nL, h->cdiag, h->bL, h->xL);
  else
    // 4 warps per row (C3: 30.8 vs 34.3 us for warp-per-row, which was removed)
    klaunch(h->s, h->pdl, gemv_row_kernel<4, 4>, h->nL, 128, h->nL, h->ldA, (const double*)h->Ainv,
            (const double*)h->bL, h->xL);
}

template <int LPR, bool WR, bool RES>
void sell_rows(msp_handle* h, DevLevel& L, int s0, int s1) {
  if (s1 <= s0) return;
  const int tpb = (LPR == 1) ? h->sell_tpb : 128;
  klaunch(h->s, h->pdl, sell_row_kernel<LPR, WR, RES>, nblk((size_t)(s1 - s0) * kSell * LPR, tpb), tpb, 
      s0, s1, L.slice_row, L.slice_off, L.col, L.val, L.diag, L.b, L.x, L.r);
  ++h->nlaunch;
}
// returns true when the kernel also packed the halo (pk given, uniform level-0 layout)
template <bool WR, bool RES>
bool sell_rows_any(msp_handle* h, DevLevel& L, int s0, int s1, HaloPack pk = HaloPack{}) {
  if (L.lpr == 1 && L.uniform_w > 0 && s1 > s0) {
    int c = 0;                                     // the color holding slice s0
    while (c + 1 < L.ncolor && L.color_slice[c + 1] <= s0) ++c;
    if (s1 <= L.color_slice[c + 1]) {              // range inside one color: uniform kernel
      const int row_first = L.color_row[c] + (s0 - L.color_slice[c]) * kSell;
      klaunch(h->s, h->pdl, sell_row_uniform_kernel<WR, RES>, nblk((size_t)(s1 - s0) * kSell, 128), 128, s0, s1,
              row_first, L.color_row[c + 1], L.uniform_w, (const int*)L.col, (const double*)L.val,
              (const double*)L.diag, (const double*)L.b, L.x, L.r, pk);
      ++h->nlaunch;
      return pk.slots != nullptr;
    }
  }
  switch (L.lpr) {
    case 2: sell_rows<2, WR, RES>(h, L, s0, s1); break;
    case 4: sell_rows<4, WR, RES>(h, L, s0, s1); break;
    case 8: sell_rows<8, WR, RES>(h, L, s0, s1); break;
    default: sell_rows<1, WR, RES>(h, L, s0, s1); break;
  }
  return false;
}

void sell_tail(msp_handle* h, DevLevel& L, int c0, int c1, bool asc, bool write_r) {
  switch (L.lpr) {
#define CASE(LP) case LP: klaunch(h->s, h->pdl, sell_tail_kernel<LP>, 1, 1024, c0, c1, asc, write_r, L.d_color_slice, \
      L.slice_row, L.slice_off, L.col, L.val, L.diag, L.b, L.x, L.r); break;
    CASE(2) CASE(4) CASE(8)
    default: klaunch(h->s, h->pdl, sell_tail_kernel<1>, 1, 1024, c0, c1, asc, write_r, L.d_color_slice, L.slice_row,
                                                       L.slice_off, L.col, L.val, L.diag, L.b, L.x, L.r);
#undef CASE
  }
  ++h->nlaunch;
}

// NEXT-4 comparison smoothers (R13): one PJAC-NO / PGS-NO sweep of level L.  The
// values at the start of the sweep are snapshotted into L.r (free during a sweep; the
// residual is written after the last pre-sweep), so neither kernel races with itself.
void no_sweep(msp_handle* h, DevLevel& L, bool ascending, bool from_zero, bool write_r) {
  if (from_zero) CK(cudaMemsetAsync(L.x, 0, sizeof(double) * L.n, h->s));
  CK(cudaMemcpyAsync(L.r, L.x, sizeof(double) * L.n, cudaMemcpyDeviceToDevice, h->s));
  if (h->prm.smoother == 1) {
    switch (L.lpr) {
#define CASE(LP) case LP: klaunch(h->s, h->pdl, sell_jacobi_kernel<LP>, nblk((size_t)L.nslices * kSell * LP, 128), 128, \
      0, L.nslices, L.slice_row, L.slice_off, L.col, L.val, L.diag, L.b, (const double*)L.r, L.x); break;
      CASE(2) CASE(4) CASE(8)
      default: klaunch(h->s, h->pdl, sell_jacobi_kernel<1>, nblk((size_t)L.nslices * kSell, 128), 128, 0, L.nslices,
                       L.slice_row, L.slice_off, L.col, L.val, L.diag, L.b, (const double*)L.r, L.x);
#undef CASE
    }
  } else {
    const int K = h->prm.gs_chunk;
    const int nchunk = (L.n + K - 1) / K;
    if (K < 16)
      klaunch(h->s, h->pdl, hybrid_gs_thread_kernel, nblk(nchunk, 128), 128, L.n, K, ascending ? 1 : 0, L.perm,
              L.inv, L.row_start, L.row_width, L.col, L.val, L.diag, L.b, (const double*)L.r, L.x);
    else
      klaunch(h->s, h->pdl, hybrid_gs_kernel, nblk(nchunk, kHgsWarps), 32 * kHgsWarps, L.n, K, ascending ? 1 : 0,
              L.perm, L.inv, L.row_start, L.row_width, L.col, L.val, L.diag, L.b, (const double*)L.r, L.x);
  }
  ++h->nlaunch;
  if (write_r) sell_rows_any<false, true>(h, L, 0, L.nslices);   // r = b - A x, every row
}

// One PGS-MC sweep of level L (Alg. 4).  write_r: the last color also writes the
// residual of its rows (caller then computes the residual of the other colors).
// from_zero: the first color starts from the zero guess; init_done: that first color was
// already computed by the kernel that produced b (fused a3 / restriction).
void pgs_sweep(msp_handle* h, DevLevel& L, bool ascending, bool from_zero, bool write_r = false,
               bool init_done = false) {
  if (h->prm.smoother != 0) {
    no_sweep(h, L, ascending, from_zero, write_r);
    return;
  }
  if (ascending) {
    int c = 0;
    if (from_zero) {
      if (!init_done) {
        klaunch(h->s, h->pdl, pgs_init_kernel, nblk(L.n, 256), 256, L.n, L.color_row[1], L.diag, L.b, L.x);
        ++h->nlaunch;
      }
      c = 1;
      if (L.ncolor == 1 && write_r) {              // single color: residual of all rows
        sell_rows_any<false, true>(h, L, 0, L.nslices);
        return;
      }
    }
    const int cend = std::min(L.ncolor, std::max(c, L.tail));
    for (; c < cend; ++c) {
      const bool last = (c == L.ncolor - 1);
      if (last && write_r) sell_rows_any<true, false>(h, L, L.color_slice[c], L.color_slice[c + 1]);
      else sell_rows_any<false, false>(h, L, L.color_slice[c], L.color_slice[c + 1]);
    }
    if (c < L.ncolor) sell_tail(h, L, c, L.ncolor - 1, true, write_r);
    if (write_r && L.ncolor > 1)                   // residual of colors 1..g-1 (not the last)
      sell_rows_any<false, true>(h, L, 0, L.color_slice[L.ncolor - 1]);
  } else {
    int c = L.ncolor - 1;
    if (L.tail <= c) {
      sell_tail(h, L, L.tail, c, false, false);
      c = L.tail - 1;
    }
    for (; c >= 0; --c) sell_rows_any<false, false>(h, L, L.color_slice[c], L.color_slice[c + 1]);
  }
}

// V-cycle on level l; input in lv[l].b (or bL), output in lv[l].x (or xL).
// init_done: the zero-guess first color of level l was fused into b's producer.
void vcycle(msp_handle* h, int l, bool init_done = false) {
  if (l == (int)h->lv.size()) {
    coarsest_solve(h);
    return;
  }
  DevLevel& L = h->lv[l];
  const bool last = (l + 1 == (int)h->lv.size());
  double* bn = last ? h->bL : h->lv[l + 1].b;
  double* xn = last ? h->xL : h->lv[l + 1].x;
  const int nn = last ? h->nL : h->lv[l + 1].n;
  for (int s = 0; s < h->prm.pre_sweeps; ++s)
    pgs_sweep(h, L, true, s == 0, s + 1 == h->prm.pre_sweeps, s == 0 && init_done);
  if (h->prm.pre_sweeps == 0) {
    CK(cudaMemsetAsync(L.x, 0, sizeof(double) * L.n, h->s));
    sell_rows_any<false, true>(h, L, 0, L.nslices);
  }
  const bool fuse_next = !last && h->prm.pre_sweeps > 0 && h->prm.smoother == 0;
  klaunch(h->s, h->pdl, restrict_kernel, nblk(nn, 256), 256, nn, L.pt_ptr, L.pt_idx, L.r, bn,
                                                   fuse_next ? h->lv[l + 1].x : nullptr,
                                                   fuse_next ? h->lv[l + 1].diag : nullptr,
                                                   fuse_next ? h->lv[l + 1].color_row[1] : 0);
  ++h->nlaunch;
  vcycle(h, l + 1, fuse_next);
  klaunch(h->s, h->pdl, prolong_kernel, nblk(L.n, 256), 256, L.n, L.agg, xn, L.x, HaloPack{}); ++h->nlaunch;
  for (int s = 0; s < h->prm.post_sweeps; ++s) pgs_sweep(h, L, false, false);
}

double* level0_b(msp_handle* h) { return h->lv.empty() ? h->bL : h->lv[0].b; }
double* level0_x(msp_handle* h) { return h->lv.empty() ? h->xL : h->lv[0].x; }

void vcycle_any(msp_handle* h, bool init_done = false) { vcycle(h, 0, init_done); }

void msp_apply_npr(msp_handle* h, const double* g, double* z);

// Distributed MSP (stages P, R): level 0 of the V-cycle is rank-local with halo
// exchanges after every color; levels >= 1 and the coarsest are replicated (allgather
// of the owned aggregates' right-hand side).
// Hand-over from the last partitioned level l (= dist_D) to the replicated part: the
// level-(l+1) right-hand side of every rank's owned aggregates (member ghosts of r
// already exchanged), allgathered and scattered with the fused first color; levels > l
// and the coarsest run on every rank (ROOT: rank 0, then a broadcast of the correction).
// Returns x_{l+1} (replicated numbering).
double* dist_handover(msp_handle* h, int l) {
  DevLevel& Lv = h->lv[l];
  const int L = (int)h->lv.size();
  if (h->n_own_l1 > 0) {
    klaunch(h->s, h->pdl, restrict_kernel, nblk(h->n_own_l1, 256), 256, h->n_own_l1, h->own_l1_pt, h->own_l1_idx,
            (const double*)Lv.r, h->l1_send, (double*)nullptr, (const double*)nullptr, 0);
    ++h->nlaunch;
  }
  h->comm->allgather(h->s, h->l1_send, h->l1_recv, h->l1_cmax);
  const bool last = l + 1 == L;
  const bool init = !last && h->prm.pre_sweeps > 0;
  double* bn = last ? h->bL : h->lv[l + 1].b;
  double* xn = last ? h->xL : h->lv[l + 1].x;
  const bool root_mode = h->prm.coarse_mode == 1;
  if (!root_mode || h->rank == 0) {
    klaunch(h->s, h->pdl, scatter_l1_kernel, nblk((size_t)h->nranks * h->l1_cmax, 256), 256, h->nranks * h->l1_cmax,
            (const int*)h->l1_scatter, (const double*)h->l1_recv, bn, init ? xn : (double*)nullptr,
            init ? (const double*)h->lv[l + 1].diag : (const double*)nullptr, init ? h->lv[l + 1].color_row[1] : 0);
    ++h->nlaunch;
    vcycle(h, l + 1, init);
  }
  if (root_mode) h->comm->broadcast(h->s, xn, last ? h->nL : h->lv[l + 1].n, 0);
  return xn;
}

// V-cycle on a partitioned level l (1 <= l <= dist_D): the level-0 pattern of
// msp_apply_dist -- a halo of the color after every color of the sweeps, the residual's
// member ghosts before the restriction, the next level's parent ghosts before the
// prolongation, all ghosts after it.  Same per-row arithmetic as the replicated V-cycle
// (bit-identical).  init_done: the first color was fused into the restriction.
void vcycle_dist(msp_handle* h, int l, bool init_done) {
  DevLevel& Lv = h->lv[l];
  const int g = Lv.ncolor;
  auto exch = [&](int c) { h->comm->halo(h->s, Lv.xh, Lv.x, Lv.n, 1, c); };
  CK(cudaMemsetAsync(Lv.x + Lv.n, 0, sizeof(double) * (Lv.ngx + Lv.ngp), h->s));   // zero guess of ghosts
  if (!init_done && Lv.n > 0) {
    klaunch(h->s, h->pdl, pgs_init_kernel, nblk(Lv.n, 256), 256, Lv.n, Lv.color_row[1], (const double*)Lv.diag,
            (const double*)Lv.b, Lv.x);
    ++h->nlaunch;
  }
  exch(0);
  for (int c = 1; c < g; ++c) {
    if (c == g - 1) sell_rows_any<true, false>(h, Lv, Lv.color_slice[c], Lv.color_slice[c + 1]);
    else sell_rows_any<false, false>(h, Lv, Lv.color_slice[c], Lv.color_slice[c + 1]);
    exch(c);
  }
  if (g > 1) sell_rows_any<false, true>(h, Lv, 0, Lv.color_slice[g - 1]);
  else sell_rows_any<false, true>(h, Lv, 0, Lv.nslices);
  h->comm->halo(h->s, Lv.mh, Lv.r, Lv.n, 1, -1);                             // member ghosts of r
  double* xn;
  if (l + 1 <= h->dist_D) {
    DevLevel& N = h->lv[l + 1];
    if (N.n > 0) {                                 // (a rank may own no row of a small level)
      klaunch(h->s, h->pdl, restrict_kernel, nblk(N.n, 256), 256, N.n, (const int*)Lv.pt_ptr, (const int*)Lv.pt_idx,
              (const double*)Lv.r, N.b, N.x, (const double*)N.diag, N.color_row[1]);
      ++h->nlaunch;
    }
    vcycle_dist(h, l + 1, true);
    h->comm->halo(h->s, N.ph, N.x, N.n + N.ngx, 1, -1);                      // parent ghosts
    xn = N.x;
  } else {
    xn = dist_handover(h, l);
  }
  if (Lv.n > 0) {
    klaunch(h->s, h->pdl, prolong_kernel, nblk(Lv.n, 256), 256, Lv.n, (const int*)Lv.agg, (const double*)xn, Lv.x,
            HaloPack{});
    ++h->nlaunch;
  }
  h->comm->halo(h->s, Lv.xh, Lv.x, Lv.n, 1, -1);
  for (int c = g - 1; c >= 0; --c) {
    sell_rows_any<false, false>(h, Lv, Lv.color_slice[c], Lv.color_slice[c + 1]);
    if (c > 0) exch(c);
  }
}

void msp_apply_dist(msp_handle* h, const double* g, double* z) {
  DevLevel& L0 = h->lv[0];
  CK(cudaMemsetAsync(L0.x + L0.n, 0, sizeof(double) * h->n0_ghost, h->s));    // zero guess of ghosts
  // producers pack the level-0 halo themselves (uniform level-0 layout)
  const HaloPack pk0 = (h->fuse_halo && h->l0_halo.d_slots) ? HaloPack{h->l0_halo.d_slots, h->l0_halo.d_sendbuf}
                                                            : HaloPack{nullptr, nullptr};
  launch_restrict_pressure(h, g, L0.b, true, pk0);                           // a3 + first color
  exch_l0(h, L0.x, 0, pk0.slots != nullptr);
  for (int c = 1; c < L0.ncolor; ++c) {
    bool packed;
    if (c == L0.ncolor - 1) packed = sell_rows_any<true, false>(h, L0, L0.color_slice[c], L0.color_slice[c + 1], pk0);
    else packed = sell_rows_any<false, false>(h, L0, L0.color_slice[c], L0.color_slice[c + 1], pk0);
    exch_l0(h, L0.x, c, packed);
  }
  if (L0.ncolor > 1) sell_rows_any<false, true>(h, L0, 0, L0.color_slice[L0.ncolor - 1]);
  else sell_rows_any<false, true>(h, L0, 0, L0.nslices);
  double* x1;
  if (h->dist_D >= 1) {                                                      // level 1 partitioned
    DevLevel& L1 = h->lv[1];
    if (L1.n > 0) {
      klaunch(h->s, h->pdl, restrict_kernel, nblk(L1.n, 256), 256, L1.n, (const int*)L0.pt_ptr, (const int*)L0.pt_idx,
              (const double*)L0.r, L1.b, L1.x, (const double*)L1.diag, L1.color_row[1]);
      ++h->nlaunch;
    }
    vcycle_dist(h, 1, true);
    h->comm->halo(h->s, L1.ph, L1.x, L1.n + L1.ngx, 1, -1);                 // parent ghosts
    x1 = L1.x;
  } else {
    x1 = dist_handover(h, 0);
  }
  klaunch(h->s, h->pdl, prolong_kernel, nblk(L0.n, 256), 256, L0.n, (const int*)L0.agg, (const double*)x1, L0.x, pk0);
  ++h->nlaunch;
  exch_l0(h, L0.x, -1, pk0.slots != nullptr);
  for (int c = L0.ncolor - 1; c >= 0; --c) {
    const bool packed = sell_rows_any<false, false>(h, L0, L0.color_slice[c], L0.color_slice[c + 1], c > 0 ? pk0 : HaloPack{});
    if (c > 0) exch_l0(h, L0.x, c, packed);
  }
  klaunch(h->s, h->pdl, gather_kernel, nblk(h->n, 256), 256, h->n, (const int*)h->l0_of_cell, (const double*)L0.x, h->wp);
  ++h->nlaunch;
  if (overlap_ok(h)) {
    spmv_overlapped(h, 2, h->wp, 1, g, h->r);                                // a8, halo overlapped
  } else {
    exch_cell(h, h->wp, 1, -1);
    launch_spmv(h, 2, h->wp, g, h->r);                                       // a8 (owned rows)
  }
  launch_bilu(h, h->r, h->wp, z);                                            // a9 with per-color halos
}

// z = B g (Alg. 1, stages P and R; internal order).  g must not alias z or h->r.

void msp_apply_dev(msp_handle* h, const double* g, double* z) {
  if (h->comm) {
    msp_apply_dist(h, g, z);
    return;
  }
  if (h->prm.stages == 3) {
    msp_apply_npr(h, g, z);
    return;
  }
  const bool fuse = h->prm.smoother == 0;
  {
    Nvtx nv("a3 pressure restriction");
    launch_restrict_pressure(h, g, level0_b(h), fuse);                 // a3: r_p = W^T g
  }
  {
    Nvtx nv("a4-a7 V-cycle (PGS-MC, transfers, coarsest)");
    vcycle_any(h, fuse);                                               // a4-a7: B_P
  }
  klaunch(h->s, h->pdl, gather_kernel, nblk(h->n, 256), 256, h->n, h->l0_of_cell, level0_x(h), h->wp); ++h->nlaunch;
  {
    Nvtx nv("a8 pressure-column residual");
    launch_spmv(h, 2, h->wp, g, h->r);                                 // a8: r = g - A Pi_P x_p
  }
  Nvtx nv("a9 BILU(0) substitution");
  launch_bilu(h, h->r, h->wp, z);                                      // a9: z = Pi_P x_p + R r
}

template <int B, int MAXC>
void launch_bgs_t(msp_handle* h, const double* r, double* w) {
  constexpr int TM = MAXC * ((B <= 4) ? 4 : 8);
  for (int c = 0; c < h->bilu_ncolor; ++c) {
    const int b0 = h->color_blk[c], b1 = h->color_blk[c + 1];
    if (b1 <= b0) continue;
    klaunch(h->s, h->pdl, bgs_block_kernel<B, MAXC>, nblk((size_t)(b1 - b0) * TM, 128), 128, b0, b1, h->blk_ptr,
            h->rp, h->ci, h->dg, h->bcnt, h->Aval, h->Dn, r, w);
    ++h->nlaunch;
  }
}
template <int B>
void launch_bgs_b(msp_handle* h, const double* r, double* w) {
  if (h->max_blk <= 1) launch_bgs_t<B, 1>(h, r, w);
  else if (h->max_blk <= 2) launch_bgs_t<B, 2>(h, r, w);
  else launch_bgs_t<B, 4>(h, r, w);
}
void launch_bgs(msp_handle* h, const double* r, double* w) {
  switch (h->b) {
#define CASE(BV) case BV: launch_bgs_b<BV>(h, r, w); break;
    CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
  }
}

// Alg. 1 with all three stages (N, P, R; Eq. 21): w = Π_N B_N Π_N^T g; r = g - A w;
// w += Π_P B_P W^T r; r = g - A w; z = w + R r.
void msp_apply_npr(msp_handle* h, const double* g, double* z) {
  launch_bgs(h, g, h->wfull);                                          // line 2 (r = g)
  launch_spmv(h, 1, h->wfull, g, h->r1);                               // line 3: r = g - A w
  const bool fuse = h->prm.smoother == 0;
  launch_restrict_pressure(h, h->r1, level0_b(h), fuse);
  vcycle(h, 0, fuse);                                                  // line 4
  klaunch(h->s, h->pdl, gather_kernel, nblk(h->n, 256), 256, h->n, h->l0_of_cell, level0_x(h), h->wp);
  ++h->nlaunch;
  klaunch(h->s, h->pdl, set_pressure_kernel, nblk(h->n, 256), 256, h->n, h->b, h->wp, h->wfull);
  ++h->nlaunch;
  launch_spmv(h, 1, h->wfull, g, h->r);                                // line 5: r = g - A w
  launch_bilu(h, h->r, h->wfull, z, true);                             // line 6: z = w + R r
}

// ----------------------------------------------------------------- GMRES pieces
template <int NV>
void multidot_t(msp_handle* h, int nv, const double* V, const double* w) {
  klaunch(h->s, h->pdl, multidot_kernel<NV>, kRedBlocks, kRedThreads, h->N, nv, V, h->N, w, h->part); ++h->nlaunch;
}
template <int NV>
void maxpy_t(msp_handle* h, int nv, const double* V, const double* coef, double* w, int from_zero, double* part) {
  klaunch(h->s, h->pdl, multiaxpy_kernel<NV>, kRedBlocks, kRedThreads, h->N, nv, V, h->N, coef, w, from_zero, part, 0); ++h->nlaunch;
}
void cgs_dot(msp_handle* h, int nv, const double* V, const double* w, double* out, const double* addend,
             double* raw, int sq);

// ||w||^2 -> out[0] = ||w||
void norm_dev(msp_handle* h, const double* w, double* out) {
  if (h->comm) {
    cgs_dot(h, 1, w, w, h->lred, nullptr, nullptr, -1);
    h->comm->allreduce_sum(h->s, h->lred, 1);
    klaunch(h->s, h->pdl, sqrt_kernel, 1, 32, (const double*)h->lred, out);
    ++h->nlaunch;
    return;
  }
  multidot_t<4>(h, 1, w, w);
  klaunch(h->s, h->pdl, reduce_parts_kernel, 1, 1024, kRedBlocks, 1, h->part, out, nullptr, 0); ++h->nlaunch;
}

constexpr bool kCgsWide32 = false;         // NV=32 basis kernels use 8-byte loads

// 16-byte basis loads need an even vector length (N odd: 8-byte loads; V slots stay
// N apart, so an odd N also breaks 16-byte alignment of V[1], V[3], ...)
bool ew2_ok(const msp_handle* h) { return (h->N % 2) == 0; }

template <int NV>
void cgs_dot_t(msp_handle* h, int nv, const double* V, const double* w, double* out, const double* addend,
               double* raw, int sq) {
  constexpr int MINB = 2;
  if ((NV <= 16 || kCgsWide32) && ew2_ok(h))
    klaunch(h->s, h->pdl, cgs_dot_kernel<NV, 2, MINB>, kRedBlocks, kRedThreads, h->N / 2, nv, V, h->N, w, h->part, out,
            addend, raw, sq, h->ticket);
  else
    klaunch(h->s, h->pdl, cgs_dot_kernel<NV, 1, MINB>, kRedBlocks, kRedThreads, h->N, nv, V, h->N, w, h->part, out,
            addend, raw, sq, h->ticket);
  ++h->nlaunch;
}
void cgs_dot(msp_handle* h, int nv, const double* V, const double* w, double* out, const double* addend,
             double* raw, int sq) {
  if (nv <= 4) cgs_dot_t<4>(h, nv, V, w, out, addend, raw, sq);
  else if (nv <= 8) cgs_dot_t<8>(h, nv, V, w, out, addend, raw, sq);
  else if (nv <= 16) cgs_dot_t<16>(h, nv, V, w, out, addend, raw, sq);
  else {
    // 16 vectors per CTA row (gridDim.y = 2), 16-byte loads: full occupancy instead of
    // 32 accumulators per thread
    if (ew2_ok(h))
      klaunch(h->s, h->pdl, cgs_dot_kernel<16, 2, 2>, dim3(kRedBlocks, (nv + 15) / 16), kRedThreads, h->N / 2, nv, V,
              h->N, w, h->part, out, addend, raw, sq, h->ticket);
    else
      klaunch(h->s, h->pdl, cgs_dot_kernel<16, 1, 2>, dim3(kRedBlocks, (nv + 15) / 16), kRedThreads, h->N, nv, V,
              h->N, w, h->part, out, addend, raw, sq, h->ticket);
    ++h->nlaunch;
  }
}
template <int NV, bool DOT>
void cgs_axpy_t(msp_handle* h, int nv, const double* V, const double* coef, double* w, double* out,
                const double* addend, double* raw, int sq) {
  constexpr int MINB = 2;
  if ((NV <= 16 || kCgsWide32) && ew2_ok(h))
    klaunch(h->s, h->pdl, cgs_axpy_kernel<NV, 2, DOT, NV, MINB>, kRedBlocks, kRedThreads, h->N / 2, nv, V, h->N, coef, w,
            h->part, out, addend, raw, sq, h->ticket);
  else
    klaunch(h->s, h->pdl, cgs_axpy_kernel<NV, 1, DOT, NV, MINB>, kRedBlocks, kRedThreads, h->N, nv, V, h->N, coef, w,
            h->part, out, addend, raw, sq, h->ticket);
  ++h->nlaunch;
}
template <bool DOT>
void cgs_axpy(msp_handle* h, int nv, const double* V, const double* coef, double* w, double* out,
              const double* addend, double* raw, int sq) {
  if (nv <= 4) cgs_axpy_t<4, DOT>(h, nv, V, coef, w, out, addend, raw, sq);
  else if (nv <= 8) cgs_axpy_t<8, DOT>(h, nv, V, coef, w, out, addend, raw, sq);
  else if (nv <= 16) cgs_axpy_t<16, DOT>(h, nv, V, coef, w, out, addend, raw, sq);
  else if (DOT) {
    // nv > 16: the fused pass would need 32 accumulators per thread (25% occupancy);
    // instead the (fast) 32-vector axpy, then the row-split dot of the updated w
    cgs_axpy_t<32, false>(h, nv, V, coef, w, h->lred, nullptr, nullptr, -1);
    cgs_dot(h, nv, V, w, out, addend, raw, sq);
  } else cgs_axpy_t<32, DOT>(h, nv, V, coef, w, out, addend, raw, sq);
}

// CGS2 (R8) on w = V[nv] against V[0..nv): hcol[0..nv) = h1 + h2, hcol[nv] = ||w||,
// V[nv] = w / ||w||.  Three passes over the basis:
//   A: h1 = V^T w;  B: w -= V h1 and h2 = V^T w (fused);  C: w -= V h2 and ||w||^2.
void cgs2_dist(msp_handle* h, int nv, double* w) {
  // local partial sums, then sums over ranks; arithmetic per element as cgs2
  cgs_dot(h, nv, h->V, w, h->dh1, nullptr, nullptr, -1);
  h->comm->allreduce_sum(h->s, h->dh1, nv);
  cgs_axpy<true>(h, nv, h->V, h->dh1, w, h->dh2, nullptr, nullptr, -1);
  h->comm->allreduce_sum(h->s, h->dh2, nv);
  klaunch(h->s, h->pdl, add_vec_kernel, 1, 64, nv, (const double*)h->dh1, (const double*)h->dh2, h->hcol);
  cgs_axpy<false>(h, nv, h->V, h->dh2, w, h->lred, nullptr, nullptr, -1);
  h->comm->allreduce_sum(h->s, h->lred, 1);
  klaunch(h->s, h->pdl, sqrt_kernel, 1, 32, (const double*)h->lred, h->hcol + nv);
  klaunch(h->s, h->pdl, scale_kernel, kRedBlocks, kRedThreads, h->N, (const double*)w, (const double*)(h->hcol + nv), w);
  h->nlaunch += 3;
}

void cgs2(msp_handle* h, int nv, double* w) {
  if (h->comm) {
    cgs2_dist(h, nv, w);
    return;
  }
  cgs_dot(h, nv, h->V, w, h->dh1, nullptr, nullptr, -1);
  cgs_axpy<true>(h, nv, h->V, h->dh1, w, h->hcol, h->dh1, h->dh2, -1);
  cgs_axpy<false>(h, nv, h->V, h->dh2, w, h->hcol + nv, nullptr, nullptr, 0);
  klaunch(h->s, h->pdl, scale_kernel, kRedBlocks, kRedThreads, h->N, w, h->hcol + nv, w);
  ++h->nlaunch;
}

// DCGS2 passes of step k (R14, kernels.cuh): w = V[k+1] = A B V[k] on entry; on exit
// V[k] final, V[k+1] = u (provisional, unnormalised), hcol = the host record (2k+4 values).
template <int NV, int TPB, int NBUF = 2>
void dcgs_staged_launch(msp_handle* h, int k, double* vk, double* w, const double* st_in) {
  constexpr size_t smem = sizeof(double2) * NBUF * (NV + 2) * TPB;
  // per device (cheap host call; inside a step it runs once, at graph capture)
  CK(cudaFuncSetAttribute(dcgs_update_staged_kernel<NV, TPB, NBUF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int nsm = 148;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, h->device));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nsm);                       // one CTA per SM, grid-stride over pairs
  cfg.blockDim = dim3(TPB);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = h->s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = h->pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, dcgs_update_staged_kernel<NV, TPB, NBUF>, h->N / 2, k, (const double*)h->V, h->N, vk, w,
                        (const double*)h->dh1, st_in, h->part, h->dsum, h->ticket));
  ++h->nlaunch;
  if (h->comm) h->comm->allreduce_sum(h->s, h->dsum, k + 2);
}

template <int NV>
void dcgs_update_t(msp_handle* h, int k, double* vk, double* w, const double* st_in) {
  constexpr bool DOT = NV <= 16;
  // staged (cp.async) pass 2, one CTA per SM: k <= 8 at 1024 threads, 9 <= k <= 16 at 512
  // and k > 16 at 256 threads, single-buffered (C3: orthogonalisation at k = 15 0.295 ->
  // 0.255 ms, at k = 25 0.503 -> 0.457 ms; double-buffered forms measured slower, removed)
  if constexpr (NV == 8) {
    if (ew2_ok(h)) { dcgs_staged_launch<8, 1024, 1>(h, k, vk, w, st_in); return; }
  }
  if constexpr (NV == 16) {
    if (ew2_ok(h)) { dcgs_staged_launch<16, 512, 1>(h, k, vk, w, st_in); return; }
  }
  if constexpr (NV == 32) {                       // fused staged pass 2 for k > 16
    if (ew2_ok(h)) { dcgs_staged_launch<32, 256, 1>(h, k, vk, w, st_in); return; }
  }
  if (ew2_ok(h))
    klaunch(h->s, h->pdl, dcgs_update_kernel<NV, 2, DOT>, kRedBlocks, kRedThreads, h->N / 2, k, (const double*)h->V,
            h->N, vk, w, (const double*)h->dh1, st_in, h->part, h->dsum, h->ticket);
  else
    klaunch(h->s, h->pdl, dcgs_update_kernel<NV, 1, DOT>, kRedBlocks, kRedThreads, h->N, k, (const double*)h->V,
            h->N, vk, w, (const double*)h->dh1, st_in, h->part, h->dsum, h->ticket);
  ++h->nlaunch;
  if (!DOT) cgs_dot(h, k + 2, h->V, w, h->dsum, nullptr, nullptr, -1);   // V[0..k]^T u and u^T u
  if (h->comm) h->comm->allreduce_sum(h->s, h->dsum, k + 2);              // distributed: global sums
}
void dcgs2(msp_handle* h, int k) {
  const size_t N = h->N;
  double* vk = h->V + (size_t)k * N;
  double* w = h->V + (size_t)(k + 1) * N;
  const double* st_in = h->dst + (size_t)((k + 1) & 1) * (kMaxV + 2);
  double* st_out = h->dst + (size_t)(k & 1) * (kMaxV + 2);
  cgs_dot(h, k + 1, h->V, w, h->dh1, nullptr, nullptr, -1);                // pass 1: a
  if (h->comm) h->comm->allreduce_sum(h->s, h->dh1, k + 1);
  if (k <= 4) dcgs_update_t<4>(h, k, vk, w, st_in);                          // pass 2
  else if (k <= 8) dcgs_update_t<8>(h, k, vk, w, st_in);
  else if (k <= 16) dcgs_update_t<16>(h, k, vk, w, st_in);
  else dcgs_update_t<32>(h, k, vk, w, st_in);
  klaunch(h->s, h->pdl, dcgs_finish_kernel, 1, 32, k, (const double*)h->dh1, st_in, (const double*)h->dsum, st_out,
          h->hcol);
  ++h->nlaunch;
}

// One Arnoldi step j: z = B v_j; w = A z (into V[j+1]); orthogonalise (CGS2 or MGS);
// hcol[0..j+1] = H(:, j); V[j+1] normalised; hcol copied to pinned host memory.
void arnoldi_step(msp_handle* h, int j, bool record_to_host = true) {
  const size_t N = h->N;
  double* vj = h->V + (size_t)j * N;
  double* w = h->V + (size_t)(j + 1) * N;
  msp_apply_dev(h, vj, h->z);
  {
    Nvtx nvt("a2 BSR SpMV");
    if (overlap_ok(h)) {
      spmv_overlapped(h, 0, h->z, h->b, nullptr, w);
    } else {
      exch_cell(h, h->z, h->b, -1);
      launch_spmv(h, 0, h->z, nullptr, w);
    }
  }
  Nvtx nvt("a10 orthogonalisation");
  const int nv = j + 1;
  if (h->prm.orth == 2) {
    dcgs2(h, j);
    if (record_to_host)
      CK(cudaMemcpyAsync(h->hrec + (size_t)j * kRecStride, h->hcol, sizeof(double) * (2 * j + 4), cudaMemcpyDeviceToHost, h->s));
    return;
  }
  if (h->prm.orth == 0) {
    cgs2(h, nv, w);
  } else {
    for (int i = 0; i < nv; ++i) {
      multidot_t<4>(h, 1, h->V + (size_t)i * N, w);
      klaunch(h->s, h->pdl, reduce_parts_kernel, 1, 1024, kRedBlocks, 1, h->part, h->hcol + i, nullptr, -1); ++h->nlaunch;
      maxpy_t<4>(h, 1, h->V + (size_t)i * N, h->hcol + i, w, 0, (i == nv - 1) ? h->part : nullptr);
    }
    klaunch(h->s, h->pdl, reduce_parts_kernel, 1, 1024, kRedBlocks, 1, h->part, h->hcol + nv, nullptr, 0); ++h->nlaunch;
    klaunch(h->s, h->pdl, scale_kernel, kRedBlocks, kRedThreads, N, w, h->hcol + nv, w); ++h->nlaunch;
  }
  if (record_to_host)
    CK(cudaMemcpyAsync(h->hrec + (size_t)j * kRecStride, h->hcol, sizeof(double) * (nv + 1), cudaMemcpyDeviceToHost, h->s));
}

// One restart cycle of GMRES(m) as ONE executable graph: a chain of m conditional (IF)
// nodes; body j = the kernels of Arnoldi step j (captured into the body) followed by
// givens_kernel, which performs the Givens update and convergence test on the device and
// enables body j+1 (its handle is reset to 0 at every launch).  The host synchronises once
// per cycle instead of once per step.  Single-GPU, CGS2 / DCGS2.
void build_cycle_graph(msp_handle* h, int m) {
  if (h->cycle_exec) { cudaGraphExecDestroy(h->cycle_exec); h->cycle_exec = nullptr; }
  cudaGraph_t root;
  CK(cudaGraphCreate(&root, 0));
  std::vector<cudaGraphConditionalHandle> hd(m);
  for (int j = 0; j < m; ++j)
    CK(cudaGraphConditionalHandleCreate(&hd[j], root, j == 0 ? 1u : 0u, cudaGraphCondAssignDefault));
  h->cycle_kernels.assign(m, 0);
  cudaGraphNode_t prev = nullptr;
  for (int j = 0; j < m; ++j) {
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = hd[j];
    np.conditional.type = cudaGraphCondTypeIf;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, root, prev ? &prev : nullptr, prev ? 1 : 0, &np));
    cudaGraph_t body = np.conditional.phGraph_out[0];
    const int64_t before = h->nlaunch;
    CK(cudaStreamBeginCaptureToGraph(h->s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    arnoldi_step(h, j, false);
    const cudaGraphConditionalHandle nx = (j + 1 < m) ? hd[j + 1] : hd[j];
    if (h->prm.orth == 2)
      klaunch(h->s, h->pdl, givens_kernel<true>, 1, 32, j, m, (const double*)h->hcol, h->gv, nx, (j + 1 < m) ? 1 : 0);
    else
      klaunch(h->s, h->pdl, givens_kernel<false>, 1, 32, j, m, (const double*)h->hcol, h->gv, nx, (j + 1 < m) ? 1 : 0);
    cudaGraph_t out;
    CK(cudaStreamEndCapture(h->s, &out));
    h->cycle_kernels[j] = h->nlaunch - before;
    h->nlaunch = before;
    prev = node;
  }
  CK(cudaGraphInstantiate(&h->cycle_exec, root, 0));
  cudaGraphDestroy(root);
  h->cycle_m = m;
  h->kernels_per_step = (int)(h->cycle_kernels.empty() ? 0 : h->cycle_kernels[0]);
}

void ensure_basis(msp_handle* h, int m) {
  if (h->V_m >= m) return;
  h->V = h->dalloc<double>((size_t)(m + 1) * h->N);
  h->V_m = m;
  for (auto g : h->graphs) if (g) cudaGraphExecDestroy(g);
  h->graphs.clear();
  h->graphs_m = -1;
  if (h->cycle_exec) { cudaGraphExecDestroy(h->cycle_exec); h->cycle_exec = nullptr; }
  h->cycle_m = -1;
}

void run_step(msp_handle* h, int j, int m) {
  if (!h->prm.use_graphs) {
    arnoldi_step(h, j);
    return;
  }
  if (h->graphs_m != m) {
    for (auto g : h->graphs) if (g) cudaGraphExecDestroy(g);
    h->graphs.assign(m, nullptr);
    h->graphs_m = m;
  }
  if (!h->graphs[j]) {
    cudaGraph_t graph;
    const int64_t before = h->nlaunch;
    CK(cudaStreamBeginCapture(h->s, cudaStreamCaptureModeThreadLocal));
    arnoldi_step(h, j);
    CK(cudaStreamEndCapture(h->s, &graph));
    if ((int)h->graph_kernels.size() < m) h->graph_kernels.assign(m, 0);
    h->graph_kernels[j] = h->nlaunch - before;
    h->nlaunch = before;
    CK(cudaGraphInstantiate(&h->graphs[j], graph, 0));
    if (j == 0) {
      h->kernels_per_step = (int)h->graph_kernels[j];
    }
    cudaGraphDestroy(graph);
  }
  CK(cudaGraphLaunch(h->graphs[j], h->s));
  h->nlaunch += h->graph_kernels[j];
}

// GMRES(m), right preconditioned (R8); vectors internal order; xin holds x0 and
// the solution; bin holds b.
constexpr double kSpecMargin = 3.0;         // enqueue the next step while est > 3 tol

msp_status gmres(msp_handle* h, double tol, int m, int maxit, int* iters, double* final_rel,
                 double* hist, int cap, int* hlen) {
  const size_t N = h->N;
  ensure_basis(h, m);
  Nvtx nv_gmres("GMRES solve");
  int it = 0, hl = 0;
  auto push = [&](double v) { if (hist && hl < cap) hist[hl] = v; ++hl; };
  norm_dev(h, h->bin, h->hcol);
  CK(cudaMemcpyAsync(h->hpin, h->hcol, sizeof(double), cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  const double bnorm = h->hpin[0];
  *iters = 0;
  if (bnorm == 0.0) {
    CK(cudaMemsetAsync(h->xin, 0, sizeof(double) * N, h->s));
    *final_rel = 0.0;
    if (hlen) *hlen = 0;
    return MSP_OK;
  }
  exch_cell(h, h->xin, h->b, -1);
  launch_spmv(h, 1, h->xin, h->bin, h->r);                    // r = b - A x0
  norm_dev(h, h->r, h->hcol);
  CK(cudaMemcpyAsync(h->hpin, h->hcol, sizeof(double), cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  double beta = h->hpin[0];
  double rel = beta / bnorm;
  msp_status status = MSP_OK;
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), gam(m + 1), y(m);
  // DCGS2 (R14): unrotated Hessenberg columns and the previous step's h2, nu, rho
  std::vector<double> Hraw((size_t)(m + 1) * m), h2p;
  double nup = 1.0, rhop = 1.0;
  if (rel > tol) {
    while (true) {
      klaunch(h->s, h->pdl, scale_kernel, kRedBlocks, kRedThreads, N, h->r, h->hcol, h->V); ++h->nlaunch;   // v_0 = r / beta
      std::fill(gam.begin(), gam.end(), 0.0);
      gam[0] = beta;
      h2p.clear();
      nup = 1.0;
      rhop = 1.0;
      int k = 0;
      bool broke = false;                    // happy breakdown: h_{j+1,j} < 1e-14 ||b||
      const bool cyc = h->prm.use_graphs && h->cycle_graphs && !h->comm && h->prm.orth != 1;
      if (cyc) {
        // the whole cycle on the device: givens_kernel replaces the host loop below
        if (h->cycle_m != m) build_cycle_graph(h, m);
        klaunch(h->s, false, givens_init_kernel, 1, 256, h->gv, (const double*)h->hcol, bnorm, tol, (double)it,
                (double)maxit);
        ++h->nlaunch;
        CK(cudaGraphLaunch(h->cycle_exec, h->s));
        CK(cudaMemcpyAsync(h->hgv, h->gv, sizeof(double) * kGvSize, cudaMemcpyDeviceToHost, h->s));
        CK(cudaStreamSynchronize(h->s));
        const double* g = h->hgv;
        k = (int)g[kGvScal + 4];
        broke = g[kGvScal + 5] != 0.0;
        for (int j = 0; j < k; ++j) {
          push(g[kGvHist + j]);
          h->nlaunch += h->cycle_kernels[j];
          for (int i = 0; i <= j + 1; ++i) H[(size_t)i * m + j] = g[kGvH + i * kGv + j];
        }
        for (int i = 0; i <= k; ++i) gam[i] = g[kGvGam + i];
        it += k;
      }
      // Step j+1 is enqueued before the host reads step j's record (its own pinned slot)
      // while the residual estimate is more than kSpecMargin x tol away: the GPU runs on
      // through the host's Givens update.  A step enqueued past convergence is wasted work
      // only (it writes V[j+2] and the DCGS2 state of step j+1; the cycle end reads V[0..j]
      // and the host's y; step 0 of a cycle reads no lagged state): identical results.
      int launched = -1;
      double est_prev = rel;
      auto launch = [&](int jj) {
        run_step(h, jj, m);
        CK(cudaEventRecord(h->ev_step[jj & 1], h->s));
        launched = jj;
      };
      for (int j = 0; j < m && !cyc; ++j) {
        if (launched < j) launch(j);
        if (h->spec_steps && j + 1 < m && it + 1 < maxit && est_prev > kSpecMargin * tol) launch(j + 1);
        CK(cudaEventSynchronize(h->ev_step[j & 1]));
        const double* hr = h->hrec + (size_t)j * kRecStride;
        auto Hc = [&](int i) -> double& { return H[(size_t)i * m + j]; };
        if (h->prm.orth == 2) {
          // column j of the final basis: (nu [c + h2'; rho'] - sum_l h2_l Hraw[:, l]) / rho
          const double* rec = hr;
          for (int i = 0; i <= j + 1; ++i) {
            double v = nup * ((i <= j) ? rec[i] : rec[j + 1]);
            for (int l = 0; l < j; ++l) v -= h2p[l] * Hraw[(size_t)i * m + l];
            Hraw[(size_t)i * m + j] = v / rhop;
            Hc(i) = Hraw[(size_t)i * m + j];
          }
          h2p.assign(rec + j + 3, rec + 2 * j + 4);
          nup = rec[j + 2];
          rhop = rec[j + 1];
        } else {
          for (int i = 0; i <= j + 1; ++i) Hc(i) = hr[i];
        }
        const double hn = Hc(j + 1);
        ++it;
        for (int i = 0; i < j; ++i) {
          const double a = Hc(i), c = Hc(i + 1);
          Hc(i) = cs[i] * a + sn[i] * c;
          Hc(i + 1) = -sn[i] * a + cs[i] * c;
        }
        const double rho = std::hypot(Hc(j), Hc(j + 1));
        cs[j] = Hc(j) / rho;
        sn[j] = Hc(j + 1) / rho;
        Hc(j) = rho;
        Hc(j + 1) = 0.0;
        gam[j + 1] = -sn[j] * gam[j];
        gam[j] = cs[j] * gam[j];
        const double est = std::fabs(gam[j + 1]) / bnorm;
        est_prev = est;
        push(est);
        k = j + 1;
        broke = hn < 1e-14 * bnorm;
        if (est <= tol || broke || it >= maxit) break;
      }
      for (int i = k - 1; i >= 0; --i) {
        double s = 0.0;
        for (int l = i + 1; l < k; ++l) s += H[(size_t)i * m + l] * y[l];
        y[i] = (gam[i] - s) / H[(size_t)i * m + i];
      }
      Nvtx nv_end("a11 cycle end");
      // u = V_k y ; x += B u ; r = b - A x
      // u = V y through the CGS axpy pass on a zeroed u with coefficients -y (the same
      // fma(y_i, V_i, .) sequence as a plain V y, with the multi-vector pass's loads)
      for (int i = 0; i < k; ++i) y[i] = -y[i];
      CK(cudaMemcpyAsync(h->dh1, y.data(), sizeof(double) * k, cudaMemcpyHostToDevice, h->s));
      CK(cudaMemsetAsync(h->u, 0, sizeof(double) * N, h->s));
      cgs_axpy<false>(h, k, h->V, h->dh1, h->u, h->lred, nullptr, nullptr, -1);
      msp_apply_dev(h, h->u, h->z);
      klaunch(h->s, h->pdl, axpy_kernel, kRedBlocks, kRedThreads, N, 1.0, h->z, h->xin); ++h->nlaunch;
      exch_cell(h, h->xin, h->b, -1);
      launch_spmv(h, 1, h->xin, h->bin, h->r);
      norm_dev(h, h->r, h->hcol);
      CK(cudaMemcpyAsync(h->hpin, h->hcol, sizeof(double), cudaMemcpyDeviceToHost, h->s));
      CK(cudaStreamSynchronize(h->s));
      beta = h->hpin[0];
      rel = beta / bnorm;
      push(rel);
      if (rel <= tol) break;
      // the Krylov space became invariant yet the true residual is above tol: restarting
      // cannot help (the preconditioned operator is singular on it)
      if (broke) { status = MSP_EBREAKDOWN; break; }
      if (it >= maxit) { status = MSP_ENOCONV; break; }
    }
  }
  *iters = it;
  *final_rel = rel;
  if (hlen) *hlen = std::min(hl, cap);
  return status;
}

msp_status fail(msp_handle* h, msp_status st, const std::string& msg) {
  if (h) h->err = msg;
  g_last_error = msg;
  return st;
}

template <class F>
msp_status guarded(msp_handle* h, F&& f) {
  try {
    return f();
  } catch (const CudaError& e) {
    return fail(h, e.e == cudaErrorMemoryAllocation ? MSP_ENOMEM : MSP_ECUDA,
                std::string("CUDA: ") + cudaGetErrorString(e.e) + " in " + e.where);
  } catch (const std::pair<int, std::string>& e) {
    return fail(h, (msp_status)e.first, e.second);
  } catch (const std::bad_alloc&) {
    return fail(h, MSP_ENOMEM, "host allocation failed");
  }
}

// Every entry point that reads caller buffers first orders the handle's (non-blocking)
// stream after the work already queued on the caller's stream, so a buffer written there
// (e.g. by PyTorch on the legacy default stream) is complete before any kernel reads it.
// Rejects handles whose last SETUP failed.
void sync_in(msp_handle* h) {
  if (!h->valid) throw std::pair<int, std::string>(MSP_EINVAL, "handle unusable: its last SETUP failed");
  if (!h->ev_in) CK(cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming));
  CK(cudaEventRecord(h->ev_in, h->caller));
  CK(cudaStreamWaitEvent(h->s, h->ev_in, 0));
}

// copy a caller vector (host or device, natural order) into internal order (dst)
void to_internal(msp_handle* h, const double* src, double* dst, size_t count_cells, int b) {
  const size_t N = count_cells * b;
  if (is_device_ptr(src)) {
    CK(cudaMemcpyAsync(h->io, src, sizeof(double) * N, cudaMemcpyDeviceToDevice, h->s));
  } else {
    CK(cudaMemcpyAsync(h->io, src, sizeof(double) * N, cudaMemcpyHostToDevice, h->s));
  }
  switch (b) {
#define CASE(BV) case BV: klaunch(h->s, h->pdl, perm_gather_kernel<BV>, nblk(N, 256), 256, h->n, h->d_order, h->io, dst); ++h->nlaunch; break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
  }
}
void from_internal(msp_handle* h, const double* src, double* dst, int b) {
  const size_t N = (size_t)h->n * b;
  switch (b) {
#define CASE(BV) case BV: klaunch(h->s, h->pdl, perm_scatter_kernel<BV>, nblk(N, 256), 256, h->n, h->d_order, src, h->io); ++h->nlaunch; break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
  }
  if (is_device_ptr(dst)) CK(cudaMemcpyAsync(dst, h->io, sizeof(double) * N, cudaMemcpyDeviceToDevice, h->s));
  else CK(cudaMemcpyAsync(dst, h->io, sizeof(double) * N, cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
}

}  // namespace

// ============================================================================ C-ABI
extern "C" {

void msp_config_default(msp_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->coarsest_max_dof = 10000;
  c->max_levels = 20;
  c->pre_sweeps = 1;
  c->post_sweeps = 1;
  c->pair_passes = 2;
  c->decoupling = 2;
  c->bilu_order = 1;
  c->stages = 2;
  c->orth = 2;
  c->use_graphs = 1;
  c->use_coop = 0;
  c->smoother = 0;
  c->gs_chunk = 32;
}

const char* msp_last_error(const msp_handle* h) { return h ? h->err.c_str() : g_last_error.c_str(); }

msp_status msp_setup(const msp_bsr* A, int nc, const msp_config* cfg, void* cuda_stream, msp_handle** out) {
  if (!out) return fail(nullptr, MSP_EINVAL, "msp_setup: out is NULL");
  *out = nullptr;
  msp_config c;
  msp_config_default(&c);
  if (cfg) c = *cfg;
  if (c.stages != 2 && c.stages != 3) return fail(nullptr, MSP_EINVAL, "msp_setup: stages must be 2 (P,R) or 3 (N,P,R)");
  if (c.pre_sweeps < 1 || c.post_sweeps < 0 || c.pair_passes < 1 || c.coarsest_max_dof < 1 ||
      c.smoother < 0 || c.smoother > 2 || c.gs_chunk < 1 || c.orth < 0 || c.orth > 2 || c.coarse_mode < 0 ||
      c.coarse_mode > 1 || c.bilu_local != 0)
    return fail(nullptr, MSP_EINVAL, "msp_setup: invalid config");
  if (c.use_coop != 0) return fail(nullptr, MSP_EINVAL, "msp_setup: use_coop (cooperative V-cycle) was removed: measured slower than graph replay");
  std::unique_ptr<msp_handle> h(new msp_handle);
  h->cfg = c;
  if (const char* e = std::getenv("MSP_SELL_TPB")) h->sell_tpb = std::atoi(e);
  if (const char* e = std::getenv("MSP_HOST_SETUP")) h->setup_on_gpu = std::atoi(e) == 0;
  if (const char* e = std::getenv("MSP_BILU_META")) h->bilu_meta = std::atoi(e);
  if (const char* e = std::getenv("MSP_A8_ELL")) h->a8_ell = std::atoi(e);
  if (const char* e = std::getenv("MSP_CYCLE_GRAPH")) h->cycle_graphs = std::atoi(e) != 0;
  if (const char* e = std::getenv("MSP_SPEC_STEPS")) h->spec_steps = std::atoi(e);
  if (const char* e = std::getenv("MSP_PDL")) h->pdl = std::atoi(e) != 0;
  h->prm = params_of(&c);
  msp::BlockMat M;
  std::string err;
  msp_status st = read_bsr(A, nc, M, err, true);
  if (st) return fail(nullptr, st, err);
  st = guarded(h.get(), [&]() -> msp_status {
    CK(cudaGetDevice(&h->device));
    if (A->device >= 0) { CK(cudaSetDevice(A->device)); h->device = A->device; }
    CK(cudaStreamCreateWithFlags(&h->s, cudaStreamNonBlocking));
    CK(cudaEventCreate(&h->ev0));
    CK(cudaEventCreate(&h->ev1));
    h->caller = (cudaStream_t)cuda_stream;
    {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      CK(cudaEventRecord(e, h->caller));
      CK(cudaStreamWaitEvent(h->s, e, 0));
      cudaEventDestroy(e);
    }
    do_setup(h.get(), M);
    return MSP_OK;
  });
  if (st) {
    g_last_error = h->err;
    h->free_all();
    return st;
  }
  *out = h.release();
  return MSP_OK;
}

msp_status msp_set_stream(msp_handle* h, void* cuda_stream) {
  if (!h) return fail(nullptr, MSP_EINVAL, "msp_set_stream: NULL handle");
  h->caller = (cudaStream_t)cuda_stream;
  return MSP_OK;
}

msp_status msp_update(msp_handle* h, const msp_bsr* A_new, int iota, int last_iterations, int mu,
                      int* did_setup) {
  if (!h) return fail(nullptr, MSP_EINVAL, "msp_update: NULL handle");
  if (!A_new || A_new->block != h->b || !A_new->row_ptr || !A_new->col_idx || !A_new->values)
    return fail(h, MSP_EINVAL, "msp_update: invalid matrix");
  // Remark 2: the preconditioner must be regenerated when the size changed.  Sizes and
  // patterns are compared GLOBALLY (the caller passes the global matrix on every rank of
  // a distributed handle, whose h->n is the owned-cell count)
  const int64_t n_glob = (int64_t)h->nat_rp.size() - 1;
  bool same = h->valid && (A_new->n_cells == n_glob);
  if (same) {
    std::vector<int32_t> rp(n_glob + 1);
    if (A_new->device >= 0) {
      if (cudaMemcpy(rp.data(), A_new->row_ptr, sizeof(int32_t) * (n_glob + 1), cudaMemcpyDeviceToHost) != cudaSuccess)
        return fail(h, MSP_ECUDA, "msp_update: row_ptr copy failed");
    } else {
      std::memcpy(rp.data(), A_new->row_ptr, sizeof(int32_t) * (n_glob + 1));
    }
    same = (rp == h->nat_rp);
    if (same) {
      std::vector<int32_t> ci(h->nat_ci.size());
      if (A_new->device >= 0) {
        if (cudaMemcpy(ci.data(), A_new->col_idx, sizeof(int32_t) * ci.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
          return fail(h, MSP_ECUDA, "msp_update: col_idx copy failed");
      } else {
        std::memcpy(ci.data(), A_new->col_idx, sizeof(int32_t) * ci.size());
      }
      same = (ci == h->nat_ci);
    }
  }
  // ASMSP rule: rebuild iff iota == 1, It^(iota-1) > mu, or size changed
  const bool rebuild = (iota <= 1) || !same || (last_iterations > mu);
  if (did_setup) *did_setup = rebuild ? 1 : 0;
  if (rebuild) {
    msp::BlockMat M;
    std::string err;
    msp_status st = read_bsr(A_new, h->nc, M, err, true);
    if (st) return fail(h, st, err);
    return guarded(h, [&]() -> msp_status {
      do_setup(h, M);
      return MSP_OK;
    });
  }
  // reuse: keep W, hierarchy and BILU factors; refresh A (SpMV, Alg. 1 residuals) on the GPU
  return guarded(h, [&]() -> msp_status {
    sync_in(h);
    const int bb = h->b * h->b;
    const size_t nv = (size_t)h->nnzb * bb;                   // local entries to refresh
    const size_t nglob = h->nat_ci.size() * (size_t)bb;        // caller's (global) values
    const double* nat = A_new->values;
    if (A_new->device < 0) {
      if (!h->stage) h->stage = h->dalloc<double>(nglob);
      h2d_large(h->s, h->stage, A_new->values, sizeof(double) * nglob);
      nat = h->stage;
    }
    switch (h->b) {
#define CASE(BV) case BV: klaunch(h->s, h->pdl, refresh_values_kernel<BV>, nblk(nv, 256), 256, (int64_t)h->nnzb, \
                                  h->d_src, nat, h->Aval, h->Pcol); break;
      CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
    }
    fill_pell(h);
    ++h->nlaunch;
    CK(cudaStreamSynchronize(h->s));
    h->st.reuse_calls++;
    return MSP_OK;
  });
}

msp_status msp_solve(msp_handle* h, const double* b, double* x, double tol, int restart, int maxit,
                     int* iterations, double* final_rel_res, double* resid_hist, int hist_cap,
                     int* hist_len) {
  if (!h || !b || !x || restart < 1 || restart > kMaxV - 2 || maxit < 0)
    return fail(h, MSP_EINVAL, "msp_solve: invalid arguments (1 <= restart <= 30)");
  int it_dummy = 0;
  double fr_dummy = 0.0;
  if (!iterations) iterations = &it_dummy;
  if (!final_rel_res) final_rel_res = &fr_dummy;
  return guarded(h, [&]() -> msp_status {
    sync_in(h);
    CK(cudaEventRecord(h->ev0, h->s));
    to_internal(h, b, h->bin, h->n, h->b);
    to_internal(h, x, h->xin, h->n, h->b);
    msp_status st = gmres(h, tol, restart, maxit, iterations, final_rel_res, resid_hist, hist_cap, hist_len);
    from_internal(h, h->xin, x, h->b);
    CK(cudaEventRecord(h->ev1, h->s));
    CK(cudaEventSynchronize(h->ev1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    h->st.solve_seconds += ms * 1e-3;
    return st;
  });
}

msp_status msp_apply(msp_handle* h, const double* g, double* w) {
  if (!h || !g || !w) return fail(h, MSP_EINVAL, "msp_apply: NULL argument");
  return guarded(h, [&]() -> msp_status {
    sync_in(h);
    to_internal(h, g, h->bin, h->n, h->b);
    msp_apply_dev(h, h->bin, h->z);
    from_internal(h, h->z, w, h->b);
    return MSP_OK;
  });
}

msp_status msp_spmv(msp_handle* h, const double* x, double* y) {
  if (!h || !x || !y) return fail(h, MSP_EINVAL, "msp_spmv: NULL argument");
  return guarded(h, [&]() -> msp_status {
    sync_in(h);
    launch_spmv(h, 0, x, nullptr, y);
    CK(cudaStreamSynchronize(h->s));
    return MSP_OK;
  });
}

msp_status msp_pgs_sweep(msp_handle* h, int level, const double* b, double* x, int ascending) {
  if (!h || level < 0 || level >= (int)h->lv.size()) return fail(h, MSP_EINVAL, "msp_pgs_sweep: bad level");
  return guarded(h, [&]() -> msp_status {
    sync_in(h);
    DevLevel& L = h->lv[level];
    klaunch(h->s, h->pdl, scalar_perm_kernel, nblk(L.n, 256), 256, L.n, L.perm, b, L.b, 1); ++h->nlaunch;
    klaunch(h->s, h->pdl, scalar_perm_kernel, nblk(L.n, 256), 256, L.n, L.perm, x, L.x, 1); ++h->nlaunch;
    pgs_sweep(h, L, ascending != 0, false);
    klaunch(h->s, h->pdl, scalar_perm_kernel, nblk(L.n, 256), 256, L.n, L.perm, L.x, x, 0); ++h->nlaunch;
    CK(cudaStreamSynchronize(h->s));
    return MSP_OK;
  });
}

msp_status msp_bilu_factors(msp_handle* h, double* F_out) {
  if (!h || !F_out) return fail(h, MSP_EINVAL, "msp_bilu_factors: NULL argument");
  if (h->comm) return fail(h, MSP_EINVAL, "msp_bilu_factors: single-GPU handles only");
  return guarded(h, [&]() -> msp_status {
    const int b = h->b, bb = b * b;
    std::vector<double> cm((size_t)h->nnzb * bb);
    CK(cudaStreamSynchronize(h->s));
    CK(cudaMemcpy(cm.data(), h->Fval, sizeof(double) * cm.size(), cudaMemcpyDeviceToHost));
    for (int64_t e = 0; e < h->nnzb; ++e) {
      double* dst = F_out + (size_t)h->src_entry[e] * bb;
      for (int r = 0; r < b; ++r)
        for (int c = 0; c < b; ++c) dst[r * b + c] = cm[(size_t)e * bb + c * b + r];
    }
    return MSP_OK;
  });
}

msp_status msp_vcycle(msp_handle* h, const double* r, double* x) {
  if (!h || !r || !x) return fail(h, MSP_EINVAL, "msp_vcycle: NULL argument");
  return guarded(h, [&]() -> msp_status {
    sync_in(h);
    if (h->lv.empty()) {
      CK(cudaMemcpyAsync(h->bL, r, sizeof(double) * h->nL, cudaMemcpyDeviceToDevice, h->s));
      vcycle_any(h);
      CK(cudaMemcpyAsync(x, h->xL, sizeof(double) * h->nL, cudaMemcpyDeviceToDevice, h->s));
    } else {
      DevLevel& L = h->lv[0];
      klaunch(h->s, h->pdl, scalar_perm_kernel, nblk(L.n, 256), 256, L.n, L.perm, r, L.b, 1); ++h->nlaunch;
      vcycle_any(h);
      klaunch(h->s, h->pdl, scalar_perm_kernel, nblk(L.n, 256), 256, L.n, L.perm, L.x, x, 0); ++h->nlaunch;
    }
    CK(cudaStreamSynchronize(h->s));
    return MSP_OK;
  });
}

msp_status msp_bilu_apply(msp_handle* h, const double* r, double* x) {
  if (!h || !r || !x) return fail(h, MSP_EINVAL, "msp_bilu_apply: NULL argument");
  return guarded(h, [&]() -> msp_status {
    sync_in(h);
    to_internal(h, r, h->r, h->n, h->b);
    CK(cudaMemsetAsync(h->wp, 0, sizeof(double) * h->n, h->s));
    launch_bilu(h, h->r, h->wp, h->z);
    from_internal(h, h->z, x, h->b);
    return MSP_OK;
  });
}

// ---- per-kernel entry points (parity tests of single hot-path steps) ----
msp_status msp_restrict_pressure(msp_handle* h, const double* g, double* rp) {
  if (!h || !g || !rp || h->comm) return fail(h, MSP_EINVAL, "msp_restrict_pressure: bad arguments");
  return guarded(h, [&]() -> msp_status {
    sync_in(h);
    to_internal(h, g, h->bin, h->n, h->b);
    launch_restrict_pressure(h, h->bin, level0_b(h), false);
    if (h->lv.empty()) {
      CK(cudaMemcpyAsync(rp, h->bL, sizeof(double) * h->n, cudaMemcpyDeviceToDevice, h->s));
    } else {
      DevLevel& L = h->lv[0];
      klaunch(h->s, h->pdl, scalar_perm_kernel, nblk(L.n, 256), 256, L.n, L.perm, (const double*)L.b, rp, 0);
      ++h->nlaunch;
    }
    CK(cudaStreamSynchronize(h->s));
    return MSP_OK;
  });
}

msp_status msp_residual_restrict(msp_handle* h, int level, const double* b, const double* x, double* bc) {
  if (!h || !b || !x || !bc || level < 0 || level >= (int)h->lv.size() || (h->comm && level == 0))
    return fail(h, MSP_EINVAL, "msp_residual_restrict: bad level/arguments");
  return guarded(h, [&]() -> msp_status {
    sync_in(h);
    DevLevel& L = h->lv[level];
    const bool last = (level + 1 == (int)h->lv.size());
    double* bn = last ? h->bL : h->lv[level + 1].b;
    const int nn = last ? h->nL : h->lv[level + 1].n;
    klaunch(h->s, h->pdl, scalar_perm_kernel, nblk(L.n, 256), 256, L.n, L.perm, b, L.b, 1); ++h->nlaunch;
    klaunch(h->s, h->pdl, scalar_perm_kernel, nblk(L.n, 256), 256, L.n, L.perm, x, L.x, 1); ++h->nlaunch;
    sell_rows_any<false, true>(h, L, 0, L.nslices);                     // r = b - A x, every row
    klaunch(h->s, h->pdl, restrict_kernel, nblk(nn, 256), 256, nn, L.pt_ptr, L.pt_idx, (const double*)L.r, bn,
            (double*)nullptr, (const double*)nullptr, 0);
    ++h->nlaunch;
    if (last) {
      CK(cudaMemcpyAsync(bc, bn, sizeof(double) * nn, cudaMemcpyDeviceToDevice, h->s));
    } else {
      klaunch(h->s, h->pdl, scalar_perm_kernel, nblk(nn, 256), 256, nn, h->lv[level + 1].perm, (const double*)bn, bc, 0);
      ++h->nlaunch;
    }
    CK(cudaStreamSynchronize(h->s));
    return MSP_OK;
  });
}

msp_status msp_prolong(msp_handle* h, int level, const double* e, double* x) {
  if (!h || !e || !x || level < 0 || level >= (int)h->lv.size() || (h->comm && level == 0))
    return fail(h, MSP_EINVAL, "msp_prolong: bad level/arguments");
  return guarded(h, [&]() -> msp_status {
    sync_in(h);
    DevLevel& L = h->lv[level];
    const bool last = (level + 1 == (int)h->lv.size());
    double* xn = last ? h->xL : h->lv[level + 1].x;
    const int nn = last ? h->nL : h->lv[level + 1].n;
    if (last) CK(cudaMemcpyAsync(xn, e, sizeof(double) * nn, cudaMemcpyDeviceToDevice, h->s));
    else { klaunch(h->s, h->pdl, scalar_perm_kernel, nblk(nn, 256), 256, nn, h->lv[level + 1].perm, e, xn, 1); ++h->nlaunch; }
    klaunch(h->s, h->pdl, scalar_perm_kernel, nblk(L.n, 256), 256, L.n, L.perm, (const double*)x, L.x, 1); ++h->nlaunch;
    klaunch(h->s, h->pdl, prolong_kernel, nblk(L.n, 256), 256, L.n, L.agg, (const double*)xn, L.x, HaloPack{}); ++h->nlaunch;
    klaunch(h->s, h->pdl, scalar_perm_kernel, nblk(L.n, 256), 256, L.n, L.perm, (const double*)L.x, x, 0); ++h->nlaunch;
    CK(cudaStreamSynchronize(h->s));
    return MSP_OK;
  });
}

msp_status msp_pcol_residual(msp_handle* h, const double* g, const double* xp, double* r) {
  if (!h || !g || !xp || !r || h->comm) return fail(h, MSP_EINVAL, "msp_pcol_residual: bad arguments");
  return guarded(h, [&]() -> msp_status {
    sync_in(h);
    to_internal(h, g, h->bin, h->n, h->b);
    klaunch(h->s, h->pdl, scalar_perm_kernel, nblk(h->n, 256), 256, h->n, h->d_order, xp, h->wp, 0);   // wp[p] = xp[order[p]]
    ++h->nlaunch;
    launch_spmv(h, 2, h->wp, h->bin, h->r);
    from_internal(h, h->r, r, h->b);
    return MSP_OK;
  });
}

msp_status msp_bilu_forward(msp_handle* h, const double* r, double* y) {
  if (!h || !r || !y || h->comm) return fail(h, MSP_EINVAL, "msp_bilu_forward: bad arguments");
  return guarded(h, [&]() -> msp_status {
    sync_in(h);
    to_internal(h, r, h->r, h->n, h->b);
    launch_bilu(h, h->r, h->wp, h->z, false, 1);
    from_internal(h, h->r, y, h->b);
    return MSP_OK;
  });
}

msp_status msp_bilu_backward(msp_handle* h, const double* y, double* x) {
  if (!h || !y || !x || h->comm) return fail(h, MSP_EINVAL, "msp_bilu_backward: bad arguments");
  return guarded(h, [&]() -> msp_status {
    sync_in(h);
    to_internal(h, y, h->r, h->n, h->b);
    CK(cudaMemsetAsync(h->wp, 0, sizeof(double) * h->n, h->s));
    launch_bilu(h, h->r, h->wp, h->z, false, 2);
    from_internal(h, h->z, x, h->b);
    return MSP_OK;
  });
}

msp_status msp_multidot(msp_handle* h, int k, const double* V, const double* w, double* out) {
  if (!h || !V || !w || !out || k < 1 || k > kMaxV || h->comm) return fail(h, MSP_EINVAL, "msp_multidot: bad arguments");
  return guarded(h, [&]() -> msp_status {
    sync_in(h);
    cgs_dot(h, k, V, w, h->dh1, nullptr, nullptr, -1);                  // a10 pass-1 kernel
    CK(cudaMemcpyAsync(h->hpin, h->dh1, sizeof(double) * k, cudaMemcpyDeviceToHost, h->s));
    CK(cudaStreamSynchronize(h->s));
    std::memcpy(out, h->hpin, sizeof(double) * k);
    return MSP_OK;
  });
}

msp_status msp_bilu_set_factors(msp_handle* h, const double* F) {
  if (!h || !F || h->comm) return fail(h, MSP_EINVAL, "msp_bilu_set_factors: bad arguments");
  return guarded(h, [&]() -> msp_status {
    const int b = h->b, bb = b * b;
    const size_t nv = (size_t)h->nnzb * bb;
    if (!h->ftmp) h->ftmp = h->dalloc<double>(nv);
    CK(cudaMemcpyAsync(h->stage, F, sizeof(double) * nv, cudaMemcpyHostToDevice, h->s));
    switch (b) {
#define CASE(BV) case BV: \
      klaunch(h->s, false, gather_blocks_kernel<BV>, nblk(nv, 256), 256, (int64_t)h->nnzb, (const int*)h->d_src, \
              (const double*)h->stage, h->ftmp); \
      klaunch(h->s, false, transpose_blocks_kernel<BV>, nblk(nv, 256), 256, (int64_t)h->nnzb, (const double*)h->ftmp, \
              h->Fval); \
      break;
      CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
    }
    h->nlaunch += 2;
    CK(cudaStreamSynchronize(h->s));
    return MSP_OK;
  });
}

msp_status msp_get_s1(const msp_handle* h, double* W, double* App, int32_t* on_gpu) {
  if (!h || !W || !App || h->W_nat.empty()) return MSP_EINVAL;
  std::memcpy(W, h->W_nat.data(), sizeof(double) * h->W_nat.size());
  std::memcpy(App, h->App_nat.data(), sizeof(double) * h->App_nat.size());
  if (on_gpu) *on_gpu = h->gpu_s1 ? 1 : 0;
  return MSP_OK;
}

msp_status msp_get_order(const msp_handle* h, int32_t* order) {
  if (!h || !order) return MSP_EINVAL;
  std::memcpy(order, h->order.data(), sizeof(int32_t) * h->n);
  return MSP_OK;
}

msp_status msp_get_stats(const msp_handle* h, msp_stats* out) {
  if (!h || !out) return MSP_EINVAL;
  *out = h->st;
  for (size_t l = 0; l < h->level_n.size() && l < 24; ++l) {
    out->level_n[l] = h->level_n[l];
    out->level_nnz[l] = h->level_nnz[l];
    out->level_colors[l] = h->level_colors[l];
  }
  out->device_bytes = h->bytes;
  out->kernels_per_iter = h->kernels_per_step;
  out->fused_a8 = 0;
  return MSP_OK;
}

void msp_destroy(msp_handle* h) {
  if (!h) return;
  h->free_all();
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->ev_in) cudaEventDestroy(h->ev_in);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  for (auto e : h->ev_step) if (e) cudaEventDestroy(e);
  if (h->s2) cudaStreamDestroy(h->s2);
  if (h->cs) cusolverDnDestroy(h->cs);
  if (h->s) cudaStreamDestroy(h->s);
  delete h;
}

int64_t msp_kernel_launches(const msp_handle* h) { return h ? h->nlaunch : 0; }

msp_status msp_time_kernel(msp_handle* h, int kind, int reps, double* ms_per_launch,
                           double* bytes_per_launch) {
  if (!h || reps < 1 || !ms_per_launch || !bytes_per_launch) return fail(h, MSP_EINVAL, "msp_time_kernel: bad args");
  const bool flush_l2 = (kind & 0x100) == 0;
  kind &= 0xff;
  if (h->comm && kind != 0 && kind != 2 && kind != 4)
    return fail(h, MSP_EINVAL, "msp_time_kernel: distributed handles time only rank-local kernels (0, 2, 4)");
  if ((kind == 1) && h->lv.empty()) return fail(h, MSP_EINVAL, "msp_time_kernel: no AMG level 0");
  return guarded(h, [&]() -> msp_status {
    const size_t kFlush = (size_t)256 << 20;
    if (!h->flush) {
      h->flush = h->dalloc<double>(kFlush / sizeof(double) + 1);
      CK(cudaMemsetAsync(h->flush, 0, kFlush + sizeof(double), h->s));
      CK(cudaStreamSynchronize(h->s));
    }
    ensure_basis(h, 30);
    const size_t N = h->N;
    const double n = h->n, b = h->b, nnzb = (double)h->nnzb;
    double bytes = 0.0;
    // deterministic non-trivial inputs
    CK(cudaMemsetAsync(h->r, 0, sizeof(double) * N, h->s));
    klaunch(h->s, h->pdl, scale_kernel, kRedBlocks, kRedThreads, N, h->V, h->hcol, h->z); ++h->nlaunch;
    std::function<void()> fn;
    switch (kind) {
      case 0:
        fn = [&]() { launch_spmv(h, 0, h->xin, nullptr, h->u); };
        bytes = nnzb * (8 * b * b + 4) + 4 * (n + 1) + 2 * 8 * (double)N;
        break;
      case 1: {
        DevLevel& L = h->lv[0];
        fn = [&]() { pgs_sweep(h, L, false, false); };
        const double nnz_off = (double)h->level_nnz[0] - L.n;
        bytes = 12 * nnz_off + 32.0 * L.n;
        break;
      }
      case 2:
        fn = [&]() { launch_spmv(h, 2, h->wp, h->bin, h->u); };
        bytes = nnzb * (8 * b + 4) + 4 * (n + 1) + 8 * n + 2 * 8 * (double)N;
        break;
      case 3:                                    // a9 as the solve runs it
        fn = [&]() { launch_bilu(h, h->r, h->wp, h->z); };
        bytes = (nnzb - n) * (8 * b * b + 4) + 8 * b * b * n + 8 * (n + 1) + 5 * 8 * (double)N;
        break;
      case 4:                                    // CGS2 pass A over 16 basis vectors
        fn = [&]() { cgs_dot(h, 16, h->V, h->u, h->dh1, nullptr, nullptr, -1); };
        bytes = 17.0 * 8 * (double)N;
        break;
      case 5:
        fn = [&]() { vcycle(h, (int)h->lv.size()); };
        bytes = h->coarse_diag ? 24.0 * h->nL : 8.0 * (double)h->nL * h->nL;
        break;
      case 6:
        fn = [&]() { msp_apply_dev(h, h->bin, h->z); };
        bytes = 0.0;
        break;
      case 7:
        fn = [&]() { vcycle_any(h); };
        bytes = 0.0;
        break;
      case 8:
        fn = [&]() { launch_bilu(h, h->r, h->wp, h->z); };
        bytes = 0.0;
        break;
      case 9:
        fn = [&]() { arnoldi_step(h, 15); };
        bytes = 0.0;
        break;
      case 10:                                   // orthogonalisation of step j=15 alone
        if (h->prm.orth == 2) {
          fn = [&]() { dcgs2(h, 15); };
          // pass 1 (16+1 vectors) + pass 2 (15 + 2 read, 2 written)
          bytes = 36.0 * 8 * (double)N;
        } else {
          fn = [&]() { cgs2(h, 16, h->V + (size_t)16 * N); };
          // pass A (16+1 vectors) + fused pass B (16 + 2) + pass C (16 + 2) + scale (2)
          bytes = 55.0 * 8 * (double)N;
        }
        break;
      case 11:
        fn = [&]() { arnoldi_step(h, 25); };
        bytes = 0.0;
        break;
      case 12:
        if (h->prm.orth == 2) {
          fn = [&]() { dcgs2(h, 25); };
          bytes = 56.0 * 8 * (double)N;        // pass 1 (25+2 vectors) + pass 2 (25 + 2 read, 2 written)
        } else {
          fn = [&]() { cgs2(h, 26, h->V + (size_t)26 * N); };
          bytes = 0.0;
        }
        break;
      case 13:                                   // a9 followed by the Arnoldi SpMV
        fn = [&]() { launch_bilu(h, h->r, h->wp, h->z); launch_spmv(h, 0, h->z, nullptr, h->u); };
        bytes = 0.0;
        break;
      case 14:                                   // MSP application followed by the SpMV
        fn = [&]() { msp_apply_dev(h, h->bin, h->z); launch_spmv(h, 0, h->z, nullptr, h->u); };
        bytes = 0.0;
        break;
      case 15:                                   // SpMV + orthogonalisation of step 15
        fn = [&]() {
          launch_spmv(h, 0, h->z, nullptr, h->V + (size_t)16 * N);
          if (h->prm.orth == 2) dcgs2(h, 15); else cgs2(h, 16, h->V + (size_t)16 * N);
        };
        bytes = 0.0;
        break;
      default:
        if (kind >= 16 && kind <= 16 + (int)h->lv.size()) {   // V-cycle from level kind-16 down
          const int l = kind - 16;
          fn = [h, l]() { vcycle(h, l); };
          bytes = 0.0;
          break;
        }
        throw std::pair<int, std::string>(MSP_EINVAL, "msp_time_kernel: unknown kind");
    }
    // replay the piece as a CUDA graph, exactly as inside the Arnoldi-step graphs
    cudaGraph_t graph;
    cudaGraphExec_t gexec;
    const int64_t before = h->nlaunch;
    CK(cudaStreamBeginCapture(h->s, cudaStreamCaptureModeThreadLocal));
    fn();
    CK(cudaStreamEndCapture(h->s, &graph));
    h->nlaunch = before;
    CK(cudaGraphInstantiate(&gexec, graph, 0));
    cudaGraphDestroy(graph);
    double total = 0.0;
    for (int r = 0; r < reps + 1; ++r) {
      // flush L2 by READING 256 MB (2x L2): the cache is left holding clean lines, so the
      // timed kernel pays no write-back of unrelated dirty data
      if (flush_l2)
        klaunch(h->s, false, flush_read_kernel, 4 * 148, 512, kFlush / sizeof(double), (const double*)h->flush,
                h->flush + kFlush / sizeof(double));
      CK(cudaEventRecord(h->ev0, h->s));
      CK(cudaGraphLaunch(gexec, h->s));
      CK(cudaEventRecord(h->ev1, h->s));
      CK(cudaEventSynchronize(h->ev1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
      if (r > 0) total += ms;                  // first replay = warm-up
    }
    cudaGraphExecDestroy(gexec);
    *ms_per_launch = total / reps;
    *bytes_per_launch = bytes;
    return MSP_OK;
  });
}

// ----------------------------------------------------------- distributed (§8(e))
static msp_status setup_dist_common(const msp_bsr* A, int nc, const msp_config* cfg, const int32_t* owner,
                                    std::unique_ptr<msp::Comm> comm, int rank, int nranks, void* cuda_stream,
                                    msp_handle** out) {
  if (!out) return fail(nullptr, MSP_EINVAL, "msp_setup_dist: out is NULL");
  *out = nullptr;
  msp_config c;
  msp_config_default(&c);
  if (cfg) c = *cfg;
  if (c.stages != 2 || c.pre_sweeps != 1 || c.post_sweeps != 1 || c.bilu_order != 1 || c.orth == 1 ||
      c.smoother != 0 || c.coarse_mode < 0 || c.coarse_mode > 1 || c.bilu_local < 0 || c.bilu_local > 1 ||
      c.dist_levels < 0)
    return fail(nullptr, MSP_EINVAL,
                "msp_setup_dist: supports stages=2, 1 pre/post sweep, ABMC order, CGS2/DCGS2, PGS-MC, coarse_mode 0/1");
  // NCCL steps are replayed as CUDA graphs (halo send/recv groups and allreduces are
  // captured with the kernels); the loopback backend synchronises host threads: direct
  const char* ng = std::getenv("MSP_DIST_NOGRAPH");
  c.use_graphs = (c.use_graphs && comm && comm->capturable() && !(ng && std::atoi(ng))) ? 1 : 0;
  c.use_coop = 0;
  std::unique_ptr<msp_handle> h(new msp_handle);
  h->cfg = c;
  h->prm = params_of(&c);
  msp::BlockMat M;
  std::string err;
  msp_status st = read_bsr(A, nc, M, err, true);
  if (st) return fail(nullptr, st, err);
  h->owner_in.resize(M.n);
  for (int32_t i = 0; i < M.n; ++i) {
    const int32_t o = owner ? owner[i] : (int32_t)(((int64_t)i * nranks) / M.n);
    if (o < 0 || o >= nranks) return fail(nullptr, MSP_EINVAL, "msp_setup_dist: owner out of range");
    h->owner_in[i] = o;
  }
  h->comm = std::move(comm);
  h->rank = rank;
  h->nranks = nranks;
  st = guarded(h.get(), [&]() -> msp_status {
    CK(cudaGetDevice(&h->device));
    CK(cudaStreamCreateWithFlags(&h->s, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&h->s2, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
    if (const char* e = std::getenv("MSP_DIST_OVERLAP")) h->overlap_halo = std::atoi(e) != 0;
    if (const char* e = std::getenv("MSP_DIST_SETUP_ALL")) h->setup_rank0 = std::atoi(e) == 0;
    if (const char* e = std::getenv("MSP_DIST_FUSE_PACK")) h->fuse_halo = std::atoi(e) != 0;
    CK(cudaEventCreate(&h->ev0));
    CK(cudaEventCreate(&h->ev1));
    h->caller = (cudaStream_t)cuda_stream;
    {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      CK(cudaEventRecord(e, h->caller));
      CK(cudaStreamWaitEvent(h->s, e, 0));
      cudaEventDestroy(e);
    }
    do_setup(h.get(), M);
    return MSP_OK;
  });
  if (st) {
    g_last_error = h->err;
    h->free_all();
    return st;
  }
  *out = h.release();
  return MSP_OK;
}

msp_status msp_nccl_unique_id(void* id128) {
  if (!id128) return MSP_EINVAL;
  return msp::nccl_unique_id(id128) ? fail(nullptr, MSP_ENCCL, "ncclGetUniqueId failed") : MSP_OK;
}

msp_status msp_setup_dist(const msp_bsr* A, int nc, const msp_config* cfg, const int32_t* owner,
                          const void* nccl_unique_id, int rank, int nranks, void* cuda_stream, msp_handle** out) {
  if (!nccl_unique_id || nranks < 1 || rank < 0 || rank >= nranks) return fail(nullptr, MSP_EINVAL, "msp_setup_dist: bad rank/id");
  int e = 0;
  auto comm = msp::make_nccl_comm(nccl_unique_id, rank, nranks, &e);
  if (!comm) return fail(nullptr, MSP_ENCCL, "ncclCommInitRank failed: " + std::to_string(e));
  return setup_dist_common(A, nc, cfg, owner, std::move(comm), rank, nranks, cuda_stream, out);
}

int32_t msp_dist_n_owned(const msp_handle* h) { return h ? h->n : 0; }

msp_status msp_dist_owned_cells(const msp_handle* h, int32_t* cells) {
  if (!h || !cells) return MSP_EINVAL;
  if (!h->comm) {
    for (int32_t i = 0; i < h->n; ++i) cells[i] = i;
    return MSP_OK;
  }
  std::memcpy(cells, h->owned_cells.data(), sizeof(int32_t) * h->owned_cells.size());
  return MSP_OK;
}

msp_status msp_loopback_solve(const msp_bsr* A, int nc, const msp_config* cfg, const int32_t* owner, int nranks,
                              const double* b, double* x, double tol, int restart, int maxit, int* iterations,
                              double* final_rel_res, int32_t* rank_info) {
  if (!A || !b || !x || nranks < 1) return fail(nullptr, MSP_EINVAL, "msp_loopback_solve: bad arguments");
  msp_config c;
  msp_config_default(&c);
  if (cfg) c = *cfg;
  c.alloc = nullptr;                 // worker threads allocate with cudaMalloc
  c.free_fn = nullptr;
  auto grp = msp::make_loopback_group(nranks);
  int dev = 0;
  cudaGetDevice(&dev);
  const int b_ = A->block;
  std::vector<msp_status> st(nranks, MSP_OK), sst(nranks, MSP_OK);
  std::vector<int> its(nranks, 0);
  std::vector<double> rel(nranks, 0.0);
  std::vector<std::string> errs(nranks);
  std::vector<int> fail_flag(nranks, 0);
  std::vector<std::thread> th;
  for (int r = 0; r < nranks; ++r)
    th.emplace_back([&, r] {
      cudaSetDevice(dev);
      msp_handle* h = nullptr;
      st[r] = setup_dist_common(A, nc, &c, owner, msp::make_loopback_comm(grp, r), r, nranks, nullptr, &h);
      if (st[r]) { errs[r] = g_last_error; fail_flag[r] = 1; }
      msp::loopback_barrier(*grp);
      bool any = false;
      for (int q = 0; q < nranks; ++q) any |= fail_flag[q] != 0;
      if (!any) {
        const int32_t no = h->n;
        std::vector<double> bl((size_t)no * b_), xl((size_t)no * b_);
        for (int32_t k = 0; k < no; ++k)
          for (int q = 0; q < b_; ++q) {
            bl[(size_t)k * b_ + q] = b[(size_t)h->owned_cells[k] * b_ + q];
            xl[(size_t)k * b_ + q] = x[(size_t)h->owned_cells[k] * b_ + q];
          }
        sst[r] = msp_solve(h, bl.data(), xl.data(), tol, restart, maxit, &its[r], &rel[r], nullptr, 0, nullptr);
        if (sst[r] != MSP_OK && sst[r] != MSP_ENOCONV) errs[r] = h->err;
        for (int32_t k = 0; k < no; ++k)
          for (int q = 0; q < b_; ++q) x[(size_t)h->owned_cells[k] * b_ + q] = xl[(size_t)k * b_ + q];
        if (rank_info) {
          rank_info[4 * r + 0] = h->n;
          rank_info[4 * r + 1] = h->n_ghost;
          rank_info[4 * r + 2] = h->lv.empty() ? 0 : h->lv[0].n;
          rank_info[4 * r + 3] = h->n0_ghost;
        }
      }
      if (h) msp_destroy(h);
    });
  for (auto& t : th) t.join();
  for (int r = 0; r < nranks; ++r) {
    if (st[r]) return fail(nullptr, st[r], "rank " + std::to_string(r) + ": " + errs[r]);
    if (sst[r] != MSP_OK && sst[r] != MSP_ENOCONV) return fail(nullptr, sst[r], "rank " + std::to_string(r) + ": " + errs[r]);
    if (its[r] != its[0]) return fail(nullptr, MSP_ECUDA, "loopback ranks disagree on the iteration count");
  }
  if (iterations) *iterations = its[0];
  if (final_rel_res) *final_rel_res = rel[0];
  return sst[0];
}

// ----------------------------------------------------------- host-setup introspection
struct msp_host_setup {
  msp::BlockMat M;                   // owns the matrix S.A points to
  msp::HostSetup S;
};

msp_status msp_host_setup_run(const msp_bsr* A, int nc, const msp_config* cfg, msp_host_setup** out) {
  if (!out) return MSP_EINVAL;
  *out = nullptr;
  std::unique_ptr<msp_host_setup> s(new msp_host_setup);
  std::string err;
  msp_status st = read_bsr(A, nc, s->M, err);
  if (st) return fail(nullptr, st, err);
  msp_config c;
  msp_config_default(&c);
  if (cfg) c = *cfg;
  msp::Params prm = params_of(&c);
  // MSP_HOST_SETUP_GPU=1: the GPU steps of NEXT-2 (S1, Galerkin) as msp_setup runs them,
  // for the bit-exact comparison with the host path (needs a GPU)
  const bool gpu = std::getenv("MSP_HOST_SETUP_GPU") && std::atoi(std::getenv("MSP_HOST_SETUP_GPU"));
  msp_status gst = MSP_OK;
  cudaStream_t stream = nullptr;
  if (gpu) {
    gst = guarded(nullptr, [&]() -> msp_status {
      CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
      gpu_setup_s1(stream, prm.decoupling, s->M, s->S);
      return MSP_OK;
    });
    if (gst) { if (stream) cudaStreamDestroy(stream); return gst; }
    prm.s1_given = true;
  }
  RapChain chain;
  chain.s = stream;
  if (gpu)
    prm.rap = [&chain](const msp::SpMat& Af, const std::vector<int32_t>& agg, int32_t na, msp::SpMat& C) {
      try {
        return gpu_rap(chain, Af, agg, na, C);
      } catch (...) {
        return 1;
      }
    };
  int rc = msp::run_host_setup(s->M, prm, s->S, err);
  chain.keep.clear();
  if (stream) cudaStreamDestroy(stream);
  if (rc) return fail(nullptr, (msp_status)rc, err);
  *out = s.release();
  return MSP_OK;
}

msp_status msp_host_setup_info(const msp_host_setup* s, int32_t* o) {
  if (!s || !o) return MSP_EINVAL;
  o[0] = (int32_t)s->S.lv.size();
  o[1] = s->S.Ac.n;
  o[2] = s->S.coarse_diag ? 1 : 0;
  o[3] = s->S.bilu_ncolor;
  return MSP_OK;
}

static const msp::SpMat* level_mat(const msp_host_setup* s, int l) {
  if (l < 0 || l > (int)s->S.lv.size()) return nullptr;
  return l < (int)s->S.lv.size() ? &s->S.lv[l].A : &s->S.Ac;
}

msp_status msp_host_setup_level_dims(const msp_host_setup* s, int l, int32_t* n, int64_t* nnz, int32_t* ncolors) {
  if (!s) return MSP_EINVAL;
  const msp::SpMat* A = level_mat(s, l);
  if (!A) return MSP_EINVAL;
  *n = A->n;
  *nnz = A->nnz();
  *ncolors = l < (int)s->S.lv.size() ? s->S.lv[l].ncolor : 0;
  return MSP_OK;
}

msp_status msp_host_setup_level_csr(const msp_host_setup* s, int l, int32_t* ptr, int32_t* col, double* val) {
  if (!s) return MSP_EINVAL;
  const msp::SpMat* A = level_mat(s, l);
  if (!A) return MSP_EINVAL;
  std::memcpy(ptr, A->rp.data(), sizeof(int32_t) * (A->n + 1));
  std::memcpy(col, A->ci.data(), sizeof(int32_t) * A->ci.size());
  std::memcpy(val, A->v.data(), sizeof(double) * A->v.size());
  return MSP_OK;
}

msp_status msp_host_setup_level_colors(const msp_host_setup* s, int l, int32_t* color) {
  if (!s || l < 0 || l >= (int)s->S.lv.size()) return MSP_EINVAL;
  std::memcpy(color, s->S.lv[l].color.data(), sizeof(int32_t) * s->S.lv[l].color.size());
  return MSP_OK;
}

msp_status msp_host_setup_level_agg(const msp_host_setup* s, int l, int32_t* agg) {
  if (!s || l < 0 || l >= (int)s->S.lv.size()) return MSP_EINVAL;
  std::memcpy(agg, s->S.lv[l].agg.data(), sizeof(int32_t) * s->S.lv[l].agg.size());
  return MSP_OK;
}

msp_status msp_host_setup_weights(const msp_host_setup* s, double* W) {
  if (!s || !W) return MSP_EINVAL;
  std::memcpy(W, s->S.W.data(), sizeof(double) * s->S.W.size());
  return MSP_OK;
}

msp_status msp_host_setup_order(const msp_host_setup* s, int32_t* order) {
  if (!s || !order) return MSP_EINVAL;
  std::memcpy(order, s->S.order.data(), sizeof(int32_t) * s->S.order.size());
  return MSP_OK;
}

msp_status msp_dist_plan(const msp_host_setup* s, const int32_t* owner, int rank, int nranks, int32_t* n_own,
                         int32_t* owned_cells, int32_t* n_ghost, int32_t* ghost_cells, int32_t* send_ptr,
                         int32_t* send_cells, int32_t* recv_ptr) {
  if (!s || nranks < 1 || rank < 0 || rank >= nranks || !n_own || !owned_cells || !n_ghost || !ghost_cells ||
      !send_ptr || !send_cells || !recv_ptr)
    return fail(nullptr, MSP_EINVAL, "msp_dist_plan: bad arguments");
  const int32_t n = s->S.n;
  std::vector<int32_t> own(n);
  for (int32_t i = 0; i < n; ++i) {
    own[i] = owner ? owner[i] : (int32_t)(((int64_t)i * nranks) / n);
    if (own[i] < 0 || own[i] >= nranks) return fail(nullptr, MSP_EINVAL, "msp_dist_plan: owner out of range");
  }
  std::vector<int32_t> rp, ci, dg, src;
  std::string err;
  if (msp::permuted_pattern(s->S, s->M, rp, ci, dg, src, err)) return fail(nullptr, MSP_EINVAL, err);
  CellPlan C = compute_cell_plan(s->S, rp, ci, own, nranks, rank);
  *n_own = (int32_t)C.posown.size();
  *n_ghost = (int32_t)C.ghosts.size();
  for (size_t l = 0; l < C.posown.size(); ++l) owned_cells[l] = s->S.order[C.posown[l]];
  for (size_t k = 0; k < C.ghosts.size(); ++k) ghost_cells[k] = s->S.order[C.ghosts[k]];
  send_ptr[0] = 0;
  recv_ptr[0] = 0;
  for (int q = 0; q < nranks; ++q) {
    int32_t ns = send_ptr[q], nr = 0;
    for (size_t c = 0; c < C.sendl[q].size(); ++c) {
      for (int32_t l : C.sendl[q][c]) send_cells[ns++] = s->S.order[C.posown[l]];
      nr += C.rcnt[q][c];
    }
    send_ptr[q + 1] = ns;
    recv_ptr[q + 1] = recv_ptr[q] + nr;
  }
  return MSP_OK;
}

msp_status msp_dist_level_plan(const msp_host_setup* s, const int32_t* owner, int rank, int nranks, int level,
                               int32_t* buf, int64_t cap, int64_t* len) {
  if (!s || !len || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(nullptr, MSP_EINVAL, "msp_dist_level_plan: bad arguments");
  const msp::HostSetup& S = s->S;
  const int L = (int)S.lv.size();
  if (level < 1 || level >= L) return fail(nullptr, MSP_EINVAL, "msp_dist_level_plan: level must be in [1, levels)");
  const int32_t n = S.n;
  std::vector<int32_t> own(n);
  for (int32_t i = 0; i < n; ++i) {
    own[i] = owner ? owner[i] : (int32_t)(((int64_t)i * nranks) / n);
    if (own[i] < 0 || own[i] >= nranks) return fail(nullptr, MSP_EINVAL, "msp_dist_level_plan: owner out of range");
  }
  std::vector<int32_t> rp, ci, dg, src;
  std::string err;
  if (msp::permuted_pattern(S, s->M, rp, ci, dg, src, err)) return fail(nullptr, MSP_EINVAL, err);
  // effective cell owners (ABMC blocks whole, as the distributed setup)
  CellPlan C = compute_cell_plan(S, rp, ci, own, nranks, rank);
  std::vector<int32_t> own_cell(n);
  for (int32_t p = 0; p < n; ++p) own_cell[S.order[p]] = C.own_pos[p];
  std::vector<std::vector<int32_t>> perms(L);
  for (int l = 0; l < L; ++l) perms[l] = level_perm(S.lv[l]);
  const auto owners = level_owners(S, own_cell, level + 1);
  const LevelPlan R = plan_level(S, perms, owners, level, rank, nranks);
  std::vector<int32_t> out = {(int32_t)R.rows.size(), (int32_t)R.gx.size(), (int32_t)R.gp.size(), (int32_t)R.gm.size()};
  for (const auto* v : {&R.rows, &R.gx, &R.gp, &R.gm}) out.insert(out.end(), v->begin(), v->end());
  for (int q = 0; q < nranks; ++q)
    for (const auto* v : {&R.needx[q], &R.needp[q], &R.needm[q]}) {
      out.push_back((int32_t)v->size());
      out.insert(out.end(), v->begin(), v->end());
    }
  out.push_back((int32_t)owners[level].size());
  out.insert(out.end(), owners[level].begin(), owners[level].end());
  out.insert(out.end(), perms[level].begin(), perms[level].end());
  *len = (int64_t)out.size();
  if (buf) {
    if (cap < *len) return fail(nullptr, MSP_EINVAL, "msp_dist_level_plan: buffer too small");
    std::memcpy(buf, out.data(), sizeof(int32_t) * out.size());
  }
  return MSP_OK;
}

void msp_host_setup_free(msp_host_setup* s) { delete s; }

msp_status msp_partition_owner(const msp_host_setup* s, int nx, int ny, int nz, int nranks, int32_t* owner) {
  if (!s || !owner || nranks < 1 || nranks > nz) return MSP_EINVAL;
  const int64_t plane = (int64_t)nx * ny;
  const int32_t n = s->S.n;
  if ((int64_t)nx * ny * nz != n) return MSP_EINVAL;
  std::vector<int32_t> zstart(nranks + 1, 0);
  const int base = nz / nranks, extra = nz % nranks;
  for (int r = 0; r < nranks; ++r) zstart[r + 1] = zstart[r] + base + (r < extra ? 1 : 0);
  auto slab = [&](int32_t c) {
    const int k = (int)(c / plane);
    return (int32_t)(std::upper_bound(zstart.begin(), zstart.end(), k) - zstart.begin() - 1);
  };
  if (s->S.prm.bilu_order == 0) {
    for (int32_t c = 0; c < n; ++c) owner[c] = slab(c);
    return MSP_OK;
  }
  const auto& blk = s->S.level1_agg;
  int32_t nb = 0;
  for (int32_t v : blk) nb = std::max(nb, v + 1);
  std::vector<int32_t> lowest(nb, INT32_MAX);
  for (int32_t c = 0; c < n; ++c) lowest[blk[c]] = std::min(lowest[blk[c]], c);
  for (int32_t c = 0; c < n; ++c) owner[c] = slab(lowest[blk[c]]);
  return MSP_OK;
}

}  // extern "C"
