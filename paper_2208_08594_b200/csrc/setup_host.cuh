// SETUP glue on the host: config / BSR intake and index checks, SELL level layouts,
// BILU per-cell tables (part of solver.cu's translation unit).
#pragma once

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
    if (cudaMemcpy(M.ci.data(), A->col_idx, sizeof(int32_t) * nnzb, cudaMemcpyDeviceToHost) != cudaSuccess) {
      err = "msp_bsr: device copy failed";
      return MSP_ECUDA;
    }
    if (view) {                                  // values stay on the device (fetched if a host step needs them)
      M.v.device_view(A->values, nv, [](double* dst, const double* src, size_t count) {
        CK(cudaMemcpy(dst, src, sizeof(double) * count, cudaMemcpyDeviceToHost));
      });
    } else if (cudaMemcpy(M.v.owned(nv), A->values, sizeof(double) * nv, cudaMemcpyDeviceToHost) != cudaSuccess) {
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

void dist_localize(msp_handle* h, const msp::BlockMat& A, const msp::HostSetup& S, const std::vector<int32_t>& rp,
                   const std::vector<int32_t>& ci, const std::vector<int32_t>& dg, const std::vector<int32_t>& src,
                   const std::vector<double>& F, const std::vector<std::vector<int32_t>>& perms,
                   const double* dF = nullptr, const double* dAnat = nullptr);



}  // namespace
