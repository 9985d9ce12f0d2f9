// Hot-path launch sequences: a2/a8 SpMV, a9 BILU, PGS-MC sweeps, V-cycles (single GPU
// and partitioned), the MSP application (part of solver.cu's translation unit).
#pragma once

namespace {

// ----------------------------------------------------------------- launches

template <int B>
void launch_spmv_t(cudaStream_t s, bool pdl, int mode, int n, const int* rp, const int* ci, const double* val,
                   const double* x, const double* g, double* y) {
  constexpr int TS = (B <= 4) ? 4 : 8;
  const unsigned grid = nblk((size_t)n * TS, 256);
  if (B == 4 && mode != 2) {
    const int* none = nullptr;
    const unsigned g4 = nblk((size_t)n * 4, MSP_SPMV_TPB);
    if (mode == 0) klaunch(s, pdl, bsr_spmv4c_kernel<0>, g4, MSP_SPMV_TPB, n, rp, ci, val, x, g, y, none);
    else klaunch(s, pdl, bsr_spmv4c_kernel<1>, g4, MSP_SPMV_TPB, n, rp, ci, val, x, g, y, none);
    return;
  }
  if constexpr (B >= 5) {
    if (mode != 2) {
      const unsigned g8 = nblk((size_t)n * 8, MSP_SPMV8_TPB);
      if (mode == 0) klaunch(s, pdl, bsr_spmv8c_kernel<B, 0>, g8, MSP_SPMV8_TPB, n, rp, ci, val, x, g, y);
      else klaunch(s, pdl, bsr_spmv8c_kernel<B, 1>, g8, MSP_SPMV8_TPB, n, rp, ci, val, x, g, y);
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
    klaunch(h->s, h->pdl, pcol_resid_ell4_kernel, nblk(h->n, MSP_A8_TPB), MSP_A8_TPB, (int)h->n, (int)h->n, (int)h->pell_w,
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
      klaunch(h->s, h->pdl, pcol_resid_ell4_kernel, nblk(nr, MSP_A8_TPB), MSP_A8_TPB, nr, (int)h->n, (int)h->pell_w,
              (const int*)h->pell_c, (const double*)h->pell_v, (const double*)x, g, y, (const int*)rows);
    else if (mode == 2)
      klaunch(h->s, h->pdl, pcol_resid4_kernel, nblk((size_t)nr * 4, 256), 256, nr, (const int*)h->rp,
              (const int*)h->ci, (const double*)h->Pcol, (const double*)x, g, y, (const int*)rows);
    else
      klaunch(h->s, h->pdl, bsr_spmv4c_kernel<0>, nblk((size_t)nr * 4, MSP_SPMV_TPB), MSP_SPMV_TPB, nr, (const int*)h->rp,
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
        klaunch(h->s, h->pdl, kf, nblk((size_t)(b1 - b0) * TM, MSP_BILU_META8_TPB), MSP_BILU_META8_TPB, b0, b1,
                (const int4*)h->bm_f, (const int4*)h->bm_cf, (const int4*)h->bm_b,
                (const int4*)h->bm_cb, (const int4*)h->bm_sl, (const int*)h->ci, (const double*)h->Fval, v, wp, z);
        return;
      }
    }
    if constexpr (B == 4 && !WF) {
      if (h->bm_f && !h->comm) {             // per-slot metadata: shorter dependent load chain
        const unsigned grid4 = nblk((size_t)(b1 - b0) * TM, MSP_BILU_META_TPB);
        if (kind == 0)
          klaunch(h->s, h->pdl, bilu_meta4_kernel<MAXC, true, false>, grid4, MSP_BILU_META_TPB, b0, b1, (const int4*)h->bm_f,
                  (const int4*)h->bm_cf, (const int4*)h->bm_b, (const int4*)h->bm_cb, (const int4*)h->bm_sl,
                  (const int*)h->ci, (const double*)h->Fval, v, wp, z);
        else if (kind == 1)
          klaunch(h->s, h->pdl, bilu_meta4_kernel<MAXC, false, true>, grid4, MSP_BILU_META_TPB, b0, b1, (const int4*)h->bm_f,
                  (const int4*)h->bm_cf, (const int4*)h->bm_b, (const int4*)h->bm_cb, (const int4*)h->bm_sl,
                  (const int*)h->ci, (const double*)h->Fval, v, wp, z);
        else
          klaunch(h->s, h->pdl, bilu_meta4_kernel<MAXC, true, true>, grid4, MSP_BILU_META_TPB, b0, b1, (const int4*)h->bm_f,
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
  const unsigned grid = nblk(h->n, MSP_XFER_TPB);
  double* x0 = nullptr;
  const double* d0 = nullptr;
  int c1 = 0;
  if (fuse_init && !h->lv.empty() && h->prm.pre_sweeps > 0) {
    x0 = h->lv[0].x;
    d0 = h->lv[0].diag;
    c1 = h->lv[0].color_row[1];
  }
  switch (h->b) {
#define CASE(BV) case BV: klaunch(h->s, h->pdl, restrict_pressure_kernel<BV>, grid, MSP_XFER_TPB, h->n, h->W, g, h->cell_of_l0, rp0, x0, d0, c1, pk); break;
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
  static const int tpb_coarse = std::getenv("MSP_SELL_TPB_COARSE") ? std::atoi(std::getenv("MSP_SELL_TPB_COARSE")) : 64;   // C3 V-cycle 277.4 -> 275.2 us vs 128
  const int tpb = (LPR == 1) ? h->sell_tpb : tpb_coarse;
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
      klaunch(h->s, h->pdl, sell_row_uniform_kernel<WR, RES>, nblk((size_t)(s1 - s0) * kSell, MSP_UNI_TPB), MSP_UNI_TPB, s0, s1,
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
  klaunch(h->s, h->pdl, restrict_kernel, nblk(nn, MSP_XFER_TPB), MSP_XFER_TPB, nn, L.pt_ptr, L.pt_idx, L.r, bn,
                                                   fuse_next ? h->lv[l + 1].x : nullptr,
                                                   fuse_next ? h->lv[l + 1].diag : nullptr,
                                                   fuse_next ? h->lv[l + 1].color_row[1] : 0);
  ++h->nlaunch;
  vcycle(h, l + 1, fuse_next);
  klaunch(h->s, h->pdl, prolong_kernel, nblk(L.n, MSP_XFER_TPB), MSP_XFER_TPB, L.n, L.agg, xn, L.x, HaloPack{}); ++h->nlaunch;
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
  klaunch(h->s, h->pdl, gather_kernel, nblk(h->n, MSP_XFER_TPB), MSP_XFER_TPB, h->n, h->l0_of_cell, level0_x(h), h->wp); ++h->nlaunch;
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


}  // namespace
