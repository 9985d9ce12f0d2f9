// C-ABI (include/msp.h): setup, update, solve, apply, stats (part of solver.cu's
// translation unit).
#pragma once

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
  if (const char* e = std::getenv("MSP_ZBASIS")) h->zbasis = std::atoi(e);
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


}  // extern "C"
