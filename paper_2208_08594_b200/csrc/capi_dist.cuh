// C-ABI of the distributed path: NCCL / loopback setups and solves (part of solver.cu's
// translation unit).
#pragma once

extern "C" {

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


}  // extern "C"
