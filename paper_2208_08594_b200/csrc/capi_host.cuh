// C-ABI host-setup introspection and host-only distributed plans (no GPU; part of
// solver.cu's translation unit).
#pragma once

extern "C" {

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
