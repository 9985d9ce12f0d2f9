// GMRES(m) on the device: orthogonalisation (DCGS2 / CGS2 / MGS), Arnoldi steps and
// their graphs, the restart-cycle graph, the solve loop (part of solver.cu's translation unit).
#pragma once

namespace {

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

#ifndef MSP_DOT_MINB
#define MSP_DOT_MINB 2
#endif
template <int NV>
void cgs_dot_t(msp_handle* h, int nv, const double* V, const double* w, double* out, const double* addend,
               double* raw, int sq) {
  constexpr int MINB = MSP_DOT_MINB;
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
      klaunch(h->s, h->pdl, cgs_dot_kernel<16, 2, MSP_DOT_MINB>, dim3(kRedBlocks, (nv + 15) / 16), kRedThreads, h->N / 2, nv, V,
              h->N, w, h->part, out, addend, raw, sq, h->ticket);
    else
      klaunch(h->s, h->pdl, cgs_dot_kernel<16, 1, MSP_DOT_MINB>, dim3(kRedBlocks, (nv + 15) / 16), kRedThreads, h->N, nv, V,
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
  // staged (cp.async) pass 2, one CTA per SM: k <= 8 at 1024 threads, 9 <= k <= 16 and
  // k > 16 at 384 threads (k > 16: 209 KB of slots; DCGS2 at j = 25 454 -> 388 us vs 256
  // threads, at j = 15 251 -> 245 us vs 512), single-buffered (C3: orthogonalisation at k = 15 0.295 ->
  // 0.255 ms, at k = 25 0.503 -> 0.457 ms; double-buffered forms measured slower, removed)
  if constexpr (NV == 8) {
    if (ew2_ok(h)) { dcgs_staged_launch<8, 1024, 1>(h, k, vk, w, st_in); return; }
  }
  if constexpr (NV == 16) {
    if (ew2_ok(h)) { dcgs_staged_launch<16, 384, 1>(h, k, vk, w, st_in); return; }
  }
  if constexpr (NV == 32) {                       // fused staged pass 2 for k > 16
    if (ew2_ok(h)) { dcgs_staged_launch<32, 384, 1>(h, k, vk, w, st_in); return; }
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

// zbasis mode: each Arnoldi step keeps z_j = B v_j (it computes it anyway), so the cycle end
// forms x += Z y' (one pass over k vectors) instead of applying B to V y (a whole MSP
// application per cycle end).  Single GPU, per-step graphs or direct launches.
bool zmode(const msp_handle* h) { return h->zbasis && !h->comm && !h->cycle_graphs; }

// One Arnoldi step j: z = B v_j; w = A z (into V[j+1]); orthogonalise (CGS2 or MGS);
// hcol[0..j+1] = H(:, j); V[j+1] normalised; hcol copied to pinned host memory.
void arnoldi_step(msp_handle* h, int j, bool record_to_host = true) {
  const size_t N = h->N;
  double* vj = h->V + (size_t)j * N;
  double* w = h->V + (size_t)(j + 1) * N;
  double* zj = (h->Z && zmode(h)) ? h->Z + (size_t)j * N : h->z;
  msp_apply_dev(h, vj, zj);
  {
    Nvtx nvt("a2 BSR SpMV");
    if (overlap_ok(h)) {
      spmv_overlapped(h, 0, zj, h->b, nullptr, w);
    } else {
      exch_cell(h, zj, h->b, -1);
      launch_spmv(h, 0, zj, nullptr, w);
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
  h->Z = zmode(h) ? h->dalloc<double>((size_t)(m + 1) * h->N) : nullptr;
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
      std::vector<double> nu_used(m, 1.0), rho_used(m, 1.0);
      std::vector<std::vector<double>> h2_used(m);
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
          nu_used[j] = nup;                  // v_j's finalisation in step j (zbasis cycle end)
          rho_used[j] = rhop;
          h2_used[j] = h2p;
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
      const bool zb = h->Z && zmode(h) && !cyc;
      if (zb && h->prm.orth == 2) {
        // DCGS2: step j applied B to the provisional v_j; the final basis vector is
        // v_j = (nu_j v_j' - sum_{l<j} h2_j[l] v_l) / rho_j, so B v_j = sum_{i<=j} T[i][j] z_i
        // with T upper triangular, and B V y = Z (T y)
        std::vector<double> T((size_t)k * k, 0.0), yt(k, 0.0);
        for (int j = 0; j < k; ++j) {
          T[(size_t)j * k + j] = nu_used[j] / rho_used[j];
          for (int i = 0; i < j; ++i) {
            double acc = 0.0;
            for (int l = i; l < j; ++l) acc += h2_used[j][l] * T[(size_t)i * k + l];
            T[(size_t)i * k + j] = -acc / rho_used[j];
          }
        }
        for (int i = 0; i < k; ++i) {
          double acc = 0.0;
          for (int j = i; j < k; ++j) acc += T[(size_t)i * k + j] * y[j];
          yt[i] = acc;
        }
        y.assign(yt.begin(), yt.end());
        y.resize(m);
      }
      for (int i = 0; i < k; ++i) y[i] = -y[i];
      CK(cudaMemcpyAsync(h->dh1, y.data(), sizeof(double) * k, cudaMemcpyHostToDevice, h->s));
      CK(cudaMemsetAsync(h->u, 0, sizeof(double) * N, h->s));
      if (zb) {
        // x += Z y (z_j = B v_j kept by the steps): no MSP application at the cycle end
        cgs_axpy<false>(h, k, h->Z, h->dh1, h->u, h->lred, nullptr, nullptr, -1);
        klaunch(h->s, h->pdl, axpy_kernel, kRedBlocks, kRedThreads, N, 1.0, h->u, h->xin); ++h->nlaunch;
      } else {
        cgs_axpy<false>(h, k, h->V, h->dh1, h->u, h->lred, nullptr, nullptr, -1);
        msp_apply_dev(h, h->u, h->z);
        klaunch(h->s, h->pdl, axpy_kernel, kRedBlocks, kRedThreads, N, 1.0, h->z, h->xin); ++h->nlaunch;
      }
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
