// SETUP on the device (NEXT-2): pinned uploads, S1, the Galerkin chain, the rank-0
// setup broadcast, the BILU factorization and do_setup (part of solver.cu's translation unit).
#pragma once

namespace {

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

// Device scratch for the GPU SETUP steps (freed on scope exit, stream-ordered).
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
  if (A.v.dptr) CK(cudaMemcpyAsync(dA.p, A.v.dptr, sizeof(double) * A.v.size(), cudaMemcpyDeviceToDevice, s));
  else h2d_large(s, dA.p, A.v.data(), sizeof(double) * A.v.size());
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
    if (A.v.dptr) CK(cudaMemcpyAsync(dAvals->p, A.v.dptr, sizeof(double) * A.v.size(), cudaMemcpyDeviceToDevice, h->s));
    else h2d_large(h->s, dAvals->p, A.v.data(), sizeof(double) * A.v.size());
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
    else if (A.v.dptr) CK(cudaMemcpyAsync(h->stage, A.v.dptr, sizeof(double) * A.v.size(), cudaMemcpyDeviceToDevice, h->s));
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


}  // namespace
