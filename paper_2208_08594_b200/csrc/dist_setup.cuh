// Distributed SETUP: partitioned level plans, halo plans, cell-space
// and level localization (part of solver.cu's translation unit).
#pragma once

namespace {

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


// ---------------------------------------------------------------------------
// Distributed setup.  Rank 0 runs the (deterministic) global host setup
// and broadcasts it (MSP_DIST_SETUP_ALL=1: every rank runs it), so colorings, aggregates,
// orderings and factors are those of 1 GPU; every rank then keeps its owned rows.  Cell ownership follows the caller's partition (z-slabs),
// with every ABMC block (= level-1 aggregate) assigned whole to the owner of its
// lowest-index cell, so BILU blocks and level-1 aggregates are never split.
//  cell space : owned cells in global ABMC position order, then ghosts grouped by
//               (owner, block color, position) -> one contiguous receive per color;
//  level 0    : owned rows in global level-0 order (color-major), then ghosts grouped
//               by (owner, level-0 color, global row);
//  levels 1..dist_levels: partitioned like level 0 (rows on the owner of their lowest-
//  index member; plan_level); the levels below and the coarsest are replicated (or on
//  rank 0), their right-hand side assembled by an allgather of every rank's owned rows.
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


}  // namespace
