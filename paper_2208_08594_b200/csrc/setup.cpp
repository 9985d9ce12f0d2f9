// Host SETUP of MSP; see setup.h.  Paper: arXiv 2208.08594
// (PAPER.md, "P:n").  Readings R1-R10: DESIGN.md §3.
#include "setup.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <future>
#include <numeric>
#include <queue>
#include <utility>

namespace msp {

// ---------------------------------------------------------------------------
// Adjacency graph of Eq. 23, symmetrised, by value (R7/c-3).
// Built from a pair list with a counting sort on the row and a per-row sort+unique.
// ---------------------------------------------------------------------------
static Graph graph_from_pairs(int32_t n, const std::vector<std::pair<int32_t, int32_t>>& pairs) {
  Graph G;
  G.xadj.assign(n + 1, 0);
  for (auto& p : pairs) G.xadj[p.first + 1]++;
  for (int32_t i = 0; i < n; ++i) G.xadj[i + 1] += G.xadj[i];
  std::vector<int32_t> tmp(pairs.size()), fill(G.xadj.begin(), G.xadj.end() - 1);
  for (auto& p : pairs) tmp[fill[p.first]++] = p.second;
  G.adj.clear();
  G.adj.reserve(pairs.size());
  std::vector<int32_t> nx(n + 1, 0);
  for (int32_t i = 0; i < n; ++i) {
    auto b = tmp.begin() + G.xadj[i], e = tmp.begin() + G.xadj[i + 1];
    std::sort(b, e);
    auto u = std::unique(b, e);
    for (auto it = b; it != u; ++it) G.adj.push_back(*it);
    nx[i + 1] = (int32_t)G.adj.size();
  }
  G.xadj = nx;
  return G;
}

Graph value_graph(const SpMat& A) {
  const int32_t n = A.n;
  std::vector<int32_t> tp(n + 1, 0), tc(A.ci.size());
  std::vector<uint8_t> tnz(A.ci.size());
  for (int32_t j : A.ci) tp[j + 1]++;
  for (int32_t i = 0; i < n; ++i) tp[i + 1] += tp[i];
  {
    std::vector<int32_t> f(tp.begin(), tp.end() - 1);
    for (int32_t i = 0; i < n; ++i)
      for (int32_t e = A.rp[i]; e < A.rp[i + 1]; ++e) {
        const int32_t q = f[A.ci[e]]++;
        tc[q] = i;
        tnz[q] = A.v[e] != 0.0;
      }
  }
  Graph G;
  G.xadj.assign(n + 1, 0);
  G.adj.reserve(2 * A.ci.size());
  for (int32_t i = 0; i < n; ++i) {
    int32_t e = A.rp[i], f = tp[i];
    const int32_t ee = A.rp[i + 1], fe = tp[i + 1];
    while (e < ee || f < fe) {
      int32_t j;
      bool on = false;
      if (f >= fe || (e < ee && A.ci[e] < tc[f])) { j = A.ci[e]; on = A.v[e] != 0.0; ++e; }
      else if (e >= ee || tc[f] < A.ci[e]) { j = tc[f]; on = tnz[f]; ++f; }
      else { j = A.ci[e]; on = (A.v[e] != 0.0) || tnz[f]; ++e; ++f; }
      if (j != i && on) G.adj.push_back(j);
    }
    G.xadj[i + 1] = (int32_t)G.adj.size();
  }
  return G;
}

Graph block_graph(const BlockMat& A, const std::vector<uint8_t>* nz_given) {
  // nonzero flag per stored block (or the flags computed on the GPU), then symmetrise by
  // merging each row with the transposed row (counting-sort transpose keeps both ascending)
  const int bb = A.b * A.b;
  const int32_t n = A.n;
  std::vector<uint8_t> nz_own;
  if (!nz_given) {
    nz_own.assign(A.ci.size(), 0);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < (int64_t)A.ci.size(); ++e) {
      const double* B = &A.v[(size_t)e * bb];
      bool f = false;
      for (int t = 0; t < bb && !f; ++t) f = (B[t] != 0.0);
      nz_own[e] = f;
    }
  }
  const std::vector<uint8_t>& nz = nz_given ? *nz_given : nz_own;
  std::vector<int32_t> tp(n + 1, 0), tc(A.ci.size());
  std::vector<uint8_t> tnz(A.ci.size());
  for (int32_t j : A.ci) tp[j + 1]++;
  for (int32_t i = 0; i < n; ++i) tp[i + 1] += tp[i];
  {
    std::vector<int32_t> f(tp.begin(), tp.end() - 1);
    for (int32_t i = 0; i < n; ++i)
      for (int32_t e = A.rp[i]; e < A.rp[i + 1]; ++e) {
        const int32_t q = f[A.ci[e]]++;
        tc[q] = i;
        tnz[q] = nz[e];
      }
  }
  Graph G;
  G.xadj.assign(n + 1, 0);
  G.adj.reserve(A.ci.size());
  for (int32_t i = 0; i < n; ++i) {
    int32_t e = A.rp[i], f = tp[i];
    const int32_t ee = A.rp[i + 1], fe = tp[i + 1];
    while (e < ee || f < fe) {
      int32_t j;
      bool on = false;
      if (f >= fe || (e < ee && A.ci[e] < tc[f])) { j = A.ci[e]; on = nz[e]; ++e; }
      else if (e >= ee || tc[f] < A.ci[e]) { j = tc[f]; on = tnz[f]; ++f; }
      else { j = A.ci[e]; on = nz[e] || tnz[f]; ++e; ++f; }
      if (j != i && on) G.adj.push_back(j);
    }
    G.xadj[i + 1] = (int32_t)G.adj.size();
  }
  return G;
}

// ---------------------------------------------------------------------------
// VerticesGrouping (Alg. 3) over VerticesSplitting (Alg. 2).
// Selection key (max static degree |S_i|, lowest index) realised as: V scanned in a
// precomputed degree-sorted order with a monotone cursor; the frontier Ŵ as a binary
// heap with lazy removal of entries that left V (stale entries have no effect in
// Alg. 2's else-branch, so skipping them yields the same accepted sequence).
// ---------------------------------------------------------------------------
int32_t color_groups(const Graph& G, std::vector<int32_t>& color) {
  const int32_t n = (int32_t)G.xadj.size() - 1;
  color.assign(n, -1);
  std::vector<int32_t> bydeg(n);
  std::iota(bydeg.begin(), bydeg.end(), 0);
  std::stable_sort(bydeg.begin(), bydeg.end(),
                   [&](int32_t a, int32_t b) { return G.deg(a) > G.deg(b); });
  std::vector<uint8_t> inV(n, 0), inFront(n, 0);
  std::vector<int32_t> stamp(n, -1);
  // frontier: pop order (max static degree, lowest index) as a bucket queue over degrees,
  // one bitset per degree (same sequence as a (-deg, index) min-heap with lazy removal)
  int32_t maxd = 0;
  for (int32_t v = 0; v < n; ++v) maxd = std::max(maxd, G.deg(v));
  const size_t nw = ((size_t)n + 63) / 64;
  std::vector<std::vector<uint64_t>> fb(maxd + 1);
  std::vector<size_t> flo(maxd + 1, nw);           // lowest possibly non-zero word per degree
  std::vector<int32_t> fcount(maxd + 1, 0), members;
  int32_t ftop = -1;                                // highest degree with members (upper bound)
  auto fpush = [&](int32_t u) {
    const int d = G.deg(u);
    if (fb[d].empty()) fb[d].assign(nw, 0);
    const size_t w = (size_t)u >> 6;
    fb[d][w] |= 1ull << (u & 63);
    flo[d] = std::min(flo[d], w);
    ++fcount[d];
    ftop = std::max(ftop, d);
    members.push_back(u);
  };
  auto fpop = [&]() -> int32_t {                    // best (max degree, min index) or -1
    while (ftop >= 0 && fcount[ftop] == 0) --ftop;
    if (ftop < 0) return -1;
    std::vector<uint64_t>& b = fb[ftop];
    size_t w = flo[ftop];
    while (!b[w]) ++w;
    flo[ftop] = w;
    const int32_t u = (int32_t)((w << 6) + __builtin_ctzll(b[w]));
    b[w] &= b[w] - 1;
    --fcount[ftop];
    return u;
  };
  std::vector<int32_t> cur = bydeg, nxt;
  int32_t g = 0;
  while (!cur.empty()) {
    for (int32_t v : cur) inV[v] = 1;
    size_t cursor = 0;
    while (true) {
      int32_t v = -1;
      for (int32_t t; (t = fpop()) >= 0;) {
        inFront[t] = 0;
        if (inV[t]) { v = t; break; }
      }
      if (v < 0) {
        while (cursor < cur.size() && !inV[cur[cursor]]) ++cursor;
        if (cursor == cur.size()) break;
        v = cur[cursor];
      }
      bool blocked = false;
      for (int32_t e = G.xadj[v]; e < G.xadj[v + 1]; ++e)
        if (color[G.adj[e]] == g) { blocked = true; break; }
      inV[v] = 0;
      if (blocked) continue;                       // -> deferred (W̄)
      color[v] = g;
      for (int32_t e = G.xadj[v]; e < G.xadj[v + 1]; ++e) {
        const int32_t u = G.adj[e];
        inV[u] = 0;                                // undetermined neighbours -> W̄
        stamp[u] = v;
      }
      stamp[v] = v;
      for (int32_t e = G.xadj[v]; e < G.xadj[v + 1]; ++e) {
        const int32_t k = G.adj[e];
        for (int32_t f = G.xadj[k]; f < G.xadj[k + 1]; ++f) {
          const int32_t u = G.adj[f];
          if (stamp[u] == v || !inV[u] || inFront[u]) continue;
          inFront[u] = 1;
          fpush(u);
        }
      }
    }
    for (int32_t u : members) {                    // empty the frontier for the next color
      const int d = G.deg(u);
      const size_t w = (size_t)u >> 6;
      if (fb[d][w] >> (u & 63) & 1ull) { fb[d][w] &= ~(1ull << (u & 63)); --fcount[d]; }
      inFront[u] = 0;
      flo[d] = nw;
    }
    members.clear();
    ftop = -1;
    nxt.clear();
    for (int32_t v : cur)
      if (color[v] < 0) nxt.push_back(v);        // keeps degree order for the next call
    cur.swap(nxt);
    ++g;
  }
  return g;
}

// ---------------------------------------------------------------------------
// NPAIR pairwise aggregation (reading R3).  Strength via t_ij = a_ij + a_ji,
// precomputed per symmetric edge from a merged (row, col) triplet list.  The
// "fewest unaggregated neighbours" selection is a lazy min-heap on (count, index).
// ---------------------------------------------------------------------------
int32_t pair_aggregate(const SpMat& A, std::vector<int32_t>& agg) {
  const int32_t n = A.n;
  // transpose (counting sort by column keeps rows ascending), then per-row merge of
  // the row (j, a_ij) and the transposed row (j, a_ji): t_ij = a_ij + a_ji
  std::vector<int32_t> tp(n + 1, 0), tc(A.ci.size());
  std::vector<double> tv(A.ci.size());
  for (int32_t j : A.ci) tp[j + 1]++;
  for (int32_t i = 0; i < n; ++i) tp[i + 1] += tp[i];
  {
    std::vector<int32_t> f(tp.begin(), tp.end() - 1);
    for (int32_t i = 0; i < n; ++i)
      for (int32_t e = A.rp[i]; e < A.rp[i + 1]; ++e) {
        const int32_t q = f[A.ci[e]]++;
        tc[q] = i;
        tv[q] = A.v[e];
      }
  }
  std::vector<int32_t> xadj(n + 1, 0), adj;
  std::vector<double> tval;
  adj.reserve(2 * A.ci.size());
  tval.reserve(2 * A.ci.size());
  for (int32_t i = 0; i < n; ++i) {
    int32_t e = A.rp[i], f = tp[i];
    const int32_t ee = A.rp[i + 1], fe = tp[i + 1];
    while (e < ee || f < fe) {
      int32_t j;
      double aij = 0.0, aji = 0.0;
      if (f >= fe || (e < ee && A.ci[e] < tc[f])) { j = A.ci[e]; aij = A.v[e]; ++e; }
      else if (e >= ee || tc[f] < A.ci[e]) { j = tc[f]; aji = tv[f]; ++f; }
      else { j = A.ci[e]; aij = A.v[e]; aji = tv[f]; ++e; ++f; }
      if (j == i) continue;
      if (aij != 0.0 || aji != 0.0) {
        adj.push_back(j);
        tval.push_back(aij + aji);
        xadj[i + 1]++;
      }
    }
  }
  for (int32_t i = 0; i < n; ++i) xadj[i + 1] += xadj[i];
  // Selection order: the unaggregated row with the fewest unaggregated neighbours, lowest
  // index on ties.  Counts are small integers, so a bucket queue does it exactly: one
  // three-level bitset per count; the next row is the lowest set bit of the first
  // non-empty bucket (same rows in the same order as a (count, index) min-heap).
  std::vector<int32_t> cnt(n);
  int32_t maxc = 0;
  for (int32_t i = 0; i < n; ++i) { cnt[i] = xadj[i + 1] - xadj[i]; maxc = std::max(maxc, cnt[i]); }
  const size_t w0 = ((size_t)n + 63) / 64, w1 = (w0 + 63) / 64, w2 = (w1 + 63) / 64;
  struct Buckets {
    size_t w0, w1, w2;
    std::vector<uint64_t> b0, b1, b2;
    std::vector<int32_t> size;
    void init(int nb, size_t a, size_t b, size_t c) {
      w0 = a; w1 = b; w2 = c;
      b0.assign((size_t)nb * w0, 0); b1.assign((size_t)nb * w1, 0); b2.assign((size_t)nb * w2, 0);
      size.assign(nb, 0);
    }
    void insert(int c, int32_t i) {
      uint64_t* l0 = &b0[(size_t)c * w0]; uint64_t* l1 = &b1[(size_t)c * w1]; uint64_t* l2 = &b2[(size_t)c * w2];
      const size_t k0 = (size_t)i >> 6, k1 = k0 >> 6, k2 = k1 >> 6;
      l0[k0] |= 1ull << (i & 63);
      l1[k1] |= 1ull << (k0 & 63);
      l2[k2] |= 1ull << (k1 & 63);
      ++size[c];
    }
    void erase(int c, int32_t i) {
      uint64_t* l0 = &b0[(size_t)c * w0]; uint64_t* l1 = &b1[(size_t)c * w1]; uint64_t* l2 = &b2[(size_t)c * w2];
      const size_t k0 = (size_t)i >> 6, k1 = k0 >> 6, k2 = k1 >> 6;
      l0[k0] &= ~(1ull << (i & 63));
      if (!l0[k0]) {
        l1[k1] &= ~(1ull << (k0 & 63));
        if (!l1[k1]) l2[k2] &= ~(1ull << (k1 & 63));
      }
      --size[c];
    }
    int32_t first(int c) const {
      const uint64_t* l0 = &b0[(size_t)c * w0]; const uint64_t* l1 = &b1[(size_t)c * w1];
      const uint64_t* l2 = &b2[(size_t)c * w2];
      for (size_t k2 = 0; k2 < w2; ++k2)
        if (l2[k2]) {
          const size_t k1 = (k2 << 6) + __builtin_ctzll(l2[k2]);
          const size_t k0 = (k1 << 6) + __builtin_ctzll(l1[k1]);
          return (int32_t)((k0 << 6) + __builtin_ctzll(l0[k0]));
        }
      return -1;
    }
  } Q;
  Q.init(maxc + 1, w0, w1, w2);
  for (int32_t i = 0; i < n; ++i) Q.insert(cnt[i], i);
  std::vector<uint8_t> done(n, 0);
  agg.assign(n, -1);
  int32_t na = 0;
  auto release = [&](int32_t m) {
    for (int32_t e = xadj[m]; e < xadj[m + 1]; ++e) {
      const int32_t k = adj[e];
      if (!done[k]) { Q.erase(cnt[k], k); --cnt[k]; Q.insert(cnt[k], k); }
    }
  };
  int c = 0;
  for (int32_t left = n; left > 0;) {
    while (Q.size[c] == 0) ++c;                       // counts only decrease: restart low
    const int32_t i = Q.first(c);
    int32_t best = -1;
    double bt = 0.0;
    for (int32_t e = xadj[i]; e < xadj[i + 1]; ++e)
      if (!done[adj[e]] && tval[e] < bt) { bt = tval[e]; best = adj[e]; }
    if (best < 0) {
      double ba = -1.0;
      for (int32_t e = xadj[i]; e < xadj[i + 1]; ++e)
        if (!done[adj[e]] && std::fabs(tval[e]) > ba) { ba = std::fabs(tval[e]); best = adj[e]; }
    }
    done[i] = 1;
    Q.erase(cnt[i], i);
    --left;
    agg[i] = na;
    if (best >= 0) {
      done[best] = 1;
      Q.erase(cnt[best], best);
      --left;
      agg[best] = na;
    }
    ++na;
    release(i);
    if (best >= 0) release(best);
    c = 0;
  }
  return na;
}

// Galerkin P^T A P (UA-AMG): per coarse row, members ascending (counting sort),
// stored entries ascending, accumulated into a marker-indexed slot from +0.0; the
// row is sorted by coarse column afterwards.  Summation order per slot equals the
// reading of SURVEY c-5, so values are bit-identical to any implementation of it.
SpMat galerkin_rap(const SpMat& A, const std::vector<int32_t>& agg, int32_t nagg) {
  std::vector<int32_t> mp(nagg + 1, 0), mem(A.n);
  for (int32_t i = 0; i < A.n; ++i) mp[agg[i] + 1]++;
  for (int32_t I = 0; I < nagg; ++I) mp[I + 1] += mp[I];
  {
    std::vector<int32_t> f(mp.begin(), mp.end() - 1);
    for (int32_t i = 0; i < A.n; ++i) mem[f[agg[i]]++] = i;
  }
  SpMat C;
  C.n = nagg;
  C.rp.assign(nagg + 1, 0);
  C.ci.reserve(A.ci.size());
  C.v.reserve(A.ci.size());
  std::vector<int32_t> mark(nagg, -1), slot(nagg);
  std::vector<std::pair<int32_t, double>> row;
  for (int32_t I = 0; I < nagg; ++I) {
    row.clear();
    for (int32_t m = mp[I]; m < mp[I + 1]; ++m) {
      const int32_t i = mem[m];
      for (int32_t e = A.rp[i]; e < A.rp[i + 1]; ++e) {
        const int32_t J = agg[A.ci[e]];
        if (mark[J] != I) { mark[J] = I; slot[J] = (int32_t)row.size(); row.push_back({J, 0.0}); }
        row[slot[J]].second += A.v[e];
      }
    }
    std::sort(row.begin(), row.end(),
              [](const std::pair<int32_t, double>& a, const std::pair<int32_t, double>& b) {
                return a.first < b.first;
              });
    for (auto& p : row) { C.ci.push_back(p.first); C.v.push_back(p.second); }
    C.rp[I + 1] = (int32_t)C.ci.size();
  }
  return C;
}

static bool off_diagonal_zero(const SpMat& A) {
  for (int32_t i = 0; i < A.n; ++i)
    for (int32_t e = A.rp[i]; e < A.rp[i + 1]; ++e)
      if (A.ci[e] != i && A.v[e] != 0.0) return false;
  return true;
}

static int32_t aggregate_passes(const SpMat& A0, int passes, std::vector<int32_t>& comp, SpMat* out,
                                const RapFn* rap = nullptr) {
  SpMat cur;                                   // product of the previous pass (pass 0 reads A0)
  comp.resize(A0.n);
  std::iota(comp.begin(), comp.end(), 0);
  int32_t na = A0.n;
  const bool verbose = std::getenv("MSP_SETUP_VERBOSE") != nullptr;
  for (int p = 0; p < passes; ++p) {
    const SpMat& in = (p == 0) ? A0 : cur;
    std::vector<int32_t> a;
    const auto t0 = std::chrono::steady_clock::now();
    na = pair_aggregate(in, a);
    for (auto& c : comp) c = a[c];
    const auto t1 = std::chrono::steady_clock::now();
    SpMat nxt;
    if (!(rap && *rap && (*rap)(in, a, na, nxt) == 0)) nxt = galerkin_rap(in, a, na);
    cur = std::move(nxt);
    if (verbose)
      std::fprintf(stderr, "[msp setup]   pass %d: NPAIR %.3f s, Galerkin %.3f s (n %d -> %d)\n", p,
                   std::chrono::duration<double>(t1 - t0).count(),
                   std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count(), (int)cur.n, (int)na);
  }
  if (out) *out = (passes > 0) ? std::move(cur) : A0;
  return na;
}

// ---------------------------------------------------------------------------
// Decoupling (R4): column sums via a CSC (counting sort on the block column, rows
// ascending), then C_NN^T y = -C_0N^T by Gaussian elimination with partial pivoting
// in the fixed operation order of DESIGN.md R4 (bit-reproducible, no FMA).
// ---------------------------------------------------------------------------
static bool weight_solve(int nc, const double* C, int b, double* y) {
  double M[8][8], r[8];
  for (int i = 0; i < nc; ++i) {
    for (int j = 0; j < nc; ++j) M[i][j] = C[(1 + j) * b + 1 + i];
    r[i] = -C[1 + i];
  }
  for (int k = 0; k < nc; ++k) {
    int p = k;
    double best = std::fabs(M[k][k]);
    for (int i = k + 1; i < nc; ++i) {
      const double a = std::fabs(M[i][k]);
      if (a > best) { best = a; p = i; }
    }
    if (M[p][k] == 0.0) return false;
    if (p != k) {
      for (int j = 0; j < nc; ++j) std::swap(M[k][j], M[p][j]);
      std::swap(r[k], r[p]);
    }
    const double piv = M[k][k];
    for (int i = k + 1; i < nc; ++i) {
      const double f = M[i][k] / piv;
      for (int j = k + 1; j < nc; ++j) {
        const double prod = f * M[k][j];
        M[i][j] = M[i][j] - prod;
      }
      const double pr = f * r[k];
      r[i] = r[i] - pr;
    }
  }
  for (int i = nc - 1; i >= 0; --i) {
    double acc = 0.0;
    for (int j = i + 1; j < nc; ++j) {
      const double prod = M[i][j] * y[j];
      acc = acc + prod;
    }
    y[i] = (r[i] - acc) / M[i][i];
  }
  return true;
}

static int make_weights(const BlockMat& A, int mode, std::vector<double>& W, std::string& err) {
  const int32_t n = A.n;
  const int b = A.b, bb = b * b, nc = b - 1;
  W.assign((size_t)n * b, 0.0);
  for (int32_t c = 0; c < n; ++c) W[(size_t)c * b] = 1.0;
  if (mode == 0 || nc == 0) return 0;
  if (nc > 8) { err = "decoupling: nc > 8 unsupported"; return 1; }
  std::vector<double> C((size_t)n * bb, 0.0);
  if (mode == 2) {
    // CSC of the block pattern (stable in row order) -> sums ascending in p
    std::vector<int32_t> cp(n + 1, 0), ce(A.ci.size());
    for (int32_t c : A.ci) cp[c + 1]++;
    for (int32_t c = 0; c < n; ++c) cp[c + 1] += cp[c];
    std::vector<int32_t> f(cp.begin(), cp.end() - 1);
    for (int32_t p = 0; p < n; ++p)
      for (int32_t e = A.rp[p]; e < A.rp[p + 1]; ++e) ce[f[A.ci[e]]++] = e;
#pragma omp parallel for schedule(static)
    for (int32_t c = 0; c < n; ++c) {
      double* Cc = &C[(size_t)c * bb];
      for (int32_t q = cp[c]; q < cp[c + 1]; ++q) {
        const double* B = &A.v[(size_t)ce[q] * bb];
        for (int t = 0; t < bb; ++t) Cc[t] = Cc[t] + B[t];
      }
    }
  } else {
    for (int32_t c = 0; c < n; ++c)
      for (int32_t e = A.rp[c]; e < A.rp[c + 1]; ++e)
        if (A.ci[e] == c) std::memcpy(&C[(size_t)c * bb], &A.v[(size_t)e * bb], sizeof(double) * bb);
  }
  int32_t bad = -1;
#pragma omp parallel for schedule(static) reduction(max : bad)
  for (int32_t c = 0; c < n; ++c) {
    double y[8];
    if (!weight_solve(nc, &C[(size_t)c * bb], b, y)) {
      bad = std::max(bad, c);
      continue;
    }
    for (int i = 0; i < nc; ++i) W[(size_t)c * b + 1 + i] = y[i];
  }
  if (bad >= 0) {
    err = "decoupling: singular N-N block at cell " + std::to_string(bad);
    return 2;
  }
  return 0;
}

static SpMat pressure_matrix(const BlockMat& A, const std::vector<double>& W) {
  const int b = A.b, bb = b * b;
  SpMat P;
  P.n = A.n;
  P.rp = A.rp;
  P.ci = A.ci;
  P.v.resize(A.ci.size());
#pragma omp parallel for schedule(static)
  for (int32_t c = 0; c < A.n; ++c) {
    const double* w = &W[(size_t)c * b];
    for (int32_t e = A.rp[c]; e < A.rp[c + 1]; ++e) {
      const double* B = &A.v[(size_t)e * bb];
      double acc = 0.0;
      for (int k = 0; k < b; ++k) {
        const double prod = w[k] * B[k * b];
        acc = acc + prod;
      }
      P.v[e] = acc;
    }
  }
  return P;
}

// Graph Laplacian of the cell graph (ABMC blocks when A_PP is diagonal, R5).
static SpMat graph_laplacian(const Graph& G) {
  SpMat L;
  L.n = (int32_t)G.xadj.size() - 1;
  L.rp.assign(L.n + 1, 0);
  for (int32_t c = 0; c < L.n; ++c) {
    bool placed = false;
    for (int32_t e = G.xadj[c]; e < G.xadj[c + 1]; ++e) {
      const int32_t d = G.adj[e];
      if (!placed && d > c) { L.ci.push_back(c); L.v.push_back((double)G.deg(c)); placed = true; }
      L.ci.push_back(d);
      L.v.push_back(-1.0);
    }
    if (!placed) { L.ci.push_back(c); L.v.push_back((double)G.deg(c)); }
    L.rp[c + 1] = (int32_t)L.ci.size();
  }
  return L;
}

namespace {
struct PhaseTimer {
  bool on = std::getenv("MSP_SETUP_VERBOSE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[msp setup] %-28s %8.3f s\n", what, std::chrono::duration<double>(n - t).count());
    t = n;
  }
};
}  // namespace

static void make_ordering(HostSetup& S, PhaseTimer& T, const HostLevel* lv0, const Graph& G) {
  const BlockMat& A = *S.A;
  const int32_t n = A.n;
  std::vector<int32_t> blk(n), bcol;
  int32_t nb;
  if (S.prm.bilu_order == 0) {
    nb = n;
    std::iota(blk.begin(), blk.end(), 0);
    S.bilu_ncolor = color_groups(G, bcol);
  } else {
    if (off_diagonal_zero(S.App)) nb = aggregate_passes(graph_laplacian(G), S.prm.pair_passes, blk, nullptr);
    else if (lv0) { blk = lv0->agg; nb = lv0->n_next; }
    else nb = aggregate_passes(S.App, S.prm.pair_passes, blk, nullptr);
    std::vector<std::pair<int32_t, int32_t>> pr;
    for (int32_t c = 0; c < n; ++c)
      for (int32_t e = G.xadj[c]; e < G.xadj[c + 1]; ++e) {
        const int32_t d = G.adj[e];
        if (blk[c] != blk[d]) pr.push_back({blk[c], blk[d]});
      }
    Graph Q = graph_from_pairs(nb, pr);
    T.mark("  ABMC: quotient graph");
    S.bilu_ncolor = color_groups(Q, bcol);
    T.mark("  ABMC: block coloring");
  }
  S.level1_agg = blk;
  // counting sort by (color, block, cell): cells ascending within a block, blocks
  // ascending within a color.
  std::vector<int32_t> bstart(nb + 1, 0);
  for (int32_t c = 0; c < n; ++c) bstart[blk[c] + 1]++;
  std::vector<int32_t> bsize(nb);
  for (int32_t I = 0; I < nb; ++I) bsize[I] = bstart[I + 1];
  std::vector<int32_t> cstart(S.bilu_ncolor + 1, 0), ccount(S.bilu_ncolor + 1, 0);
  for (int32_t I = 0; I < nb; ++I) { cstart[bcol[I] + 1] += bsize[I]; ccount[bcol[I] + 1]++; }
  for (int32_t g = 0; g < S.bilu_ncolor; ++g) { cstart[g + 1] += cstart[g]; ccount[g + 1] += ccount[g]; }
  std::vector<int32_t> boff(nb), bpos(nb);
  {
    std::vector<int32_t> cf(cstart.begin(), cstart.end() - 1), kf(ccount.begin(), ccount.end() - 1);
    for (int32_t I = 0; I < nb; ++I) { boff[I] = cf[bcol[I]]; cf[bcol[I]] += bsize[I]; bpos[I] = kf[bcol[I]]++; }
  }
  S.order.assign(n, 0);
  S.pos.assign(n, 0);
  {
    std::vector<int32_t> f = boff;
    for (int32_t c = 0; c < n; ++c) { S.pos[c] = f[blk[c]]++; S.order[S.pos[c]] = c; }
  }
  S.blk_ptr.assign(nb + 1, 0);
  std::vector<int32_t> blk_by_pos(nb);
  for (int32_t I = 0; I < nb; ++I) blk_by_pos[bpos[I]] = I;
  for (int32_t k = 0; k < nb; ++k) S.blk_ptr[k + 1] = S.blk_ptr[k] + bsize[blk_by_pos[k]];
  S.color_blk_ptr = ccount;
}


int run_host_setup(const BlockMat& A, const Params& prm, HostSetup& S, std::string& err) {
  PhaseTimer T;
  S.prm = prm;
  S.A = &A;
  S.n = A.n;
  if (!prm.s1_given) {                 // else: S.W and S.App computed on the GPU (NEXT-2)
    int rc = make_weights(A, prm.decoupling, S.W, err);
    if (rc) return rc;
    T.mark("decoupling weights");
    S.App = pressure_matrix(A, S.W);
    T.mark("A_PP");
  }
  S.lv.clear();
  S.lv.reserve(prm.max_levels + 1);    // levels stay in place while their colorings run
  S.coarse_diag = false;
  // The greedy steps are sequential by definition, but independent of one another once
  // their input exists: the Alg. 2/3 coloring of level l needs only A_l, the ABMC order
  // only level 0's aggregates and A's cell graph.  They run as host tasks concurrently
  // with the NPAIR + Galerkin chain (same functions, same inputs: identical results).
  std::vector<std::future<void>> jobs;
  std::future<void> abmc;
  // A's cell graph (the ABMC input besides level 0's aggregates) from the start
  std::shared_future<Graph> cell_graph =
      std::async(std::launch::async, [&S, &A]() { return block_graph(A, S.block_nz.empty() ? nullptr : &S.block_nz); })
          .share();
  // (level 0 is passed explicitly: the task never reads S.lv while the chain appends)
  auto start_abmc = [&](const HostLevel* lv0) {
    abmc = std::async(std::launch::async, [&S, lv0, cell_graph]() {
      PhaseTimer Tq;
      Tq.on = false;
      make_ordering(S, Tq, lv0, cell_graph.get());
    });
  };
  SpMat cur = S.App;
  int rc_loop = 0;
  for (int l = 0;; ++l) {
    if (cur.n <= prm.coarsest_max_dof) break;
    if (l + 1 >= prm.max_levels) { err = "AMG: max_levels reached above coarsest_max_dof"; rc_loop = 5; break; }
    HostLevel L;
    SpMat nxt;
    const int32_t nn = aggregate_passes(cur, prm.pair_passes, L.agg, &nxt, &prm.rap);
    T.mark("NPAIR + Galerkin level");
    if ((double)nn > 0.9 * (double)cur.n) {
      if (off_diagonal_zero(cur)) { S.coarse_diag = true; break; }
      err = "AMG: coarsening stalled at level " + std::to_string(l);
      rc_loop = 5;
      break;
    }
    L.n_next = nn;
    L.A = std::move(cur);
    S.lv.push_back(std::move(L));
    HostLevel* Lp = &S.lv.back();
    jobs.push_back(std::async(std::launch::async, [Lp]() { Lp->ncolor = color_groups(value_graph(Lp->A), Lp->color); }));
    if (l == 0) start_abmc(Lp);
    cur = std::move(nxt);
  }
  for (auto& j : jobs) j.get();
  if (rc_loop) {
    if (abmc.valid()) abmc.get();
    return rc_loop;
  }
  T.mark("colorings (concurrent)");
  S.Ac = std::move(cur);
  for (int32_t i = 0; i < S.Ac.n; ++i) {
    bool has = false;
    for (int32_t e = S.Ac.rp[i]; e < S.Ac.rp[i + 1]; ++e)
      if (S.Ac.ci[e] == i && S.Ac.v[e] != 0.0) has = true;
    if (!has && S.coarse_diag) { err = "coarsest: zero diagonal at row " + std::to_string(i); return 2; }
  }
  for (size_t l = 0; l < S.lv.size(); ++l) {
    const SpMat& M = S.lv[l].A;
    for (int32_t i = 0; i < M.n; ++i) {
      bool has = false;
      for (int32_t e = M.rp[i]; e < M.rp[i + 1]; ++e)
        if (M.ci[e] == i && M.v[e] != 0.0) has = true;
      if (!has) { err = "PGS-MC: zero diagonal at level " + std::to_string(l) + " row " + std::to_string(i); return 2; }
    }
  }
  T.mark("checks");
  if (!abmc.valid()) start_abmc(S.lv.empty() ? nullptr : &S.lv[0]);
  abmc.get();
  T.mark("ABMC ordering (concurrent)");
  return 0;
}

// ---------------------------------------------------------------------------
// Block ILU(0) over A's pattern in the ordering positions (R5).  The matrix is
// first permuted (rows and columns to positions, columns sorted); then for each row
// i, for each k < i stored in row i (ascending): L_ik = A_ik D~_k^-1, and every
// stored (k, j), j > k, that is also stored in row i updates A_ij -= L_ik A_kj
// (row-marker lookup).  D~_i^-1 by Gauss-Jordan with partial pivoting.
// ---------------------------------------------------------------------------
bool invert_block(int b, const double* D, double* Dinv) {
  double a[8][8], r[8][8];
  for (int i = 0; i < b; ++i)
    for (int j = 0; j < b; ++j) { a[i][j] = D[i * b + j]; r[i][j] = (i == j) ? 1.0 : 0.0; }
  for (int k = 0; k < b; ++k) {
    int p = k;
    for (int i = k + 1; i < b; ++i) if (std::fabs(a[i][k]) > std::fabs(a[p][k])) p = i;
    if (a[p][k] == 0.0) return false;
    if (p != k) for (int j = 0; j < b; ++j) { std::swap(a[k][j], a[p][j]); std::swap(r[k][j], r[p][j]); }
    const double piv = a[k][k];                 // row divided by the pivot (R5)
    for (int j = 0; j < b; ++j) { a[k][j] /= piv; r[k][j] /= piv; }
    for (int i = 0; i < b; ++i) {
      if (i == k) continue;
      const double f = a[i][k];
      if (f == 0.0) continue;
      for (int j = 0; j < b; ++j) { a[i][j] -= f * a[k][j]; r[i][j] -= f * r[k][j]; }
    }
  }
  for (int i = 0; i < b; ++i) for (int j = 0; j < b; ++j) Dinv[i * b + j] = r[i][j];
  return true;
}

int permuted_pattern(const HostSetup& S, const BlockMat& A, std::vector<int32_t>& rp, std::vector<int32_t>& ci,
                     std::vector<int32_t>& dg, std::vector<int32_t>& src, std::string& err) {
  const int32_t n = A.n;
  rp.assign(n + 1, 0);
  for (int32_t p = 0; p < n; ++p) {
    const int32_t c = S.order[p];
    rp[p + 1] = rp[p] + (A.rp[c + 1] - A.rp[c]);
  }
  ci.resize(A.ci.size());
  src.resize(A.ci.size());
  dg.assign(n, -1);
  int32_t bad = -1;
#pragma omp parallel reduction(max : bad)
  {
    std::vector<std::pair<int32_t, int32_t>> tmp;   // rows are independent (disjoint output ranges)
#pragma omp for schedule(static)
    for (int32_t p = 0; p < n; ++p) {
      const int32_t c = S.order[p];
      tmp.clear();
      for (int32_t e = A.rp[c]; e < A.rp[c + 1]; ++e) tmp.push_back({S.pos[A.ci[e]], e});
      std::sort(tmp.begin(), tmp.end());
      for (size_t t = 0; t < tmp.size(); ++t) {
        ci[rp[p] + t] = tmp[t].first;
        src[rp[p] + t] = tmp[t].second;
        if (tmp[t].first == p) dg[p] = rp[p] + (int32_t)t;
      }
      if (dg[p] < 0) bad = std::max(bad, c);
    }
  }
  if (bad >= 0) { err = "BILU: missing diagonal block at cell " + std::to_string(bad); return 1; }
  return 0;
}

int bilu_factor_permuted(const HostSetup& S, const BlockMat& A, std::vector<int32_t>& rp,
                         std::vector<int32_t>& ci, std::vector<int32_t>& dg,
                         std::vector<int32_t>& src, std::vector<double>& F, std::string& err) {
  const int32_t n = A.n;
  const int b = A.b, bb = b * b;
  int rc0 = permuted_pattern(S, A, rp, ci, dg, src, err);
  if (rc0) return rc0;
  F.resize(A.v.size());
  for (size_t e = 0; e < src.size(); ++e)
    std::memcpy(&F[e * bb], &A.v[(size_t)src[e] * bb], sizeof(double) * bb);
  // rows of one block color are independent (ABMC / RB orders); cells inside an
  // aggregate block are eliminated in order by one thread
  int32_t bad = -1;
  const int ncol = (int)S.color_blk_ptr.size() - 1;
  for (int col = 0; col < ncol; ++col) {
#pragma omp parallel reduction(max : bad)
    {
      std::vector<int32_t> mark(n, -1);
      double T[64];
#pragma omp for schedule(dynamic, 256)
      for (int32_t k = S.color_blk_ptr[col]; k < S.color_blk_ptr[col + 1]; ++k) {
        for (int32_t i = S.blk_ptr[k]; i < S.blk_ptr[k + 1]; ++i) {
          for (int32_t e = rp[i]; e < rp[i + 1]; ++e) mark[ci[e]] = e;
          for (int32_t e = rp[i]; e < dg[i]; ++e) {
            const int32_t kk = ci[e];
            double* Lik = &F[(size_t)e * bb];
            const double* Dk = &F[(size_t)dg[kk] * bb];      // holds D~_k^-1
            for (int r = 0; r < b; ++r)
              for (int c = 0; c < b; ++c) {
                double sum = 0.0;
                for (int t = 0; t < b; ++t) sum += Lik[r * b + t] * Dk[t * b + c];
                T[r * b + c] = sum;
              }
            std::memcpy(Lik, T, sizeof(double) * bb);
            for (int32_t f = dg[kk] + 1; f < rp[kk + 1]; ++f) {
              const int32_t m = mark[ci[f]];
              if (m < 0) continue;
              const double* Ukj = &F[(size_t)f * bb];
              double* Aij = &F[(size_t)m * bb];
              for (int r = 0; r < b; ++r)
                for (int c = 0; c < b; ++c) {
                  double sum = 0.0;
                  for (int t = 0; t < b; ++t) sum += Lik[r * b + t] * Ukj[t * b + c];
                  Aij[r * b + c] -= sum;
                }
            }
          }
          for (int32_t e = rp[i]; e < rp[i + 1]; ++e) mark[ci[e]] = -1;
          double* Dd = &F[(size_t)dg[i] * bb];
          if (!invert_block(b, Dd, T)) {
            bad = std::max(bad, i);
            continue;
          }
          std::memcpy(Dd, T, sizeof(double) * bb);
        }
      }
    }
    if (bad >= 0) {
      err = "BILU: singular pivot block at cell " + std::to_string(S.order[bad]);
      return 2;
    }
  }
  return 0;
}

}  // namespace msp
