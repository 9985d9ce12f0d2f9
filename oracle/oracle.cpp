// ============================================================================
// ORACLE — plain, slow, sequential CPU C++ implementation of MSP-GMRES.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load or call this library.  It shares
// no code, header, table or helper with the product (paper_2208_08594_b200/);
// the only common input source is gen/ (seeded inputs, no method arithmetic).
//
// Paper: Zhao, Zhang, Feng, Shu, "An Improved Multi-Stage Preconditioner on GPUs
// for Compositional Reservoir Simulation" (arXiv 2208.08594) = /root/reference/
// PAPER.md; "P:n" = PAPER.md line n.  Readings of gaps are SURVEY.md §8(c) c-1..c-13,
// listed in DESIGN.md §3.
//
// Everything is in NATURAL cell order; color orders and the ABMC elimination
// order are applied logically (loops over groups / positions), a deliberately
// different storage path from the GPU's permuted storage (SURVEY c-1).
// FP64 throughout; compiled with -ffp-contract=off; every sum starts at +0.0
// and runs in ascending index order unless stated.
//
// Timing switch (SURVEY §8(d) "Mode SEQ / Mode OMP"): orc_set_threads(n) runs the loops
// whose per-element arithmetic is independent (SpMV rows, PGS-MC rows of one color, BILU
// blocks of one color, vector updates, the CGS2 dots over basis vectors) on n OpenMP
// threads.  Every sum keeps its sequential order, so results are BIT-IDENTICAL for any n
// (tests/test_oracle.py::test_omp_mode_bit_identical).
//
// Parity status: every function is pinned by a -m "not gpu"
// test except NPAIR's correspondence to the cited Napov-Notay scheme, which the
// paper only names: "parity unpinned" w.r.t. the paper for NPAIR; the
// reading itself is pinned by the SPEC examples.
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <set>
#include <string>
#include <utility>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace orc {

static int g_threads = 1;        // OMP timing mode (1 = SEQ)
#define ORC_PAR _Pragma("omp parallel for schedule(static) num_threads(g_threads) if(g_threads > 1)")

struct Csr {                  // scalar CSR, columns ascending per row
  int n = 0;
  std::vector<int> ptr, col;
  std::vector<double> val;
};

struct Bsr {                  // block CSR, b x b blocks ROW-major (Eq. 20 order)
  int n = 0, b = 0;
  std::vector<int> ptr, col;
  std::vector<double> val;
  const double* blk(int e) const { return &val[(size_t)e * b * b]; }
  double* blk(int e) { return &val[(size_t)e * b * b]; }
};

using Graph = std::vector<std::vector<int>>;   // sorted neighbour lists S_i (Table 1)

static std::string g_err;

// ---------------------------------------------------------------------------
// c-1: BSR matrix-vector product y = A x (the residuals r = g - Aw of Alg. 1,
// P:271-275, and the GMRES operator).  Plain definition: y_c = sum_d A_cd x_d.
// ---------------------------------------------------------------------------
static void bsr_spmv(const Bsr& A, const double* x, double* y) {
  const int b = A.b;
  ORC_PAR
  for (int c = 0; c < A.n; ++c)
    for (int r = 0; r < b; ++r) {
      double s = 0.0;
      for (int e = A.ptr[c]; e < A.ptr[c + 1]; ++e) {
        const double* B = A.blk(e);
        const int d = A.col[e];
        for (int k = 0; k < b; ++k) s += B[r * b + k] * x[(size_t)d * b + k];
      }
      y[(size_t)c * b + r] = s;
    }
}

static void csr_spmv(const Csr& A, const double* x, double* y) {
  ORC_PAR
  for (int i = 0; i < A.n; ++i) {
    double s = 0.0;
    for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e) s += A.val[e] * x[A.col[e]];
    y[i] = s;
  }
}

static double dot(const std::vector<double>& a, const std::vector<double>& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
static double nrm2(const std::vector<double>& a) { return std::sqrt(dot(a, a)); }

// ---------------------------------------------------------------------------
// c-3: adjacency graph G_A(V,E) of Eq. 23: edge (i,j) iff i != j and
// a_ij != 0 (by VALUE; -0.0 counts as zero), symmetrised (a_ij != 0 or a_ji != 0)
// because the paper assumes symmetry "for simplicity".
// ---------------------------------------------------------------------------
static Graph adjacency(const Csr& A) {
  std::vector<std::set<int>> s(A.n);
  for (int i = 0; i < A.n; ++i)
    for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e) {
      int j = A.col[e];
      if (j != i && A.val[e] != 0.0) { s[i].insert(j); s[j].insert(i); }
    }
  Graph g(A.n);
  for (int i = 0; i < A.n; ++i) g[i].assign(s[i].begin(), s[i].end());
  return g;
}

// Cell graph of the block system: edge iff block (c,d) or (d,c) has a nonzero entry.
static Graph cell_graph(const Bsr& A) {
  std::vector<std::set<int>> s(A.n);
  const int bb = A.b * A.b;
  for (int c = 0; c < A.n; ++c)
    for (int e = A.ptr[c]; e < A.ptr[c + 1]; ++e) {
      int d = A.col[e];
      if (d == c) continue;
      bool nz = false;
      for (int t = 0; t < bb; ++t) if (A.blk(e)[t] != 0.0) nz = true;
      if (nz) { s[c].insert(d); s[d].insert(c); }
    }
  Graph g(A.n);
  for (int c = 0; c < A.n; ++c) g[c].assign(s[c].begin(), s[c].end());
  return g;
}

// ---------------------------------------------------------------------------
// c-4: Alg. 2 VerticesSplitting and Alg. 3 VerticesGrouping
// with the readings of SURVEY c-4 / DESIGN.md R7:
//  - "Any take v_i with |S_i| >= |S_j|": maximum STATIC degree |S_i| (full
//    graph), lowest index on ties;
//  - S̄_i / Ŝ_i restricted to undetermined vertices (those still in V);
//  - W_i (Table 1) = union over k in S_i of S_k, minus S_i ∪ {i};
//  - line 406 moves only the undetermined neighbours S_i ∩ V into W̄;
//  - Ŵ is reset per Alg. 2 call (line 391).
// Followed literally, including stale Ŵ entries (handled by the else branch).
// ---------------------------------------------------------------------------
static void vertices_splitting(const Graph& S, const std::vector<int>& deg,
                               const std::vector<int>& Vin, std::vector<int>& Wout,
                               std::vector<int>& Wbar_out) {
  const int n = (int)S.size();
  using Key = std::pair<int, int>;              // (-|S_i|, i): begin() = max degree, lowest index
  std::set<Key> V, What;
  std::vector<char> inV(n, 0), inW(n, 0), inWbar(n, 0);
  for (int v : Vin) { V.insert({-deg[v], v}); inV[v] = 1; }
  std::vector<int> W, Wbar;                     // line 1
  while (!V.empty()) {                          // line 2
    int vi;
    if (!What.empty()) vi = What.begin()->second;   // lines 3-4
    else vi = V.begin()->second;                    // lines 5-6
    bool connected = false;                     // line 8
    for (int j : S[vi]) if (inW[j]) { connected = true; break; }
    if (!connected) {
      W.push_back(vi); inW[vi] = 1;             // line 9
      V.erase({-deg[vi], vi}); inV[vi] = 0;
      What.erase({-deg[vi], vi});               // lines 10-12
      for (int j : S[vi])                       // line 13: W̄ ∪= S̄_i, V \= S_i
        if (inV[j]) {
          if (!inWbar[j]) { Wbar.push_back(j); inWbar[j] = 1; }
          V.erase({-deg[j], j}); inV[j] = 0;
        }
      for (int k : S[vi])                       // line 13: Ŵ ∪= Ŝ_i (second circle, undetermined)
        for (int j : S[k]) {
          if (j == vi) continue;
          if (std::binary_search(S[vi].begin(), S[vi].end(), j)) continue;
          if (inV[j]) What.insert({-deg[j], j});
        }
    } else {
      if (!inWbar[vi]) { Wbar.push_back(vi); inWbar[vi] = 1; }   // line 15
      V.erase({-deg[vi], vi}); inV[vi] = 0;
      What.erase({-deg[vi], vi});               // lines 16-18
    }
  }
  std::sort(W.begin(), W.end());
  std::sort(Wbar.begin(), Wbar.end());
  Wout = W;
  Wbar_out = Wbar;
}

// Alg. 3: returns groups V_1..V_g (creation order), each ascending.
static std::vector<std::vector<int>> vertices_grouping(const Graph& S) {
  const int n = (int)S.size();
  std::vector<int> deg(n);
  for (int i = 0; i < n; ++i) deg[i] = (int)S[i].size();
  std::vector<int> V(n);
  for (int i = 0; i < n; ++i) V[i] = i;
  std::vector<std::vector<int>> groups;
  while (!V.empty()) {
    std::vector<int> W, Wbar;
    vertices_splitting(S, deg, V, W, Wbar);
    groups.push_back(W);
    V = Wbar;
  }
  return groups;
}

// ---------------------------------------------------------------------------
// c-6: PGS-MC sweep, Alg. 4: for each group V_l in order (ascending
// for the pre-sweep, descending for the post-sweep), update every row of the
// group: x_i <- (b_i - sum_{j != i} a_ij x_j) / a_ii.  Rows of one group are
// independent (A_l diagonal), so this sequential loop is the parallel
// result exactly.
// ---------------------------------------------------------------------------
static bool pgs_mc_sweep(const Csr& A, const std::vector<std::vector<int>>& groups,
                         const double* b, double* x, bool ascending) {
  const int g = (int)groups.size();
  for (int t = 0; t < g; ++t) {
    const std::vector<int>& Vl = groups[ascending ? t : g - 1 - t];
    int bad = -1;
    ORC_PAR
    for (size_t k = 0; k < Vl.size(); ++k) {        // rows of one color: independent
      const int i = Vl[k];
      double s = 0.0, d = 0.0;
      for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e) {
        if (A.col[e] == i) d = A.val[e];
        else s += A.val[e] * x[A.col[e]];
      }
      if (d == 0.0) {
#pragma omp critical
        bad = std::max(bad, i);
        continue;
      }
      x[i] = (b[i] - s) / d;
    }
    if (bad >= 0) { g_err = "pgs_mc: zero diagonal at row " + std::to_string(bad); return false; }
  }
  return true;
}

// ---------------------------------------------------------------------------
// NEXT-4 comparison smoothers (Table 2: "parallel GS and Jacobi methods based
// on natural ordering, denoted as PGS-NO and PJAC-NO"; reading R13 in DESIGN.md).
// PJAC-NO: one undamped Jacobi sweep, x_i <- (b_i - sum_{j != i} a_ij x_j^old) / a_ii.
// PGS-NO: the hybrid Jacobi/GS of P:318 ("combines the Jacobi and GS methods"): the
// natural-order rows are cut into chunks of K consecutive rows (one per parallel
// worker); inside a chunk rows are relaxed in order (ascending for the pre-sweep,
// descending for the post-sweep) with the newest values of the chunk, while every
// coupling to another chunk uses the value from the start of the sweep.  K = 1 is
// Jacobi, K >= n is sequential natural-order GS.
// ---------------------------------------------------------------------------
static bool jacobi_sweep(const Csr& A, const double* b, double* x) {
  std::vector<double> xo(x, x + A.n);
  for (int i = 0; i < A.n; ++i) {
    double s = 0.0, d = 0.0;
    for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e) {
      if (A.col[e] == i) d = A.val[e];
      else s += A.val[e] * xo[A.col[e]];
    }
    if (d == 0.0) { g_err = "jacobi: zero diagonal at row " + std::to_string(i); return false; }
    x[i] = (b[i] - s) / d;
  }
  return true;
}

static bool hybrid_gs_sweep(const Csr& A, int K, const double* b, double* x, bool ascending) {
  if (K < 1) { g_err = "hybrid_gs: chunk < 1"; return false; }
  std::vector<double> xo(x, x + A.n);       // values at the start of the sweep
  const int nchunk = (A.n + K - 1) / K;
  for (int c = 0; c < nchunk; ++c) {
    const int q0 = c * K, q1 = std::min(A.n, q0 + K);
    for (int t = 0; t < q1 - q0; ++t) {
      const int i = ascending ? q0 + t : q1 - 1 - t;
      double s = 0.0, d = 0.0;
      for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e) {
        const int j = A.col[e];
        if (j == i) { d = A.val[e]; continue; }
        const bool fresh = (j >= q0 && j < q1) && (ascending ? j < i : j > i);
        s += A.val[e] * (fresh ? x[j] : xo[j]);
      }
      if (d == 0.0) { g_err = "hybrid_gs: zero diagonal at row " + std::to_string(i); return false; }
      x[i] = (b[i] - s) / d;
    }
  }
  return true;
}

// ---------------------------------------------------------------------------
// c-5: NPAIR pairwise aggregation (P:459 names NPAIR [Napov-Notay] only; reading
// from SPEC S:304/S:344, R3).  Neighbours from the c-3 graph; strength
// via t_ij = a_ij + a_ji (s_ij = -t_ij/2).  Repeatedly take the unaggregated row
// with the fewest unaggregated neighbours (lowest index on ties); pair it with
// the unaggregated neighbour of maximal s_ij > 0 (minimal t < 0; lowest j on
// ties), else with the one of maximal |t| (lowest j), else singleton.
// ---------------------------------------------------------------------------
static double entry(const Csr& A, int i, int j) {
  auto b = A.col.begin() + A.ptr[i], e = A.col.begin() + A.ptr[i + 1];
  auto it = std::lower_bound(b, e, j);
  if (it != e && *it == j) return A.val[it - A.col.begin()];
  return 0.0;
}

static int npair(const Csr& A, std::vector<int>& agg) {
  const int n = A.n;
  Graph S = adjacency(A);
  std::vector<int> cnt(n);
  std::set<std::pair<int, int>> Q;
  for (int i = 0; i < n; ++i) { cnt[i] = (int)S[i].size(); Q.insert({cnt[i], i}); }
  std::vector<char> done(n, 0);
  agg.assign(n, -1);
  int nagg = 0;
  auto dec = [&](int m) {
    for (int k : S[m])
      if (!done[k]) { Q.erase({cnt[k], k}); --cnt[k]; Q.insert({cnt[k], k}); }
  };
  while (!Q.empty()) {
    int i = Q.begin()->second;
    Q.erase(Q.begin());
    int best = -1;
    double bt = 0.0;
    for (int j : S[i]) {
      if (done[j]) continue;
      double t = entry(A, i, j) + entry(A, j, i);
      if (t < bt) { bt = t; best = j; }
    }
    if (best < 0) {
      double ba = -1.0;
      for (int j : S[i]) {
        if (done[j]) continue;
        double a = std::fabs(entry(A, i, j) + entry(A, j, i));
        if (a > ba) { ba = a; best = j; }
      }
    }
    done[i] = 1;
    agg[i] = nagg;
    if (best >= 0) { Q.erase({cnt[best], best}); done[best] = 1; agg[best] = nagg; }
    ++nagg;
    dec(i);
    if (best >= 0) dec(best);
  }
  return nagg;
}

// Galerkin coarse operator A_c = P^T A P for the piecewise-constant P of an
// aggregation (UA-AMG): A_c[I,J] = sum_{i in I} sum_{j in J} a_ij, summed
// in the order (I ascending; members i ascending; stored j ascending), each slot
// starting from +0.0.  Pattern = structural union (explicit zeros kept).
static Csr galerkin(const Csr& A, const std::vector<int>& agg, int nagg) {
  std::vector<std::vector<int>> mem(nagg);
  for (int i = 0; i < A.n; ++i) mem[agg[i]].push_back(i);
  Csr C;
  C.n = nagg;
  C.ptr.push_back(0);
  for (int I = 0; I < nagg; ++I) {
    std::map<int, double> row;
    for (int i : mem[I])
      for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e) {
        int J = agg[A.col[e]];
        if (!row.count(J)) row[J] = 0.0;
        row[J] += A.val[e];
      }
    for (auto& kv : row) { C.col.push_back(kv.first); C.val.push_back(kv.second); }
    C.ptr.push_back((int)C.col.size());
  }
  return C;
}

static bool is_diagonal(const Csr& A) {
  for (int i = 0; i < A.n; ++i)
    for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e)
      if (A.col[e] != i && A.val[e] != 0.0) return false;
  return true;
}

// ---------------------------------------------------------------------------
// Dense LU with partial pivoting: the coarsest "direct solver".
// ---------------------------------------------------------------------------
struct DenseLU {
  int n = 0;
  std::vector<double> a;      // row-major, L (unit) and U
  std::vector<int> piv;
  bool factor(const Csr& A) {
    n = A.n;
    a.assign((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i)
      for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e) a[(size_t)i * n + A.col[e]] = A.val[e];
    return factor_dense();
  }
  bool factor_dense() {
    piv.resize(n);
    for (int k = 0; k < n; ++k) {
      int p = k;
      double m = std::fabs(a[(size_t)k * n + k]);
      for (int i = k + 1; i < n; ++i)
        if (std::fabs(a[(size_t)i * n + k]) > m) { m = std::fabs(a[(size_t)i * n + k]); p = i; }
      if (m == 0.0) { g_err = "dense LU: singular at column " + std::to_string(k); return false; }
      piv[k] = p;
      if (p != k)
        for (int j = 0; j < n; ++j) std::swap(a[(size_t)k * n + j], a[(size_t)p * n + j]);
      const double* rk = &a[(size_t)k * n];
      for (int i = k + 1; i < n; ++i) {
        double* ri = &a[(size_t)i * n];
        double f = ri[k] / rk[k];
        ri[k] = f;
        if (f != 0.0)
          for (int j = k + 1; j < n; ++j) ri[j] -= f * rk[j];
      }
    }
    return true;
  }
  void solve(const double* b, double* x) const {
    std::vector<double> y(b, b + n);
    for (int k = 0; k < n; ++k) std::swap(y[k], y[piv[k]]);
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int j = 0; j < i; ++j) s += a[(size_t)i * n + j] * y[j];
      y[i] -= s;
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = 0.0;
      for (int j = i + 1; j < n; ++j) s += a[(size_t)i * n + j] * y[j];
      y[i] = (y[i] - s) / a[(size_t)i * n + i];
    }
    for (int i = 0; i < n; ++i) x[i] = y[i];
  }
};

// Small dense helpers for b x b blocks (row-major).
static void blk_mul(int b, const double* X, const double* Y, double* Z) {   // Z = X*Y
  for (int i = 0; i < b; ++i)
    for (int j = 0; j < b; ++j) {
      double s = 0.0;
      for (int k = 0; k < b; ++k) s += X[i * b + k] * Y[k * b + j];
      Z[i * b + j] = s;
    }
}
// Gauss-Jordan inverse with partial pivoting. returns false if singular.
static bool blk_inv(int b, const double* D, double* Dinv) {
  std::vector<double> a(D, D + b * b), r(b * b, 0.0);
  for (int i = 0; i < b; ++i) r[i * b + i] = 1.0;
  for (int k = 0; k < b; ++k) {
    int p = k;
    for (int i = k + 1; i < b; ++i) if (std::fabs(a[i * b + k]) > std::fabs(a[p * b + k])) p = i;
    if (a[p * b + k] == 0.0) return false;
    for (int j = 0; j < b; ++j) { std::swap(a[k * b + j], a[p * b + j]); std::swap(r[k * b + j], r[p * b + j]); }
    double piv = a[k * b + k];
    for (int j = 0; j < b; ++j) { a[k * b + j] /= piv; r[k * b + j] /= piv; }
    for (int i = 0; i < b; ++i) {
      if (i == k) continue;
      double f = a[i * b + k];
      for (int j = 0; j < b; ++j) { a[i * b + j] -= f * a[k * b + j]; r[i * b + j] -= f * r[k * b + j]; }
    }
  }
  std::copy(r.begin(), r.end(), Dinv);
  return true;
}

// ---------------------------------------------------------------------------
// Configuration (mirrors the product's msp_config fields, own definition).
// ---------------------------------------------------------------------------
struct Config {
  int coarsest_max_dof = 10000;
  int max_levels = 20;
  int pre_sweeps = 1, post_sweeps = 1;
  int pair_passes = 2;           // R3
  int decoupling = 2;            // 0 NONE, 1 QI, 2 TI (R4)
  int bilu_order = 1;            // 0 RB, 1 ABMC1 (R5)
  int stages = 2;                // 2 = PR (north_star), 3 = NPR (Eq. 21 full)
  int orth = 0;                  // 0 CGS2 (R8, default: the textbook reference), 1 MGS, 2 DCGS2 (R14)
  int smoother = 0;              // 0 PGS-MC (Alg. 4), 1 PJAC-NO, 2 PGS-NO (R13)
  int gs_chunk = 32;             // PGS-NO chunk size K (R13)
};

// ---------------------------------------------------------------------------
// c-2: decoupling weights W and pressure matrix A_PP (R4; Π_P of P:254).
// TI: C_c = sum_p A[p,c] (block column sum, ascending p); w_c = [1, y] with
// C_NN^T y = -C_0N^T solved by Gaussian elimination with partial pivoting
// (first maximal |pivot|), no FMA, back-substitution sums ascending from 0.0.
// QI: same with the diagonal block D_c.  NONE: w_c = e_0 (paper-literal Π_P).
// A_PP[c,d] = sum_{k=0}^{b-1} w_c[k] * A[c,d][k][0], ascending k from +0.0.
// ---------------------------------------------------------------------------
static bool solve_weights(int nc, const double* C /* b x b row-major */, double* y) {
  const int b = nc + 1;
  std::vector<double> M(nc * nc), r(nc);
  for (int i = 0; i < nc; ++i) {
    for (int j = 0; j < nc; ++j) M[i * nc + j] = C[(1 + j) * b + (1 + i)];   // (C_NN)^T
    r[i] = -C[0 * b + (1 + i)];                                             // -(C_0N)^T
  }
  for (int k = 0; k < nc; ++k) {
    int p = k;
    for (int i = k + 1; i < nc; ++i) if (std::fabs(M[i * nc + k]) > std::fabs(M[p * nc + k])) p = i;
    if (M[p * nc + k] == 0.0) return false;
    if (p != k) {
      for (int j = 0; j < nc; ++j) std::swap(M[k * nc + j], M[p * nc + j]);
      std::swap(r[k], r[p]);
    }
    for (int i = k + 1; i < nc; ++i) {
      double f = M[i * nc + k] / M[k * nc + k];
      for (int j = k + 1; j < nc; ++j) M[i * nc + j] = M[i * nc + j] - f * M[k * nc + j];
      r[i] = r[i] - f * r[k];
    }
  }
  for (int i = nc - 1; i >= 0; --i) {
    double s = 0.0;
    for (int j = i + 1; j < nc; ++j) s = s + M[i * nc + j] * y[j];
    y[i] = (r[i] - s) / M[i * nc + i];
  }
  return true;
}

static bool decoupling_weights(const Bsr& A, int mode, std::vector<double>& W) {
  const int n = A.n, b = A.b, bb = b * b, nc = b - 1;
  W.assign((size_t)n * b, 0.0);
  if (mode == 0) {
    for (int c = 0; c < n; ++c) W[(size_t)c * b] = 1.0;
    return true;
  }
  std::vector<double> C((size_t)n * bb, 0.0);
  if (mode == 2) {
    // block column sums, p ascending: iterate rows p ascending, add into column c
    for (int p = 0; p < n; ++p)
      for (int e = A.ptr[p]; e < A.ptr[p + 1]; ++e) {
        int c = A.col[e];
        for (int t = 0; t < bb; ++t) C[(size_t)c * bb + t] += A.blk(e)[t];
      }
  } else {
    for (int c = 0; c < n; ++c)
      for (int e = A.ptr[c]; e < A.ptr[c + 1]; ++e)
        if (A.col[e] == c)
          for (int t = 0; t < bb; ++t) C[(size_t)c * bb + t] = A.blk(e)[t];
  }
  std::vector<double> y(nc);
  for (int c = 0; c < n; ++c) {
    if (!solve_weights(nc, &C[(size_t)c * bb], y.data())) {
      g_err = "decoupling: singular N-N block at cell " + std::to_string(c);
      return false;
    }
    W[(size_t)c * b] = 1.0;
    for (int i = 0; i < nc; ++i) W[(size_t)c * b + 1 + i] = y[i];
  }
  return true;
}

static Csr extract_app(const Bsr& A, const std::vector<double>& W) {
  const int b = A.b;
  Csr P;
  P.n = A.n;
  P.ptr = A.ptr;
  P.col = A.col;
  P.val.resize(A.col.size());
  for (int c = 0; c < A.n; ++c)
    for (int e = A.ptr[c]; e < A.ptr[c + 1]; ++e) {
      double s = 0.0;
      for (int k = 0; k < b; ++k) s = s + W[(size_t)c * b + k] * A.blk(e)[k * b + 0];
      P.val[e] = s;
    }
  return P;
}

// ---------------------------------------------------------------------------
// AMG hierarchy (UA-AMG, NPAIR, V-cycle, PGS-MC smoother, direct coarsest).
// ---------------------------------------------------------------------------
struct Level {
  Csr A;
  std::vector<std::vector<int>> groups;   // PGS-MC colors of A (Alg. 3)
  std::vector<int> agg;                   // composite aggregate of each row (next level row)
  std::vector<std::vector<int>> pass_agg; // per pass
  int n_next = 0;
};

struct Hierarchy {
  std::vector<Level> lv;                  // smoothing levels 0..L-1
  Csr Ac;                                 // coarsest matrix A_L
  bool coarse_diag = false;
  DenseLU lu;
};

// pair_passes NPAIR passes; returns composite agg and the final Galerkin matrix.
static int multi_pass_aggregate(const Csr& A, int passes, std::vector<int>& agg,
                                std::vector<std::vector<int>>* pass_agg, Csr* Anext) {
  Csr cur = A;
  agg.resize(A.n);
  for (int i = 0; i < A.n; ++i) agg[i] = i;
  int nagg = A.n;
  for (int p = 0; p < passes; ++p) {
    std::vector<int> a;
    nagg = npair(cur, a);
    if (pass_agg) pass_agg->push_back(a);
    for (int i = 0; i < A.n; ++i) agg[i] = a[agg[i]];
    cur = galerkin(cur, a, nagg);
  }
  if (Anext) *Anext = cur;
  return nagg;
}

static int build_hierarchy(const Csr& A0, const Config& cfg, Hierarchy& H) {
  Csr A = A0;
  H.lv.clear();
  for (int l = 0;; ++l) {
    if (A.n <= cfg.coarsest_max_dof) break;
    if (l + 1 >= cfg.max_levels) { g_err = "AMG: max_levels reached above coarsest_max_dof"; return 5; }
    Level L;
    Csr An;
    int nn = multi_pass_aggregate(A, cfg.pair_passes, L.agg, &L.pass_agg, &An);
    if ((double)nn > 0.9 * (double)A.n) {
      if (is_diagonal(A)) { H.coarse_diag = true; break; }
      g_err = "AMG: coarsening stalled at level " + std::to_string(l);
      return 5;
    }
    L.A = A;
    L.groups = vertices_grouping(adjacency(A));
    L.n_next = nn;
    H.lv.push_back(std::move(L));
    A = std::move(An);
  }
  H.Ac = A;
  if (!H.coarse_diag) {
    if (!H.lu.factor(A)) return 2;
  } else {
    for (int i = 0; i < A.n; ++i)
      if (entry(A, i, i) == 0.0) { g_err = "coarsest diagonal zero"; return 2; }
  }
  return 0;
}

static void coarse_solve(const Hierarchy& H, const double* b, double* x) {
  if (H.coarse_diag) {
    for (int i = 0; i < H.Ac.n; ++i) x[i] = b[i] / entry(H.Ac, i, i);
  } else {
    H.lu.solve(b, x);
  }
}

// one smoothing sweep of level L with the configured smoother (pre: ascending)
static bool smooth(const Level& L, const Config& cfg, const double* b, double* x, bool pre) {
  if (cfg.smoother == 1) return jacobi_sweep(L.A, b, x);
  if (cfg.smoother == 2) return hybrid_gs_sweep(L.A, cfg.gs_chunk, b, x, pre);
  return pgs_mc_sweep(L.A, L.groups, b, x, pre);
}

// a5: residual and restriction r_{l+1}[I] = sum_{i in I} (b_i - (A_l x)_i) (P^T with the
// piecewise-constant UA-AMG prolongation P): the residual of every row,
// then the members of each aggregate summed in ascending row order (from +0.0).
static void residual_restrict(const Level& L, const double* b, const double* x, double* bc) {
  const int n = L.A.n;
  std::vector<double> Ax(n);
  csr_spmv(L.A, x, Ax.data());
  for (int I = 0; I < L.n_next; ++I) bc[I] = 0.0;
  for (int i = 0; i < n; ++i) bc[L.agg[i]] += b[i] - Ax[i];
}

// a7: prolongation and correction x_i += e[agg(i)] (P e, P piecewise constant).
static void prolong_correct(const Level& L, const double* e, double* x) {
  for (int i = 0; i < L.A.n; ++i) x[i] += e[L.agg[i]];
}

// c-7: V-cycle from zero initial guess: pre-smooth (colors ascending), restrict
// r_{l+1} = P^T (b - A x), recurse, x += P e, post-smooth (colors descending).
static bool vcycle(const Hierarchy& H, const Config& cfg, int l, const std::vector<double>& b,
                   std::vector<double>& x) {
  if (l == (int)H.lv.size()) {
    x.assign(H.Ac.n, 0.0);
    coarse_solve(H, b.data(), x.data());
    return true;
  }
  const Level& L = H.lv[l];
  const int n = L.A.n;
  x.assign(n, 0.0);
  for (int s = 0; s < cfg.pre_sweeps; ++s)
    if (!smooth(L, cfg, b.data(), x.data(), true)) return false;
  std::vector<double> bc(L.n_next, 0.0);
  residual_restrict(L, b.data(), x.data(), bc.data());
  std::vector<double> e;
  if (!vcycle(H, cfg, l + 1, bc, e)) return false;
  prolong_correct(L, e.data(), x.data());
  for (int s = 0; s < cfg.post_sweeps; ++s)
    if (!smooth(L, cfg, b.data(), x.data(), false)) return false;
  return true;
}

// ---------------------------------------------------------------------------
// c-9: BILU(0) (R = "Block ILU (BILU)") in aggregate-block multicolor
// (ABMC) order (R5).  Blocks = pair_passes-pass NPAIR aggregates of A_PP (the
// level-1 aggregates); quotient of the cell graph colored by Alg. 2/3; cells
// ordered by (block color, block id, cell id).  RB: Alg. 2/3 on the cell graph,
// order (color, cell id).  Factorization: block IKJ ILU(0) over A's pattern.
// ---------------------------------------------------------------------------
static Csr cell_laplacian(const Graph& G) {
  Csr L;
  L.n = (int)G.size();
  L.ptr.push_back(0);
  for (int c = 0; c < L.n; ++c) {
    bool diag_done = false;
    for (int d : G[c]) {
      if (!diag_done && d > c) { L.col.push_back(c); L.val.push_back((double)G[c].size()); diag_done = true; }
      L.col.push_back(d); L.val.push_back(-1.0);
    }
    if (!diag_done) { L.col.push_back(c); L.val.push_back((double)G[c].size()); }
    L.ptr.push_back((int)L.col.size());
  }
  return L;
}

static std::vector<int> bilu_ordering(const Bsr& A, const Csr& App, const Config& cfg,
                                      std::vector<int>& color, std::vector<int>& blk) {
  const int n = A.n;
  Graph G = cell_graph(A);
  color.assign(n, 0);
  blk.assign(n, 0);
  if (cfg.bilu_order == 0) {
    auto groups = vertices_grouping(G);
    for (size_t g = 0; g < groups.size(); ++g) for (int c : groups[g]) color[c] = (int)g;
    for (int c = 0; c < n; ++c) blk[c] = c;
  } else {
    std::vector<int> agg;
    int nb;
    if (is_diagonal(App)) nb = multi_pass_aggregate(cell_laplacian(G), cfg.pair_passes, agg, nullptr, nullptr);
    else nb = multi_pass_aggregate(App, cfg.pair_passes, agg, nullptr, nullptr);
    std::vector<std::set<int>> q(nb);
    for (int c = 0; c < n; ++c)
      for (int d : G[c])
        if (agg[c] != agg[d]) { q[agg[c]].insert(agg[d]); q[agg[d]].insert(agg[c]); }
    Graph Q(nb);
    for (int I = 0; I < nb; ++I) Q[I].assign(q[I].begin(), q[I].end());
    auto groups = vertices_grouping(Q);
    std::vector<int> bcol(nb);
    for (size_t g = 0; g < groups.size(); ++g) for (int I : groups[g]) bcol[I] = (int)g;
    for (int c = 0; c < n; ++c) { color[c] = bcol[agg[c]]; blk[c] = agg[c]; }
  }
  std::vector<int> order(n);
  for (int c = 0; c < n; ++c) order[c] = c;
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    if (color[a] != color[b]) return color[a] < color[b];
    if (blk[a] != blk[b]) return blk[a] < blk[b];
    return a < b;
  });
  return order;
}

struct Bilu {
  std::vector<int> order, pos;
  std::vector<int> color, blk;  // block color and ABMC block (aggregate) of every cell
  Bsr F;                       // factors in A's (natural) storage: L_ik (k before i), U_ij (j after i)
  std::vector<double> Dinv;    // n * b*b
  std::vector<std::vector<int>> rowe;   // entries of row i sorted by position of column
};

static int find_entry(const Bsr& A, int i, int j) {
  auto b = A.col.begin() + A.ptr[i], e = A.col.begin() + A.ptr[i + 1];
  auto it = std::lower_bound(b, e, j);
  if (it != e && *it == j) return (int)(it - A.col.begin());
  return -1;
}

static bool bilu_factor(const Bsr& A, const std::vector<int>& order, Bilu& R) {
  const int n = A.n, b = A.b, bb = b * b;
  R.order = order;
  R.pos.assign(n, 0);
  for (int p = 0; p < n; ++p) R.pos[order[p]] = p;
  R.F = A;
  R.Dinv.assign((size_t)n * bb, 0.0);
  R.rowe.assign(n, {});
  for (int i = 0; i < n; ++i) {
    for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e) R.rowe[i].push_back(e);
    std::sort(R.rowe[i].begin(), R.rowe[i].end(),
              [&](int x, int y) { return R.pos[A.col[x]] < R.pos[A.col[y]]; });
  }
  std::vector<double> T(bb), T2(bb);
  for (int p = 0; p < n; ++p) {
    const int i = order[p];
    const auto& ents = R.rowe[i];
    for (size_t a = 0; a < ents.size(); ++a) {
      const int ek = ents[a], k = A.col[ek];
      if (R.pos[k] >= p) break;
      blk_mul(b, R.F.blk(ek), &R.Dinv[(size_t)k * bb], T.data());     // A_ik <- A_ik * D~_k^-1
      std::copy(T.begin(), T.end(), R.F.blk(ek));
      for (size_t c = a + 1; c < ents.size(); ++c) {
        const int ej = ents[c], j = A.col[ej];
        const int ekj = find_entry(A, k, j);
        if (ekj < 0) continue;                                          // ILU(0): no fill
        blk_mul(b, R.F.blk(ek), R.F.blk(ekj), T2.data());               // A_ij -= A_ik * A_kj
        for (int t = 0; t < bb; ++t) R.F.blk(ej)[t] -= T2[t];
      }
    }
    const int ed = find_entry(A, i, i);
    if (ed < 0 || !blk_inv(b, R.F.blk(ed), &R.Dinv[(size_t)i * bb])) {
      g_err = "BILU: singular pivot block at cell " + std::to_string(i);
      return false;
    }
  }
  return true;
}

// Alg. 1 line 6 (R r) with the BILU(0) factors, sequentially in the elimination order:
// forward  y_i = r_i - sum_{k before i} L_ik y_k                 (positions ascending)
// backward x_i = D~_i^-1 (y_i - sum_{j after i} U_ij x_j)        (positions descending)
// Sums run over row i's entries sorted by position, components ascending, from +0.0.
// absmode: the same recurrences on |L|, |U|, |D~^-1| and |inputs| with every minus a
// plus -- the componentwise magnitude bounds (I - |N|)^-1 |r| used by the parity tests.
static void bilu_forward(const Bilu& R, const double* r, double* y, bool absmode = false) {
  const Bsr& F = R.F;
  const int n = F.n, b = F.b;
  for (int p = 0; p < n; ++p) {
    const int i = R.order[p];
    for (int q = 0; q < b; ++q) {
      double s = 0.0;
      for (int e : R.rowe[i]) {
        const int k = F.col[e];
        if (R.pos[k] >= p) break;
        for (int t = 0; t < b; ++t) {
          const double f = F.blk(e)[q * b + t];
          s += (absmode ? std::fabs(f) : f) * y[(size_t)k * b + t];
        }
      }
      const double ri = r[(size_t)i * b + q];
      y[(size_t)i * b + q] = absmode ? std::fabs(ri) + s : ri - s;
    }
  }
}

static void bilu_backward(const Bilu& R, const double* y, double* x, bool absmode = false) {
  const Bsr& F = R.F;
  const int n = F.n, b = F.b, bb = b * b;
  std::vector<double> t(b);
  for (int p = n - 1; p >= 0; --p) {
    const int i = R.order[p];
    for (int q = 0; q < b; ++q) {
      double s = 0.0;
      for (int e : R.rowe[i]) {
        const int j = F.col[e];
        if (R.pos[j] <= p) continue;
        for (int u = 0; u < b; ++u) {
          const double f = F.blk(e)[q * b + u];
          s += (absmode ? std::fabs(f) : f) * x[(size_t)j * b + u];
        }
      }
      const double yi = y[(size_t)i * b + q];
      t[q] = absmode ? std::fabs(yi) + s : yi - s;
    }
    for (int q = 0; q < b; ++q) {
      double s = 0.0;
      for (int u = 0; u < b; ++u) {
        const double d = R.Dinv[(size_t)i * bb + q * b + u];
        s += (absmode ? std::fabs(d) : d) * t[u];
      }
      x[(size_t)i * b + q] = s;
    }
  }
}

static void bilu_apply_omp(const Bilu& R, const double* r, double* x);

static void bilu_apply(const Bilu& R, const double* r, double* x) {
  if (g_threads > 1) { bilu_apply_omp(R, r, x); return; }
  std::vector<double> y((size_t)R.F.n * R.F.b);
  bilu_forward(R, r, y.data());
  bilu_backward(R, y.data(), x);
}

// The same substitutions executed "in parallel by color" (P:258 with the block multicolor
// reading R5, P:434's independence argument): every cell of block color c reads the
// values of OTHER blocks from a snapshot taken before color c starts (colors < c final
// in the forward phase, > c in the backward phase) and only its own block's cells
// live, in order.  Identical summation order to bilu_forward/backward, so the result
// is bit-identical to the sequential one exactly when same-color blocks are uncoupled.
static void bilu_apply_by_color(const Bilu& R, const double* r, double* x) {
  const Bsr& F = R.F;
  const int n = F.n, b = F.b, bb = b * b;
  int g = 0;
  for (int c = 0; c < n; ++c) g = std::max(g, R.color[c] + 1);
  std::vector<double> y((size_t)n * b, 0.0), snap;
  for (int col = 0; col < g; ++col) {
    snap = y;
    for (int p = 0; p < n; ++p) {
      const int i = R.order[p];
      if (R.color[i] != col) continue;
      for (int q = 0; q < b; ++q) {
        double s = 0.0;
        for (int e : R.rowe[i]) {
          const int k = F.col[e];
          if (R.pos[k] >= p) break;
          const double* src = (R.blk[k] == R.blk[i]) ? y.data() : snap.data();
          for (int t = 0; t < b; ++t) s += F.blk(e)[q * b + t] * src[(size_t)k * b + t];
        }
        y[(size_t)i * b + q] = r[(size_t)i * b + q] - s;
      }
    }
  }
  std::vector<double> xv((size_t)n * b, 0.0), t(b);
  for (int col = g - 1; col >= 0; --col) {
    snap = xv;
    for (int p = n - 1; p >= 0; --p) {
      const int i = R.order[p];
      if (R.color[i] != col) continue;
      for (int q = 0; q < b; ++q) {
        double s = 0.0;
        for (int e : R.rowe[i]) {
          const int j = F.col[e];
          if (R.pos[j] <= p) continue;
          const double* src = (R.blk[j] == R.blk[i]) ? xv.data() : snap.data();
          for (int u = 0; u < b; ++u) s += F.blk(e)[q * b + u] * src[(size_t)j * b + u];
        }
        t[q] = y[(size_t)i * b + q] - s;
      }
      for (int q = 0; q < b; ++q) {
        double s = 0.0;
        for (int u = 0; u < b; ++u) s += R.Dinv[(size_t)i * bb + q * b + u] * t[u];
        xv[(size_t)i * b + q] = s;
      }
    }
  }
  std::copy(xv.begin(), xv.end(), x);
}

// OMP timing mode of bilu_apply: the blocks of one color in parallel (their cells in
// order), every sum in the sequential order -- bit-identical to bilu_forward/backward
// because same-color blocks are uncoupled (ABMC validity, pinned by
// test_abmc_order_validity_bruteforce / test_bilu_parallel_by_color_equals_sequential).
static void bilu_apply_omp(const Bilu& R, const double* r, double* x) {
  const Bsr& F = R.F;
  const int n = F.n, b = F.b, bb = b * b;
  std::vector<int> run;                      // position ranges of the blocks, in order
  std::vector<int> color_run;                // first run of every color
  for (int p = 0; p < n; ++p) {
    const int i = R.order[p];
    if (p == 0 || R.blk[i] != R.blk[R.order[p - 1]]) {
      if (p == 0 || R.color[i] != R.color[R.order[p - 1]]) color_run.push_back((int)run.size());
      run.push_back(p);
    }
  }
  run.push_back(n);
  color_run.push_back((int)run.size() - 1);
  const int g = (int)color_run.size() - 1;
  std::vector<double> y((size_t)n * b);
  for (int c = 0; c < g; ++c) {
    ORC_PAR
    for (int k = color_run[c]; k < color_run[c + 1]; ++k)
      for (int p = run[k]; p < run[k + 1]; ++p) {
        const int i = R.order[p];
        for (int q = 0; q < b; ++q) {
          double s = 0.0;
          for (int e : R.rowe[i]) {
            const int kk = F.col[e];
            if (R.pos[kk] >= p) break;
            for (int t = 0; t < b; ++t) s += F.blk(e)[q * b + t] * y[(size_t)kk * b + t];
          }
          y[(size_t)i * b + q] = r[(size_t)i * b + q] - s;
        }
      }
  }
  for (int c = g - 1; c >= 0; --c) {
    ORC_PAR
    for (int k = color_run[c]; k < color_run[c + 1]; ++k) {
      std::vector<double> t(b);
      for (int p = run[k + 1] - 1; p >= run[k]; --p) {
        const int i = R.order[p];
        for (int q = 0; q < b; ++q) {
          double s = 0.0;
          for (int e : R.rowe[i]) {
            const int j = F.col[e];
            if (R.pos[j] <= p) continue;
            for (int u = 0; u < b; ++u) s += F.blk(e)[q * b + u] * x[(size_t)j * b + u];
          }
          t[q] = y[(size_t)i * b + q] - s;
        }
        for (int q = 0; q < b; ++q) {
          double s = 0.0;
          for (int u = 0; u < b; ++u) s += R.Dinv[(size_t)i * bb + q * b + u] * t[u];
          x[(size_t)i * b + q] = s;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// NEXT-1: B_N = block GS on A_NN = Π_N^T A Π_N (R12): one forward
// block Gauss-Seidel sweep from the zero guess over the nc x nc N-N blocks, in the
// BILU (ABMC) cell order of c-9: w_i = D_NN,i^-1 (r_N,i - sum_{k before i} A_NN,ik w_k).
// ---------------------------------------------------------------------------
struct Bgs {
  std::vector<double> Dinv;   // n * nc*nc inverse of the N-N diagonal block
};

// ---------------------------------------------------------------------------
// The MSP preconditioner (Eq. 21, Alg. 1).
// ---------------------------------------------------------------------------
struct Msp {
  Config cfg;
  Bsr A;
  std::vector<double> W;
  Csr App;
  Hierarchy H;
  Bilu R;
  Bgs N;
  int setup_calls = 0;
};

static int msp_setup(Msp& M) {
  if (!decoupling_weights(M.A, M.cfg.decoupling, M.W)) return 2;
  M.App = extract_app(M.A, M.W);
  int rc = build_hierarchy(M.App, M.cfg, M.H);
  if (rc) return rc;
  {
    std::vector<int> color, blk;
    std::vector<int> order = bilu_ordering(M.A, M.App, M.cfg, color, blk);
    if (!bilu_factor(M.A, order, M.R)) return 2;
    M.R.color = color;
    M.R.blk = blk;
  }
  if (M.cfg.stages == 3) {
    const int b = M.A.b, nc = b - 1;
    M.N.Dinv.assign((size_t)M.A.n * nc * nc, 0.0);
    std::vector<double> D(nc * nc);
    for (int c = 0; c < M.A.n; ++c) {
      int e = find_entry(M.A, c, c);
      for (int i = 0; i < nc; ++i)
        for (int j = 0; j < nc; ++j) D[i * nc + j] = M.A.blk(e)[(1 + i) * b + 1 + j];
      if (!blk_inv(nc, D.data(), &M.N.Dinv[(size_t)c * nc * nc])) {
        g_err = "BGS: singular N-N block at cell " + std::to_string(c);
        return 2;
      }
    }
  }
  M.setup_calls++;
  return 0;
}

// a3: decoupled pressure restriction r_p = W^T r (R4; Π_P^T of Alg. 1 line 4, with
// the decoupling weights in the middle factor): r_p[c] = sum_k w_c[k] r[c*b+k], k ascending.
static void restrict_pressure(const Msp& M, const double* r, double* rp) {
  const int b = M.A.b;
  ORC_PAR
  for (int c = 0; c < M.A.n; ++c) {
    double s = 0.0;
    for (int k = 0; k < b; ++k) s += M.W[(size_t)c * b + k] * r[(size_t)c * b + k];
    rp[c] = s;
  }
}

static bool pressure_stage(const Msp& M, const std::vector<double>& r, std::vector<double>& xp) {
  const int n = M.A.n;
  std::vector<double> rp(n);
  restrict_pressure(M, r.data(), rp.data());
  return vcycle(M.H, M.cfg, 0, rp, xp);
}

static void bgs_stage(const Msp& M, const std::vector<double>& r, std::vector<double>& wN) {
  // one forward block GS sweep on A_NN in the BILU cell order, zero initial guess
  const int n = M.A.n, b = M.A.b, nc = b - 1;
  wN.assign((size_t)n * nc, 0.0);
  std::vector<double> t(nc);
  for (int p = 0; p < n; ++p) {
    const int c = M.R.order[p];
    for (int i = 0; i < nc; ++i) {
      double s = 0.0;
      for (int e = M.A.ptr[c]; e < M.A.ptr[c + 1]; ++e) {
        const int d = M.A.col[e];
        if (M.R.pos[d] >= p) continue;        // only cells before c in the order
        for (int k = 0; k < nc; ++k) s += M.A.blk(e)[(1 + i) * b + 1 + k] * wN[(size_t)d * nc + k];
      }
      t[i] = r[(size_t)c * b + 1 + i] - s;
    }
    for (int i = 0; i < nc; ++i) {
      double s = 0.0;
      for (int k = 0; k < nc; ++k) s += M.N.Dinv[(size_t)c * nc * nc + i * nc + k] * t[k];
      wN[(size_t)c * nc + i] = s;
    }
  }
}

// Alg. 1 with w = 0 on entry (keeps B linear).  stages PR: lines 3-6;
// stages NPR: lines 1-6.
static bool msp_apply(const Msp& M, const double* g, double* wout) {
  const int n = M.A.n, b = M.A.b;
  const size_t N = (size_t)n * b;
  std::vector<double> w(N, 0.0), r(g, g + N), Aw(N);
  if (M.cfg.stages == 3) {
    std::vector<double> wN;
    bgs_stage(M, r, wN);                                 // line 2 (r = g since w = 0)
    for (int c = 0; c < n; ++c)
      for (int i = 0; i < b - 1; ++i) w[(size_t)c * b + 1 + i] += wN[(size_t)c * (b - 1) + i];
    bsr_spmv(M.A, w.data(), Aw.data());                  // line 3
    ORC_PAR
    for (size_t t = 0; t < N; ++t) r[t] = g[t] - Aw[t];
  }
  std::vector<double> xp;
  if (!pressure_stage(M, r, xp)) return false;         // line 4: w += Π_P B_P W^T r
  for (int c = 0; c < n; ++c) w[(size_t)c * b] += xp[c];
  bsr_spmv(M.A, w.data(), Aw.data());                  // line 5: r = g - A w
  ORC_PAR
  for (size_t t = 0; t < N; ++t) r[t] = g[t] - Aw[t];
  std::vector<double> z(N);
  bilu_apply(M.R, r.data(), z.data());                 // line 6: w += R r
  ORC_PAR
  for (size_t t = 0; t < N; ++t) wout[t] = w[t] + z[t];
  return true;
}

// ---------------------------------------------------------------------------
// c-11: restarted right-preconditioned GMRES(m), CGS2 or MGS,
// Givens rotations, convergence on ||b - A x|| / ||b|| <= tol; iterations
// counted as Arnoldi steps; history = |gamma_{j+1}|/||b|| per step, then the true
// relative residual at each cycle end.
// ---------------------------------------------------------------------------
struct GmresOut {
  int iters = 0;
  double final_rel = 0.0;
  int status = 0;    // 0 ok, 3 no convergence, 4 breakdown above tol
  std::vector<double> hist;
};

static GmresOut gmres(size_t N, const std::function<void(const double*, double*)>& Aop,
                      const std::function<bool(const double*, double*)>& Bop, const double* b,
                      double* x, double tol, int m, int maxit, int orth) {
  GmresOut out;
  std::vector<double> bv(b, b + N), r(N), t(N), z(N);
  const double bnorm = nrm2(bv);
  if (bnorm == 0.0) {
    for (size_t i = 0; i < N; ++i) x[i] = 0.0;
    return out;
  }
  Aop(x, t.data());
  ORC_PAR
  for (size_t i = 0; i < N; ++i) r[i] = b[i] - t[i];
  double beta = nrm2(r);
  out.final_rel = beta / bnorm;
  if (out.final_rel <= tol) return out;
  std::vector<std::vector<double>> V(m + 1, std::vector<double>(N));
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), gam(m + 1);
  // DCGS2 state (orth == 2, R14): unrotated Hessenberg columns, the reorthogonalisation
  // coefficients h2 of the provisional V[j] and its scalars nu (its normalisation) and
  // rho (its norm after reorthogonalisation)
  std::vector<double> Hraw((size_t)(m + 1) * m), h2p;
  double nu = 1.0, rhop = 1.0;
  while (true) {
    ORC_PAR
    for (size_t i = 0; i < N; ++i) V[0][i] = r[i] / beta;
    std::fill(gam.begin(), gam.end(), 0.0);
    gam[0] = beta;
    h2p.clear();
    nu = 1.0;                                           // V[0] is final
    rhop = 1.0;
    double next_scale = 0.0;
    int k = 0;
    bool broke = false;                                 // happy breakdown
    for (int j = 0; j < m; ++j) {
      if (!Bop(V[j].data(), z.data())) { out.status = 2; return out; }
      Aop(z.data(), t.data());
      std::vector<double>& w = t;
      auto h = [&](int i) -> double& { return H[(size_t)i * m + j]; };
      for (int i = 0; i <= j + 1; ++i) h(i) = 0.0;
      if (orth == 0) {                                  // CGS2
        for (int pass = 0; pass < 2; ++pass) {
          std::vector<double> hh(j + 1);
          ORC_PAR
          for (int i = 0; i <= j; ++i) hh[i] = dot(V[i], w);
          // w -= sum_i hh_i V_i: for every element the subtractions run in the order i = 0..j
          ORC_PAR
          for (size_t q = 0; q < N; ++q)
            for (int i = 0; i <= j; ++i) w[q] -= hh[i] * V[i][q];
          for (int i = 0; i <= j; ++i) h(i) += hh[i];
        }
      } else if (orth == 1) {                           // MGS
        for (int i = 0; i <= j; ++i) {
          double hi = dot(V[i], w);
          for (size_t q = 0; q < N; ++q) w[q] -= hi * V[i][q];
          h(i) = hi;
        }
      }
      double hn;
      if (orth == 2) {
        // DCGS2 (R14), textbook form with a NORMALISED provisional vector (the product
        // stores it unnormalised; the two agree in exact arithmetic).  V[0..j) final;
        // V[j] provisional = u_{j-1} / nu with nu = ||u_{j-1}|| (V[0] is final: nu = rho
        // = 1); h2p = V[0..j)^T u_{j-1} and rho = ||u_{j-1} - V[0..j) h2p|| are known from
        // the previous step; w = A B V[j].
        // (1) a_i = V[i]^T w for i <= j (one pass)
        std::vector<double> a(j + 1);
        for (int i = 0; i <= j; ++i) a[i] = dot(V[i], w);
        // (2) c_j = (final v_j)^T w = (nu a_j - h2p^T a_{0..j}) / rho
        double cj = nu * a[j];
        for (int i = 0; i < j; ++i) cj -= h2p[i] * a[i];
        cj /= rhop;
        // (3) finalise v_j = (nu V[j] - V[0..j) h2p) / rho and project w once onto the
        //     final basis: u = w - V[0..j) a - v_j c_j (one pass)
        for (size_t q = 0; q < N; ++q) {
          double s1 = 0.0;
          for (int i = 0; i < j; ++i) s1 += h2p[i] * V[i][q];
          V[j][q] = (nu * V[j][q] - s1) / rhop;
        }
        for (size_t q = 0; q < N; ++q) {
          double s2 = 0.0;
          for (int i = 0; i < j; ++i) s2 += a[i] * V[i][q];
          w[q] = w[q] - s2 - cj * V[j][q];
        }
        // (4) second-projection coefficients of u (used at the next step) and ||u||
        std::vector<double> h2n(j + 1);
        for (int i = 0; i <= j; ++i) h2n[i] = dot(V[i], w);
        const double uu = dot(w, w);
        double ss = 0.0;
        for (int i = 0; i <= j; ++i) ss += h2n[i] * h2n[i];
        const double nun = std::sqrt(uu);
        const double rhon = std::sqrt(std::max(uu - ss, 0.0));
        // (5) Hessenberg column j of the final basis:
        //     A B v_j = (nu A B V[j] - sum_{l<j} h2p_l A B v_l) / rho,
        //     A B V[j] = w = V[0..j] (c + h2n) + rhon v_{j+1}
        for (int i = 0; i <= j + 1; ++i) {
          double ci = (i < j) ? a[i] : (i == j ? cj : 0.0);
          double v = (i <= j) ? nu * (ci + h2n[i]) : nu * rhon;
          for (int l = 0; l < j; ++l) v -= h2p[l] * Hraw[(size_t)i * m + l];
          Hraw[(size_t)i * m + j] = v / rhop;
          h(i) = Hraw[(size_t)i * m + j];
        }
        hn = h(j + 1);
        next_scale = nun;                                // V[j+1] provisional = u / ||u||
        h2p = h2n;
        nu = nun;
        rhop = rhon;
      } else {
        hn = nrm2(w);
        h(j + 1) = hn;
        next_scale = hn;
      }
      out.iters++;
      for (int i = 0; i < j; ++i) {                     // previous rotations
        double a = h(i), c = h(i + 1);
        h(i) = cs[i] * a + sn[i] * c;
        h(i + 1) = -sn[i] * a + cs[i] * c;
      }
      double rho = std::hypot(h(j), h(j + 1));
      cs[j] = h(j) / rho;
      sn[j] = h(j + 1) / rho;
      h(j) = rho;
      h(j + 1) = 0.0;
      gam[j + 1] = -sn[j] * gam[j];
      gam[j] = cs[j] * gam[j];
      const double est = std::fabs(gam[j + 1]) / bnorm;
      out.hist.push_back(est);
      k = j + 1;
      broke = hn < 1e-14 * bnorm;
      if (est <= tol || broke || out.iters >= maxit) break;
      ORC_PAR
      for (size_t q = 0; q < N; ++q) V[j + 1][q] = w[q] / next_scale;
    }
    std::vector<double> y(k);
    for (int i = k - 1; i >= 0; --i) {
      double s = 0.0;
      for (int l = i + 1; l < k; ++l) s += H[(size_t)i * m + l] * y[l];
      y[i] = (gam[i] - s) / H[(size_t)i * m + i];
    }
    std::vector<double> u(N, 0.0);
    ORC_PAR
    for (size_t q = 0; q < N; ++q)
      for (int i = 0; i < k; ++i) u[q] += y[i] * V[i][q];
    if (!Bop(u.data(), z.data())) { out.status = 2; return out; }
    ORC_PAR
    for (size_t q = 0; q < N; ++q) x[q] += z[q];
    Aop(x, t.data());
    ORC_PAR
    for (size_t i = 0; i < N; ++i) r[i] = b[i] - t[i];
    beta = nrm2(r);
    out.final_rel = beta / bnorm;
    out.hist.push_back(out.final_rel);
    if (out.final_rel <= tol) return out;
    // invariant Krylov space with the true residual above tol: MSP_EBREAKDOWN (4)
    if (broke) { out.status = 4; return out; }
    if (out.iters >= maxit) { out.status = 3; return out; }
  }
}

// c-12: ASMSP decision (Remark 2): rebuild iff iota == 1, or
// It^(iota-1) > mu, or the matrix size changed.
static int asmsp_decide(int iota, int last_it, int mu, int dims_changed) {
  if (iota <= 1 || dims_changed || last_it > mu) return 1;
  return 0;
}

}  // namespace orc

// ============================================================================
// C interface for the Python test harness (ctypes).
// ============================================================================
using namespace orc;

extern "C" {

typedef struct {
  int32_t coarsest_max_dof, max_levels, pre_sweeps, post_sweeps, pair_passes, decoupling,
      bilu_order, stages, orth, smoother, gs_chunk;
} orc_config;

const char* orc_last_error() { return g_err.c_str(); }

// OMP timing mode (results bit-identical for any thread count); returns the count in use
int orc_set_threads(int n) {
#ifdef _OPENMP
  g_threads = n > 0 ? n : omp_get_max_threads();
#else
  (void)n;
  g_threads = 1;
#endif
  return g_threads;
}

static Csr mkcsr(int n, const int* ptr, const int* col, const double* val) {
  Csr A;
  A.n = n;
  A.ptr.assign(ptr, ptr + n + 1);
  A.col.assign(col, col + ptr[n]);
  A.val.assign(val, val + ptr[n]);
  return A;
}
static Bsr mkbsr(int n, int b, const int* ptr, const int* col, const double* val) {
  Bsr A;
  A.n = n;
  A.b = b;
  A.ptr.assign(ptr, ptr + n + 1);
  A.col.assign(col, col + ptr[n]);
  A.val.assign(val, val + (size_t)ptr[n] * b * b);
  return A;
}
static void put_graph(const Graph& G, int* optr, int* ocol) {
  optr[0] = 0;
  for (size_t i = 0; i < G.size(); ++i) {
    optr[i + 1] = optr[i] + (int)G[i].size();
    std::copy(G[i].begin(), G[i].end(), ocol + optr[i]);
  }
}
static Config mkcfg(const orc_config* c) {
  Config k;
  if (!c) return k;
  k.coarsest_max_dof = c->coarsest_max_dof;
  k.max_levels = c->max_levels;
  k.pre_sweeps = c->pre_sweeps;
  k.post_sweeps = c->post_sweeps;
  k.pair_passes = c->pair_passes;
  k.decoupling = c->decoupling;
  k.bilu_order = c->bilu_order;
  k.stages = c->stages;
  k.orth = c->orth;
  k.smoother = c->smoother;
  k.gs_chunk = c->gs_chunk;
  return k;
}

int orc_bsr_spmv(int n, int b, const int* ptr, const int* col, const double* val, const double* x,
                 double* y) {
  bsr_spmv(mkbsr(n, b, ptr, col, val), x, y);
  return 0;
}

int orc_csr_adjacency(int n, const int* ptr, const int* col, const double* val, int* optr, int* ocol) {
  Graph G = adjacency(mkcsr(n, ptr, col, val));
  put_graph(G, optr, ocol);
  return optr[n];
}

int orc_cell_graph(int n, int b, const int* ptr, const int* col, const double* val, int* optr, int* ocol) {
  Graph G = cell_graph(mkbsr(n, b, ptr, col, val));
  put_graph(G, optr, ocol);
  return optr[n];
}

// Alg. 3 on a given graph (sorted symmetric neighbour lists).  color[i] = group index.
int orc_grouping(int n, const int* gptr, const int* gcol, int* color) {
  Graph G(n);
  for (int i = 0; i < n; ++i) G[i].assign(gcol + gptr[i], gcol + gptr[i + 1]);
  auto groups = vertices_grouping(G);
  for (size_t g = 0; g < groups.size(); ++g) for (int v : groups[g]) color[v] = (int)g;
  return (int)groups.size();
}

// single Alg. 2 call on the vertex subset V (returns |W|; W and Wbar ascending)
int orc_splitting(int n, const int* gptr, const int* gcol, int nv, const int* V, int* W, int* Wbar) {
  Graph G(n);
  for (int i = 0; i < n; ++i) G[i].assign(gcol + gptr[i], gcol + gptr[i + 1]);
  std::vector<int> deg(n);
  for (int i = 0; i < n; ++i) deg[i] = (int)G[i].size();
  std::vector<int> Wv, Wb;
  vertices_splitting(G, deg, std::vector<int>(V, V + nv), Wv, Wb);
  std::copy(Wv.begin(), Wv.end(), W);
  std::copy(Wb.begin(), Wb.end(), Wbar);
  return (int)Wv.size();
}

int orc_csr_grouping(int n, const int* ptr, const int* col, const double* val, int* color) {
  auto groups = vertices_grouping(adjacency(mkcsr(n, ptr, col, val)));
  for (size_t g = 0; g < groups.size(); ++g) for (int v : groups[g]) color[v] = (int)g;
  return (int)groups.size();
}

int orc_npair(int n, const int* ptr, const int* col, const double* val, int* agg) {
  std::vector<int> a;
  int na = npair(mkcsr(n, ptr, col, val), a);
  std::copy(a.begin(), a.end(), agg);
  return na;
}

int orc_galerkin(int n, const int* ptr, const int* col, const double* val, const int* agg, int nagg,
                 int* optr, int* ocol, double* oval) {
  Csr C = galerkin(mkcsr(n, ptr, col, val), std::vector<int>(agg, agg + n), nagg);
  std::copy(C.ptr.begin(), C.ptr.end(), optr);
  std::copy(C.col.begin(), C.col.end(), ocol);
  std::copy(C.val.begin(), C.val.end(), oval);
  return (int)C.col.size();
}

// one PGS-MC sweep with a given coloring (color[i] in [0,g)); returns 0 or 2
int orc_pgs_mc(int n, const int* ptr, const int* col, const double* val, const int* color, int g,
               const double* b, double* x, int ascending) {
  std::vector<std::vector<int>> groups(g);
  for (int i = 0; i < n; ++i) groups[color[i]].push_back(i);
  return pgs_mc_sweep(mkcsr(n, ptr, col, val), groups, b, x, ascending != 0) ? 0 : 2;
}

// one PJAC-NO / PGS-NO sweep (R13); returns 0 or 2
int orc_jacobi(int n, const int* ptr, const int* col, const double* val, const double* b, double* x) {
  return jacobi_sweep(mkcsr(n, ptr, col, val), b, x) ? 0 : 2;
}
int orc_hybrid_gs(int n, const int* ptr, const int* col, const double* val, int K, const double* b, double* x,
                  int ascending) {
  return hybrid_gs_sweep(mkcsr(n, ptr, col, val), K, b, x, ascending != 0) ? 0 : 2;
}

int orc_dense_lu_solve(int n, const double* M, const double* b, double* x) {
  DenseLU lu;
  lu.n = n;
  lu.a.assign(M, M + (size_t)n * n);
  if (!lu.factor_dense()) return 2;
  lu.solve(b, x);
  return 0;
}

int orc_blk_inv(int b, const double* D, double* Dinv) { return blk_inv(b, D, Dinv) ? 0 : 2; }

// identity- or diagonal-preconditioned GMRES on a CSR matrix (pins for c-11)
int orc_gmres_csr(int n, const int* ptr, const int* col, const double* val, const double* b, double* x,
                  double tol, int m, int maxit, int orth, const double* Minv_dense, int* iters,
                  double* final_rel, double* hist, int cap, int* hlen) {
  Csr A = mkcsr(n, ptr, col, val);
  auto Aop = [&](const double* v, double* y) { csr_spmv(A, v, y); };
  auto Bop = [&](const double* v, double* y) -> bool {
    if (!Minv_dense) { std::copy(v, v + n, y); return true; }
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int j = 0; j < n; ++j) s += Minv_dense[(size_t)i * n + j] * v[j];
      y[i] = s;
    }
    return true;
  };
  GmresOut o = gmres((size_t)n, Aop, Bop, b, x, tol, m, maxit, orth);
  *iters = o.iters;
  *final_rel = o.final_rel;
  int L = std::min<int>(cap, (int)o.hist.size());
  std::copy(o.hist.begin(), o.hist.begin() + L, hist);
  *hlen = L;
  return o.status;
}

int orc_asmsp_decide(int iota, int last_it, int mu, int dims_changed) {
  return asmsp_decide(iota, last_it, mu, dims_changed);
}

// ---- full MSP ----
void* orc_msp_setup(int n, int b, const int* ptr, const int* col, const double* val,
                    const orc_config* cfg, int* status) {
  Msp* M = new Msp;
  M->cfg = mkcfg(cfg);
  M->A = mkbsr(n, b, ptr, col, val);
  int rc = msp_setup(*M);
  *status = rc;
  if (rc) { delete M; return nullptr; }
  return M;
}

// ASMSP reuse: replace A's values, keep the stage operators (SURVEY c-12)
int orc_msp_update_values(void* h, const double* val) {
  Msp* M = (Msp*)h;
  std::copy(val, val + M->A.val.size(), M->A.val.begin());
  return 0;
}

void orc_msp_destroy(void* h) { delete (Msp*)h; }

// info[0]=levels L (smoothing), info[1]=coarsest n, info[2]=coarse_diag
int orc_msp_info(void* h, int* info) {
  Msp* M = (Msp*)h;
  info[0] = (int)M->H.lv.size();
  info[1] = M->H.Ac.n;
  info[2] = M->H.coarse_diag ? 1 : 0;
  return 0;
}
int orc_msp_level_n(void* h, int l, int* n, int* nnz, int* ncolors) {
  Msp* M = (Msp*)h;
  const Csr& A = (l < (int)M->H.lv.size()) ? M->H.lv[l].A : M->H.Ac;
  *n = A.n;
  *nnz = (int)A.col.size();
  *ncolors = (l < (int)M->H.lv.size()) ? (int)M->H.lv[l].groups.size() : 0;
  return 0;
}
int orc_msp_level_csr(void* h, int l, int* ptr, int* col, double* val) {
  Msp* M = (Msp*)h;
  const Csr& A = (l < (int)M->H.lv.size()) ? M->H.lv[l].A : M->H.Ac;
  std::copy(A.ptr.begin(), A.ptr.end(), ptr);
  std::copy(A.col.begin(), A.col.end(), col);
  std::copy(A.val.begin(), A.val.end(), val);
  return 0;
}
int orc_msp_level_colors(void* h, int l, int* color) {
  Msp* M = (Msp*)h;
  const auto& G = M->H.lv[l].groups;
  for (size_t g = 0; g < G.size(); ++g) for (int v : G[g]) color[v] = (int)g;
  return (int)G.size();
}
int orc_msp_level_agg(void* h, int l, int* agg) {
  Msp* M = (Msp*)h;
  std::copy(M->H.lv[l].agg.begin(), M->H.lv[l].agg.end(), agg);
  return M->H.lv[l].n_next;
}
int orc_msp_weights(void* h, double* W) {
  Msp* M = (Msp*)h;
  std::copy(M->W.begin(), M->W.end(), W);
  return 0;
}
int orc_msp_order(void* h, int* order) {
  Msp* M = (Msp*)h;
  std::copy(M->R.order.begin(), M->R.order.end(), order);
  return 0;
}
// BILU factors in natural BSR storage (row-major blocks) + Dinv per cell
int orc_msp_bilu_factors(void* h, double* F, double* Dinv) {
  Msp* M = (Msp*)h;
  std::copy(M->R.F.val.begin(), M->R.F.val.end(), F);
  std::copy(M->R.Dinv.begin(), M->R.Dinv.end(), Dinv);
  return 0;
}
int orc_msp_vcycle(void* h, const double* r, double* x) {
  Msp* M = (Msp*)h;
  std::vector<double> b(r, r + M->A.n), xv;
  if (!vcycle(M->H, M->cfg, 0, b, xv)) return 2;
  std::copy(xv.begin(), xv.end(), x);
  return 0;
}
int orc_msp_bilu_apply(void* h, const double* r, double* x) {
  bilu_apply(((Msp*)h)->R, r, x);
  return 0;
}
int orc_msp_apply(void* h, const double* g, double* w) { return msp_apply(*(Msp*)h, g, w) ? 0 : 2; }

// per-step entry points of the hot path (parity tests of the individual kernels)
int orc_msp_restrict_pressure(void* h, const double* g, double* rp) {      // a3
  restrict_pressure(*(Msp*)h, g, rp);
  return 0;
}
int orc_msp_level_resid_restrict(void* h, int l, const double* b, const double* x, double* bc) {   // a5
  Msp* M = (Msp*)h;
  if (l < 0 || l >= (int)M->H.lv.size()) return 1;
  residual_restrict(M->H.lv[l], b, x, bc);
  return 0;
}
int orc_msp_level_prolong(void* h, int l, const double* e, double* x) {   // a7 (x updated in place)
  Msp* M = (Msp*)h;
  if (l < 0 || l >= (int)M->H.lv.size()) return 1;
  prolong_correct(M->H.lv[l], e, x);
  return 0;
}
int orc_msp_bilu_forward(void* h, const double* r, double* y, int absmode) {
  bilu_forward(((Msp*)h)->R, r, y, absmode != 0);
  return 0;
}
int orc_msp_bilu_backward(void* h, const double* y, double* x, int absmode) {
  bilu_backward(((Msp*)h)->R, y, x, absmode != 0);
  return 0;
}
int orc_msp_bilu_apply_by_color(void* h, const double* r, double* x) {
  bilu_apply_by_color(((Msp*)h)->R, r, x);
  return 0;
}
// test hook: replace the BILU factors (natural BSR storage, row-major blocks) and D~^-1,
// e.g. by integer-valued factors for the bit-exact substitution tests
int orc_msp_bilu_set_factors(void* h, const double* F, const double* Dinv) {
  Msp* M = (Msp*)h;
  std::copy(F, F + M->R.F.val.size(), M->R.F.val.begin());
  std::copy(Dinv, Dinv + M->R.Dinv.size(), M->R.Dinv.begin());
  return 0;
}
// test hook: refactorize the BILU(0) in the SAME elimination order from the given values
// (e.g. A with the couplings between ranks removed: the rank-local BILU of the distributed
// product); the hierarchy and W stay those of the setup matrix
int orc_msp_bilu_refactor(void* h, const double* vals) {
  Msp* M = (Msp*)h;
  Bsr B = M->A;
  std::copy(vals, vals + B.val.size(), B.val.begin());
  std::vector<int> color = M->R.color, blk = M->R.blk, order = M->R.order;
  if (!bilu_factor(B, order, M->R)) return 2;
  M->R.color = color;
  M->R.blk = blk;
  return 0;
}
// block color and ABMC block id of every cell (natural numbering); returns #colors
int orc_msp_bilu_blocks(void* h, int* color, int* blk) {
  Msp* M = (Msp*)h;
  int g = 0;
  for (int c = 0; c < M->A.n; ++c) {
    color[c] = M->R.color[c];
    blk[c] = M->R.blk[c];
    g = std::max(g, color[c] + 1);
  }
  return g;
}
// a10: out[i] = V[i]^T w for k vectors of length N stored consecutively (index-ascending
// sums from +0.0, the plain definition)
int orc_dots(long long N, int k, const double* V, const double* w, double* out) {
  for (int i = 0; i < k; ++i) {
    double s = 0.0;
    for (long long q = 0; q < N; ++q) s += V[(size_t)i * N + q] * w[q];
    out[i] = s;
  }
  return 0;
}

// B_N r (stages = 3 handles only): N-part of the result, n*nc doubles
int orc_msp_bgs_apply(void* h, const double* r, double* wN) {
  Msp* M = (Msp*)h;
  if (M->cfg.stages != 3) return 1;
  std::vector<double> rv(r, r + (size_t)M->A.n * M->A.b), w;
  bgs_stage(*M, rv, w);
  std::copy(w.begin(), w.end(), wN);
  return 0;
}

int orc_msp_solve(void* h, const double* b, double* x, double tol, int restart, int maxit, int* iters,
                  double* final_rel, double* hist, int cap, int* hlen) {
  Msp* M = (Msp*)h;
  const size_t N = (size_t)M->A.n * M->A.b;
  auto Aop = [&](const double* v, double* y) { bsr_spmv(M->A, v, y); };
  auto Bop = [&](const double* v, double* y) -> bool { return msp_apply(*M, v, y); };
  GmresOut o = gmres(N, Aop, Bop, b, x, tol, restart, maxit, M->cfg.orth);
  *iters = o.iters;
  *final_rel = o.final_rel;
  int L = std::min<int>(cap, (int)o.hist.size());
  std::copy(o.hist.begin(), o.hist.begin() + L, hist);
  *hlen = L;
  return o.status;
}

}  // extern "C"
