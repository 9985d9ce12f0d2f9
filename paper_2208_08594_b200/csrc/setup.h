// Host-side SETUP of the MSP preconditioner.  Product code:
// written independently of oracle/ (different data structures: binary heaps with
// lazy deletion, degree-sorted scans, counting sorts, marker arrays), reproducing
// the same deterministic readings so that colorings, aggregates and
// Galerkin values are bit-identical.  Compiled with -ffp-contract=off.
#pragma once
#include <cstdint>
#include <string>
#include <functional>
#include <vector>

namespace msp {

struct SpMat {                       // scalar CSR, ascending columns
  int32_t n = 0;
  std::vector<int32_t> rp, ci;
  std::vector<double> v;
  int64_t nnz() const { return (int64_t)ci.size(); }
};

// Block values: owned, a read-only view of the caller's host buffer, or (dptr) the caller's
// DEVICE buffer, for the duration of one SETUP call -- no multi-GB copy of A before the
// setup uploads it; a host copy of device values is fetched (d2h) only if a host step
// reads them.
struct Values {
  mutable std::vector<double> own;
  mutable const double* p = nullptr;
  const double* dptr = nullptr;
  void (*d2h)(double* dst, const double* src, size_t count) = nullptr;
  size_t n = 0;
  Values() = default;
  Values(const Values& o) { *this = o; }
  Values& operator=(const Values& o) {
    if (this == &o) return *this;
    own = o.own;
    n = o.n;
    dptr = o.dptr;
    d2h = o.d2h;
    p = own.empty() ? o.p : own.data();
    return *this;
  }
  const double* host() const {
    if (!p && dptr) {
      own.resize(n);
      d2h(own.data(), dptr, n);
      p = own.data();
    }
    return p;
  }
  const double& operator[](size_t i) const { return p ? p[i] : host()[i]; }
  const double* data() const { return host(); }
  size_t size() const { return n; }
  bool empty() const { return n == 0; }
  void device_view(const double* d, size_t count, void (*fetch)(double*, const double*, size_t)) {
    own.clear();
    p = nullptr;
    dptr = d;
    d2h = fetch;
    n = count;
  }
  double* owned(size_t count) {               // (re)allocate an owned buffer of count values
    own.resize(count);
    p = own.data();
    dptr = nullptr;
    n = count;
    return own.data();
  }
  void view(const double* q, size_t count) {
    own.clear();
    own.shrink_to_fit();
    p = q;
    dptr = nullptr;
    n = count;
  }
};

struct BlockMat {                    // BSR, row-major b x b blocks (ABI layout)
  int32_t n = 0, b = 0;
  std::vector<int32_t> rp, ci;
  Values v;
};

struct Graph {                       // symmetric adjacency, ascending neighbours
  std::vector<int32_t> xadj, adj;
  int32_t deg(int32_t i) const { return xadj[i + 1] - xadj[i]; }
};

struct SpMat;
// Galerkin product hook (GPU, NEXT-2): returns 0 and fills C, or nonzero -> host product
using RapFn = std::function<int(const SpMat& A, const std::vector<int32_t>& agg, int32_t nagg, SpMat& C)>;

struct Params {
  int32_t coarsest_max_dof = 10000, max_levels = 20, pre_sweeps = 1, post_sweeps = 1,
          pair_passes = 2, decoupling = 2, bilu_order = 1, stages = 2, orth = 0, use_graphs = 1,
          use_coop = 1, smoother = 0, gs_chunk = 32, coarse_mode = 0, bilu_local = 0,
          dist_levels = 0;
  RapFn rap;                           // optional: S3 Galerkin products of the hierarchy
  bool s1_given = false;               // S.W and S.App already computed (GPU S1)
};

struct HostLevel {
  SpMat A;                           // natural level numbering
  int32_t ncolor = 0;
  std::vector<int32_t> color;        // PGS-MC group of each row (Alg. 3)
  std::vector<int32_t> agg;          // composite aggregate -> row of level l+1
  int32_t n_next = 0;
};

struct HostSetup {
  Params prm;
  const BlockMat* A = nullptr;       // caller-owned; valid during setup only
  int32_t n = 0;
  std::vector<double> W;             // decoupling weights, n*b
  SpMat App;                         // W^T A Pi_P
  std::vector<HostLevel> lv;         // smoothing levels
  SpMat Ac;                          // coarsest
  bool coarse_diag = false;
  // BILU ordering (positions -> cells) and its block/color structure
  std::vector<int32_t> order, pos;
  int32_t bilu_ncolor = 0;
  std::vector<int32_t> blk_ptr;        // cell-position ranges of the ordering blocks
  std::vector<int32_t> color_blk_ptr;  // block ranges per block color
  std::vector<int32_t> level1_agg;     // ABMC blocks (cell -> block id)
  std::vector<uint8_t> block_nz;       // optional: nonzero flag per stored block (GPU S1)
};

// status codes mirror msp_status
int run_host_setup(const BlockMat& A, const Params& prm, HostSetup& S, std::string& err);

// Block ILU(0) in the ordering of S (positions).  Outputs, in POSITION numbering:
// rp/ci (ascending positions) of the permuted pattern, diag index per row, and the
// factor values (row-major blocks; the diagonal slot holds D~^-1).
int bilu_factor_permuted(const HostSetup& S, const BlockMat& A, std::vector<int32_t>& rp,
                         std::vector<int32_t>& ci, std::vector<int32_t>& dg,
                         std::vector<int32_t>& src_entry, std::vector<double>& F, std::string& err);

// Pattern of A in the ordering positions (rows/cols permuted, columns sorted), without
// factorization; src[e] = natural entry of permuted entry e.
int permuted_pattern(const HostSetup& S, const BlockMat& A, std::vector<int32_t>& rp, std::vector<int32_t>& ci,
                     std::vector<int32_t>& dg, std::vector<int32_t>& src, std::string& err);

// Building blocks (exposed for the host-setup introspection entry points / tests)
Graph value_graph(const SpMat& A);
Graph block_graph(const BlockMat& A, const std::vector<uint8_t>* nz_given = nullptr);
int32_t color_groups(const Graph& G, std::vector<int32_t>& color);
int32_t pair_aggregate(const SpMat& A, std::vector<int32_t>& agg);
SpMat galerkin_rap(const SpMat& A, const std::vector<int32_t>& agg, int32_t nagg);
bool invert_block(int b, const double* D, double* Dinv);

}  // namespace msp
