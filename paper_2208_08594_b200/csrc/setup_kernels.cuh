// GPU-side SETUP kernels (§8(a) S1 and the Galerkin products of S3).
//
// Bit-exact with the host setup (setup.cpp) and the oracle: every floating-point
// operation is an explicitly rounded __dadd_rn / __dsub_rn / __dmul_rn / __ddiv_rn in the
// order DESIGN.md R4 / R3 fixes (no FMA contraction), so the decisions taken downstream
// on these values (NPAIR pairing, colorings, ABMC order) are identical.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mspk {

// S1 (R4, TI): block column sums C_c = sum_p A[p,c], p ascending, from +0.0.
// cp/ce: CSC of the block pattern (entries of column c in ascending row order);
// A: natural-order row-major blocks.  One thread per (cell, block element).
template <int B>
__global__ void colsum_kernel(int n, const int* __restrict__ cp, const int* __restrict__ ce,
                              const double* __restrict__ A, double* __restrict__ C) {
  constexpr int BB = B * B;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)n * BB) return;
  const int c = (int)(t / BB), k = (int)(t - (int64_t)c * BB);
  double acc = 0.0;
  for (int q = cp[c]; q < cp[c + 1]; ++q) acc = __dadd_rn(acc, A[(size_t)ce[q] * BB + k]);
  C[t] = acc;
}

// S1 (R4, QI): C_c = the diagonal block (dg: entry of (c, c) in natural storage).
template <int B>
__global__ void diagblock_kernel(int n, const int* __restrict__ dg, const double* __restrict__ A,
                                 double* __restrict__ C) {
  constexpr int BB = B * B;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)n * BB) return;
  const int c = (int)(t / BB), k = (int)(t - (int64_t)c * BB);
  C[t] = A[(size_t)dg[c] * BB + k];
}

// S1 (R4): w_c = [1, y] with C_NN^T y = -C_0N^T, Gaussian elimination with partial
// pivoting (first maximal |pivot|), f = a_ik / a_kk, a_ij = a_ij - f a_kj (j > k),
// back substitution s = sum_{j>i} a_ij y_j ascending from +0.0, y_i = (r_i - s) / a_ii.
// One thread per cell; *bad = max cell with a zero pivot (-1 if none).
template <int B>
__global__ void weights_kernel(int n, const double* __restrict__ C, double* __restrict__ W, int* bad) {
  constexpr int NC = B - 1, BB = B * B;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  W[(size_t)c * B] = 1.0;
  if constexpr (NC > 0) {
    double M[NC][NC], r[NC], y[NC];
    const double* Cc = C + (size_t)c * BB;
#pragma unroll
    for (int i = 0; i < NC; ++i) {
#pragma unroll
      for (int j = 0; j < NC; ++j) M[i][j] = Cc[(1 + j) * B + 1 + i];
      r[i] = -Cc[1 + i];
    }
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      int p = k;
      double best = fabs(M[k][k]);
#pragma unroll
      for (int i = k + 1; i < NC; ++i) {
        const double a = fabs(M[i][k]);
        if (a > best) { best = a; p = i; }
      }
      double piv = 0.0;
#pragma unroll
      for (int i = k; i < NC; ++i) if (i == p) piv = M[i][k];
      if (piv == 0.0) {
        atomicMax(bad, c);
        return;
      }
      if (p != k) {                                  // swap rows k and p (registers: unrolled)
#pragma unroll
        for (int i = k + 1; i < NC; ++i) {
          if (i == p) {
#pragma unroll
            for (int j = 0; j < NC; ++j) { const double tmp = M[k][j]; M[k][j] = M[i][j]; M[i][j] = tmp; }
            const double tr = r[k]; r[k] = r[i]; r[i] = tr;
          }
        }
      }
      piv = M[k][k];
#pragma unroll
      for (int i = k + 1; i < NC; ++i) {
        const double f = __ddiv_rn(M[i][k], piv);
#pragma unroll
        for (int j = k + 1; j < NC; ++j) M[i][j] = __dsub_rn(M[i][j], __dmul_rn(f, M[k][j]));
        r[i] = __dsub_rn(r[i], __dmul_rn(f, r[k]));
      }
    }
#pragma unroll
    for (int i = NC - 1; i >= 0; --i) {
      double acc = 0.0;
#pragma unroll
      for (int j = i + 1; j < NC; ++j) acc = __dadd_rn(acc, __dmul_rn(M[i][j], y[j]));
      y[i] = __ddiv_rn(__dsub_rn(r[i], acc), M[i][i]);
    }
#pragma unroll
    for (int i = 0; i < NC; ++i) W[(size_t)c * B + 1 + i] = y[i];
  }
}

// S1: A_PP[c, d] = sum_{k=0}^{b-1} w_c[k] * A[c,d][k][0], k ascending from +0.0 (R4).
// One thread per cell row.
template <int B>
__global__ void app_kernel(int n, const int* __restrict__ rp, const double* __restrict__ W,
                           const double* __restrict__ A, double* __restrict__ P) {
  constexpr int BB = B * B;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  double w[B];
#pragma unroll
  for (int k = 0; k < B; ++k) w[k] = W[(size_t)c * B + k];
  for (int e = rp[c]; e < rp[c + 1]; ++e) {
    const double* Ae = A + (size_t)e * BB;
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < B; ++k) acc = __dadd_rn(acc, __dmul_rn(w[k], Ae[k * B]));
    P[e] = acc;
  }
}

// S2 input: nz[e] = block e has a nonzero entry (the cell graph of R5 / c-3).
template <int B>
__global__ void block_nonzero_kernel(int64_t nnzb, const double* __restrict__ A, uint8_t* __restrict__ nz) {
  constexpr int BB = B * B;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nnzb) return;
  bool f = false;
#pragma unroll
  for (int t = 0; t < BB; ++t) f = f || (A[(size_t)e * BB + t] != 0.0);
  nz[e] = f ? 1 : 0;
}

// S3 Galerkin product A_c = P^T A P for a piecewise-constant P (R3): coarse row I gets
// the union of agg[col] over the rows of its members (pattern sorted ascending, exact
// zeros kept) and, for members i ascending and their stored entries ascending, the value
// a_ij added into the slot of J = agg[j] -- the specified summation order (SURVEY c-5).
// One thread per coarse row; a row's candidate columns are collected in a local buffer of
// kRapMax entries (rows with more set *overflow; the caller then uses the host product).
constexpr int kRapMax = 192;

__device__ __forceinline__ int rap_collect(int I, const int* __restrict__ mp, const int* __restrict__ mi,
                                           const int* __restrict__ rp, const int* __restrict__ ci,
                                           const int* __restrict__ agg, int* cols) {
  int m = 0;
  for (int q = mp[I]; q < mp[I + 1]; ++q) {
    const int i = mi[q];
    for (int e = rp[i]; e < rp[i + 1]; ++e) {
      const int J = agg[ci[e]];
      // insertion into the sorted, unique list
      int pos = m;
      while (pos > 0 && cols[pos - 1] > J) --pos;
      if (pos > 0 && cols[pos - 1] == J) continue;
      if (m >= kRapMax) return -1;
      for (int t = m; t > pos; --t) cols[t] = cols[t - 1];
      cols[pos] = J;
      ++m;
    }
  }
  return m;
}

__global__ void rap_count_kernel(int nc, const int* __restrict__ mp, const int* __restrict__ mi,
                                 const int* __restrict__ rp, const int* __restrict__ ci,
                                 const int* __restrict__ agg, int* __restrict__ cnt, int* overflow) {
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= nc) return;
  int cols[kRapMax];
  const int m = rap_collect(I, mp, mi, rp, ci, agg, cols);
  if (m < 0) {
    atomicExch(overflow, 1);
    cnt[I] = 0;
    return;
  }
  cnt[I] = m;
}

__global__ void rap_fill_kernel(int nc, const int* __restrict__ mp, const int* __restrict__ mi,
                                const int* __restrict__ rp, const int* __restrict__ ci,
                                const double* __restrict__ v, const int* __restrict__ agg,
                                const int* __restrict__ crp, int* __restrict__ cci, double* __restrict__ cv) {
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= nc) return;
  int cols[kRapMax];
  const int m = rap_collect(I, mp, mi, rp, ci, agg, cols);
  const int o = crp[I];
  for (int t = 0; t < m; ++t) {
    cci[o + t] = cols[t];
    cv[o + t] = 0.0;
  }
  for (int q = mp[I]; q < mp[I + 1]; ++q) {
    const int i = mi[q];
    for (int e = rp[i]; e < rp[i + 1]; ++e) {
      const int J = agg[ci[e]];
      int lo = 0, hi = m - 1;                       // slot of J (binary search)
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cols[mid] < J) lo = mid + 1;
        else hi = mid;
      }
      cv[o + lo] = __dadd_rn(cv[o + lo], v[e]);
    }
  }
}

// Rank-local BILU (NEXT-3 option): zero the blocks of the couplings between cells of
// different owners before the factorization (list of entries, bb doubles each).
__global__ void zero_blocks_kernel(int64_t count, int bb, const int* __restrict__ idx, double* __restrict__ F) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count * bb) return;
  const int64_t q = t / bb;
  F[(size_t)idx[q] * bb + (t - q * bb)] = 0.0;
}

// Coarsest level (a6 setup): dense row-major A_L from its CSR and the identity right-hand
// side (leading dimension ld) for the inverse; both outputs zeroed by the caller.
__global__ void dense_identity_kernel(int m, int ld, const int* __restrict__ rp, const int* __restrict__ ci,
                                      const double* __restrict__ v, double* __restrict__ dense,
                                      double* __restrict__ ident) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  for (int e = rp[i]; e < rp[i + 1]; ++e) dense[(size_t)i * m + ci[e]] = v[e];
  ident[(size_t)i * ld + i] = 1.0;
}

}  // namespace mspk
