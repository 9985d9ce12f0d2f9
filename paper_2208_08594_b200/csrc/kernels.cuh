// sm_100a kernels of the MSP-GMRES SOLVE phase.
// Paper: arXiv 2208.08594 (PAPER.md "P:n").  All FP64, HBM-bound (no dense
// contraction: no tensor cores).  Layouts:
//  - cell vectors: internal (ABMC) cell order, cell-interleaved, length n*B;
//  - BSR / BILU factors: row_ptr/col int32 in internal positions, b x b blocks
//    COLUMN-major (the pressure column of a block is one contiguous 32 B sector);
//  - AMG level l: rows permuted by PGS-MC color, SELL-32 slices that never straddle
//    a color: entry (row lane l, k) at slice_off[s] + 32*k + l; padding col = row,
//    val = 0.  Diagonal separate.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mspk {

constexpr int kSell = 32;
#ifndef MSP_BILU_PREFETCH
#define MSP_BILU_PREFETCH 1
#endif
constexpr bool kBiluPrefetch = MSP_BILU_PREFETCH != 0;
#ifndef MSP_UNI_TPB
#define MSP_UNI_TPB 128              // CTA size of the level-0 (uniform SELL) sweep kernel
#endif
#ifndef MSP_A8_TPB
#define MSP_A8_TPB 64                // CTA size of the ELL a8 kernel (C3: 65.6 -> 63.2 us vs 256)
#endif
#ifndef MSP_SPMV_TPB
#define MSP_SPMV_TPB 256             // CTA size of the 4x4 SpMV
#endif
#ifndef MSP_XFER_TPB
#define MSP_XFER_TPB 256             // CTA size of a3, restriction, prolongation, gather
#endif
#ifndef MSP_SELL_PFL
#define MSP_SELL_PFL 8               // matrix entries per lane prefetched by the LPR > 1 (coarse) sweeps
#endif
#ifndef MSP_SELL_PF1
#define MSP_SELL_PF1 6
#endif
#ifndef MSP_BILU_PFE
#define MSP_BILU_PFE 2
#endif
#ifndef MSP_BILU_MINB
#define MSP_BILU_MINB 12
#endif

__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }
__device__ __forceinline__ int ldg(const int* p) { return __ldg(p); }

// Streaming (evict-first, ld.global.cs) loads for large single-use operands (matrix and
// factor blocks), so that the gathered vectors stay L2-resident.  MSP_STREAM_HINT=0
// equivalent: define MSP_NO_CS.
#ifndef MSP_NO_CS
__device__ __forceinline__ double2 ldstream2(const double2* p) { return __ldcs(p); }
#else
__device__ __forceinline__ double2 ldstream2(const double2* p) { return __ldg(p); }
#endif

// Programmatic dependent launch (PDL).  Every kernel is launched with programmatic
// stream serialisation: it may start while its predecessor still runs, so it must
// call pdl_wait() before touching anything a predecessor produced (vectors); only
// immutable data (matrix values/indices) may be read before.  pdl_trigger() right
// after the wait lets the successor start its own prologue (at most two kernels
// overlap).  Both are no-ops when the kernel was launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#define PDL_ENTRY() do { pdl_wait(); pdl_trigger(); } while (0)

// Distributed mode: the producer of a halo-exchanged vector also writes each of its rows'
// values to their (<= 2) positions in the send buffer (HaloPlan::d_slots), so no separate
// pack kernel runs before the exchange.  slots == null: nothing to pack.
struct HaloPack {
  const int2* slots;
  double* buf;
};
__device__ __forceinline__ void halo_pack(const HaloPack& pk, int row, double v) {
  if (!pk.slots) return;
  const int2 q = __ldg(pk.slots + row);
  if (q.x >= 0) pk.buf[q.x] = v;
  if (q.y >= 0) pk.buf[q.y] = v;
}

// ---------------------------------------------------------------------------
// a2 (K1): BSR SpMV.  One team of TS lanes per block row (TS = 4 for b=4, 8 for b=7);
// lane q < B owns output row q of the cell.  Each block column-major: lane q reads
// val[e*B*B + t*B + q] for t = 0..B-1, so a team reads each 8-byte column slice of a
// block as one contiguous B*8-byte segment.  x of the neighbour is loaded once per
// lane (component q) and broadcast with shuffles.
//   MODE 0: y = A x          MODE 1: y = g - A x (residual, Alg. 1 lines 3/5)
//   MODE 2: y = g - A[:,P] xp  (a8: pressure column only, xp per cell); `val` is then
//           the contiguous pressure-column array Pcol[e*B + q] = A_e[q][0] (one 32 B
//           sector per block for b=4, consecutive blocks contiguous).
// ---------------------------------------------------------------------------
template <int B, int MODE>
__global__ void __launch_bounds__(256) bsr_spmv_kernel(int n, const int* __restrict__ rp,
                                                       const int* __restrict__ ci,
                                                       const double* __restrict__ val,
                                                       const double* __restrict__ x,
                                                       const double* __restrict__ g,
                                                       double* __restrict__ y) {
  constexpr int TS = (B <= 4) ? 4 : 8;
  constexpr int BB = B * B;
  constexpr int PF = 4;                        // MODE 2: entries prefetched before the PDL wait
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int row = gtid / TS;
  const int q = threadIdx.x % TS;
  const int lane = threadIdx.x & 31;
  const int base = lane - q;
  const bool live = row < n;                   // whole teams (n*TS threads padded per team)
  const int e0 = live ? ldg(rp + row) : 0, e1 = live ? ldg(rp + row + 1) : 0;
  int pc[PF];
  double pv[PF];
  if (MODE == 2) {                             // immutable columns and pressure columns
#pragma unroll
    for (int m = 0; m < PF; ++m) {
      const int e = e0 + m;
      pc[m] = (e < e1) ? ldg(ci + e) : 0;
      pv[m] = (e < e1 && q < B) ? ldg(val + (size_t)e * B + q) : 0.0;
    }
  }
  pdl_wait();
  pdl_trigger();
  if (!live) return;
  double acc = 0.0;
  const unsigned mask = (TS == 32) ? 0xffffffffu : (((1u << TS) - 1u) << base);
  if (MODE == 2) {
#pragma unroll
    for (int m = 0; m < PF; ++m)
      if (e0 + m < e1) {
        const double xc = ldg(x + pc[m]);
        if (q < B) acc = fma(pv[m], xc, acc);
      }
#pragma unroll 4
    for (int e = e0 + PF; e < e1; ++e) {
      const int c = ldg(ci + e);
      const double xc = ldg(x + c);
      if (q < B) acc = fma(ldg(val + (size_t)e * B + q), xc, acc);
    }
  } else {
#pragma unroll 2
    for (int e = e0; e < e1; ++e) {
      const int c = ldg(ci + e);
      const double xq = (q < B) ? ldg(x + (size_t)c * B + q) : 0.0;
      const double* blk = val + (size_t)e * BB;
#pragma unroll
      for (int t = 0; t < B; ++t) {
        const double xt = __shfl_sync(mask, xq, base + t);
        if (q < B) acc = fma(ldg(blk + t * B + q), xt, acc);
      }
    }
  }
  if (q < B) {
    const size_t o = (size_t)row * B + q;
    y[o] = (MODE == 0) ? acc : (g[o] - acc);
  }
}

// 4-lane reduce-scatter: lane q of a 4-lane group holds a[0..3] (partial sums of rows
// 0..3); returns sum over the group of a[q] (fixed butterfly order: deterministic).
// m4: mask of the (aligned) 4-lane group; xor offsets 1, 2 stay inside the group.
__device__ __forceinline__ double reduce_scatter4(double a0, double a1, double a2, double a3, int q,
                                                  unsigned m4) {
  const bool hi = (q & 2) != 0;
  const double s0 = hi ? a0 : a2, s1 = hi ? a1 : a3;
  const double r0 = __shfl_xor_sync(m4, s0, 2), r1 = __shfl_xor_sync(m4, s1, 2);
  const double k0 = (hi ? a2 : a0) + r0, k1 = (hi ? a3 : a1) + r1;
  const bool odd = (q & 1) != 0;
  const double r = __shfl_xor_sync(m4, odd ? k0 : k1, 1);
  return (odd ? k1 : k0) + r;
}

// 8-lane reduce-scatter of a[0..7] (lane q of an aligned 8-lane group) -> sum of a[q]
// over the group; 4 + 2 + 1 shuffles, fixed order.
__device__ __forceinline__ double reduce_scatter8(const double (&a)[8], int q, unsigned m8) {
  const bool b2 = (q & 4) != 0;
  double k[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const double send = b2 ? a[u] : a[u + 4];
    const double keep = b2 ? a[u + 4] : a[u];
    k[u] = keep + __shfl_xor_sync(m8, send, 4);
  }
  const bool b1 = (q & 2) != 0;
  double l[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const double send = b1 ? k[u] : k[u + 2];
    const double keep = b1 ? k[u + 2] : k[u];
    l[u] = keep + __shfl_xor_sync(m8, send, 2);
  }
  const bool b0 = (q & 1) != 0;
  const double send = b0 ? l[0] : l[1];
  const double keep = b0 ? l[1] : l[0];
  return keep + __shfl_xor_sync(m8, send, 1);
}

// column-per-lane partial sums for a B x B block (5 <= B <= 8, 8-lane group): lane q < B
// adds column q of the column-major block times v_q into a[0..B-1]
template <int B>
__device__ __forceinline__ void col_accum8(const double* __restrict__ blk, double vq, int q, double (&a)[8]) {
  if (q < B) {
#pragma unroll
    for (int r = 0; r < B; ++r) a[r] = fma(__ldcs(blk + q * B + r), vq, a[r]);
  }
}

// a2 for 5x5..8x8 blocks, column-per-lane (8 lanes per block row, lane 7 idle for B = 7).
// The row's first MSP_SPMV8_PF entries (columns and block columns) are immutable and
// loaded before the PDL wait; the rest stream with two entries in flight.  Entries are
// accumulated in ascending order either way (same fma sequence as col_accum8).
#ifndef MSP_SPMV8_PF
#define MSP_SPMV8_PF 2
#endif
template <int B, int MODE>
#ifndef MSP_SPMV8_TPB
#define MSP_SPMV8_TPB 256
#endif
__global__ void __launch_bounds__(MSP_SPMV8_TPB) bsr_spmv8c_kernel(int n, const int* __restrict__ rp,
                                                         const int* __restrict__ ci,
                                                         const double* __restrict__ val,
                                                         const double* __restrict__ x,
                                                         const double* __restrict__ g,
                                                         double* __restrict__ y) {
  constexpr int BB = B * B;
  constexpr int PF = MSP_SPMV8_PF;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int row = gtid >> 3, q = threadIdx.x & 7;
  const bool live = row < n;                   // whole 8-lane groups
  const int e0 = live ? ldg(rp + row) : 0, e1 = live ? ldg(rp + row + 1) : 0;
  int pc[PF];
  double pv[PF][B];
#pragma unroll
  for (int m = 0; m < PF; ++m) {
    const int e = e0 + m;
    pc[m] = (e < e1) ? ldg(ci + e) : 0;
#pragma unroll
    for (int r = 0; r < B; ++r) pv[m][r] = (e < e1 && q < B) ? __ldcs(val + (size_t)e * BB + q * B + r) : 0.0;
  }
  pdl_wait();
  pdl_trigger();
  if (!live) return;
  double a[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) a[r] = 0.0;
#pragma unroll
  for (int m = 0; m < PF; ++m) {
    if (e0 + m < e1 && q < B) {
      const double xq = ldg(x + (size_t)pc[m] * B + q);
#pragma unroll
      for (int r = 0; r < B; ++r) a[r] = fma(pv[m][r], xq, a[r]);
    }
  }
#pragma unroll 2
  for (int e = e0 + PF; e < e1; ++e) {
    const int c = ldg(ci + e);
    const double xq = (q < B) ? ldg(x + (size_t)c * B + q) : 0.0;
    col_accum8<B>(val + (size_t)e * BB, xq, q, a);
  }
  const double acc = reduce_scatter8(a, q, 0xFFu << ((threadIdx.x & 31) & ~7));
  if (q < B) {
    const size_t o = (size_t)row * B + q;
    y[o] = (MODE == 0) ? acc : (g[o] - acc);
  }
}

// a2 for 4x4 blocks, column-per-lane: lane q loads block column q (two 16-byte loads,
// column-major storage), multiplies by its own x_q (no broadcast), keeps 4 row partial
// sums and reduce-scatters once per block row.  MODE 0: y = A x; MODE 1: y = g - A x.
template <int MODE>
// rows != null: process only the n rows listed (distributed mode: the slab-interior rows
// while the z halo is in flight, then the boundary rows)
__global__ void __launch_bounds__(MSP_SPMV_TPB) bsr_spmv4c_kernel(int n, const int* __restrict__ rp,
                                                         const int* __restrict__ ci,
                                                         const double* __restrict__ val,
                                                         const double* __restrict__ x,
                                                         const double* __restrict__ g,
                                                         double* __restrict__ y,
                                                         const int* __restrict__ rows = nullptr) {
  PDL_ENTRY();
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int slot = gtid >> 2, q = threadIdx.x & 3;
  if (slot >= n) return;                      // whole 4-lane groups exit together
  const int row = rows ? ldg(rows + slot) : slot;
  const int e0 = ldg(rp + row), e1 = ldg(rp + row + 1);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll 2
  for (int e = e0; e < e1; ++e) {
    const int c = ldg(ci + e);
    const double xq = ldg(x + (size_t)c * 4 + q);
    const double2* colp = reinterpret_cast<const double2*>(val + (size_t)e * 16 + q * 4);
    const double2 lo = ldstream2(colp), hi = ldstream2(colp + 1);
    a0 = fma(lo.x, xq, a0);
    a1 = fma(lo.y, xq, a1);
    a2 = fma(hi.x, xq, a2);
    a3 = fma(hi.y, xq, a3);
  }
  const double acc = reduce_scatter4(a0, a1, a2, a3, q, 0xFu << ((threadIdx.x & 31) & ~3));
  const size_t o = (size_t)row * 4 + q;
  y[o] = (MODE == 0) ? acc : (g[o] - acc);
}

// a8 for 4x4 blocks: r = g - A[:,P] x with the contiguous pressure columns Pcol (one
// 32 B sector per block entry).  Entry-per-lane: lane q of the row's 4-lane group
// takes entries e0+q, e0+q+4, ... (the group reads 128 contiguous bytes of Pcol and
// 4 consecutive ci per round), accumulates all 4 rows, then one reduce-scatter.
__global__ void __launch_bounds__(256) pcol_resid4_kernel(int n, const int* __restrict__ rp,
                                                          const int* __restrict__ ci,
                                                          const double* __restrict__ pcol,
                                                          const double* __restrict__ x,
                                                          const double* __restrict__ g,
                                                          double* __restrict__ y,
                                                          const int* __restrict__ rows = nullptr) {
  PDL_ENTRY();
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int slot = gtid >> 2, q = threadIdx.x & 3;
  if (slot >= n) return;                      // whole 4-lane groups exit together
  const int row = rows ? ldg(rows + slot) : slot;
  const int e0 = ldg(rp + row), e1 = ldg(rp + row + 1);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll 2
  for (int e = e0 + q; e < e1; e += 4) {
    const double xc = ldg(x + ldg(ci + e));
    const double2* cp = reinterpret_cast<const double2*>(pcol + (size_t)e * 4);
    const double2 lo = ldstream2(cp), hi = ldstream2(cp + 1);
    a0 = fma(lo.x, xc, a0);
    a1 = fma(lo.y, xc, a1);
    a2 = fma(hi.x, xc, a2);
    a3 = fma(hi.y, xc, a3);
  }
  const double acc = reduce_scatter4(a0, a1, a2, a3, q, 0xFu << ((threadIdx.x & 31) & ~3));
  const size_t o = (size_t)row * 4 + q;
  y[o] = g[o] - acc;
}

// a8, 4x4 blocks, ELL layout of the pressure columns: pe[(k*ld + row)*4 + j] = A[row, col k]
// column 0 entry j, ce[k*ld + row] = that column, k < w (padding: zero block column, ce =
// row).  One thread per row: the w column indices and 32-byte pressure columns are
// immutable and loaded before the PDL wait (coalesced: a warp reads 1 KB of pe per k),
// then w independent gathers of x_p, one 32-byte g load and one 32-byte y store.
constexpr int kEllMax = 8;
#ifndef MSP_A8_MINB
#define MSP_A8_MINB 1
#endif
__global__ void __launch_bounds__(MSP_A8_TPB, MSP_A8_MINB) pcol_resid_ell4_kernel(int n, int ld, int w, const int* __restrict__ ce,
                                                              const double* __restrict__ pe,
                                                              const double* __restrict__ x,
                                                              const double* __restrict__ g,
                                                              double* __restrict__ y,
                                                              const int* __restrict__ rows = nullptr) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = t < n;
  const int row = live ? (rows ? ldg(rows + t) : t) : 0;
  int c[kEllMax];
  double2 lo[kEllMax], hi[kEllMax];
#pragma unroll
  for (int k = 0; k < kEllMax; ++k) {
    if (live && k < w) {
      const size_t o = (size_t)k * ld + row;
      c[k] = ldg(ce + o);
      const double2* q = reinterpret_cast<const double2*>(pe + o * 4);
      lo[k] = ldstream2(q);
      hi[k] = ldstream2(q + 1);
    }
  }
  pdl_wait();
  pdl_trigger();
  if (!live) return;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
  for (int k = 0; k < kEllMax; ++k) {
    if (k < w) {
      const double xc = ldg(x + c[k]);
      a0 = fma(lo[k].x, xc, a0);
      a1 = fma(lo[k].y, xc, a1);
      a2 = fma(hi[k].x, xc, a2);
      a3 = fma(hi[k].y, xc, a3);
    }
  }
  const double2* gp = reinterpret_cast<const double2*>(g + (size_t)row * 4);
  const double2 g0 = __ldg(gp), g1 = __ldg(gp + 1);
  double2* yp = reinterpret_cast<double2*>(y + (size_t)row * 4);
  yp[0] = make_double2(g0.x - a0, g0.y - a1);
  yp[1] = make_double2(g1.x - a2, g1.y - a3);
}

// ELL copy of the pressure columns (setup and msp_update): one thread per row.
__global__ void pcol_ell_fill_kernel(int n, int w, const int* __restrict__ rp, const int* __restrict__ ci,
                                     const double* __restrict__ pcol, int* __restrict__ ce, double* __restrict__ pe) {
  PDL_ENTRY();
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  const int e0 = rp[row], e1 = rp[row + 1];
  for (int k = 0; k < w; ++k) {
    const size_t o = (size_t)k * n + row;
    const int e = e0 + k;
    ce[o] = (e < e1) ? ci[e] : row;
#pragma unroll
    for (int j = 0; j < 4; ++j) pe[o * 4 + j] = (e < e1) ? pcol[(size_t)e * 4 + j] : 0.0;
  }
}

// ---------------------------------------------------------------------------
// a3: pressure restriction with decoupling weights (R4): rp_l0[dst[c]] = sum_k
// W[c][k] * g[c*B+k]; dst maps internal cell positions to level-0 rows.
// ---------------------------------------------------------------------------
// One thread per LEVEL-0 row i (coalesced writes); src[i] = the internal cell of row i
// (its W row and g block are one aligned 32-byte sector each for b = 4).
// Fused first color of the level-0 pre-sweep (zero guess): when x0 != null, also
// x0[i] = b_i / a_ii for rows of color 1 (i < c1_end), 0 otherwise.
template <int B>
__global__ void restrict_pressure_kernel(int n, const double* __restrict__ W,
                                         const double* __restrict__ g, const int* __restrict__ src,
                                         double* __restrict__ rp, double* __restrict__ x0,
                                         const double* __restrict__ diag0, int c1_end, HaloPack pk) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = i < n;
  // PDL prologue: the cell map, its weight row and the level-0 diagonal are immutable
  const int c = live ? ldg(src + i) : 0;
  double wk[B];
#pragma unroll
  for (int k = 0; k < B; ++k) wk[k] = live ? ldg(W + (size_t)c * B + k) : 0.0;
  const double d = (live && x0 && i < c1_end) ? ldg(diag0 + i) : 1.0;
  pdl_wait();
  pdl_trigger();
  if (!live) return;
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < B; ++k) s = fma(wk[k], ldg(g + (size_t)c * B + k), s);
  rp[i] = s;
  if (x0) {
    const double xv = (i < c1_end) ? s / d : 0.0;
    x0[i] = xv;
    halo_pack(pk, i, xv);
  }
}

// gather of the level-0 correction into cell order: wp[c] = x0[dst[c]]
__global__ void gather_kernel(int n, const int* __restrict__ idx, const double* __restrict__ src,
                              double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = (c < n) ? ldg(idx + c) : 0;      // immutable map: before the PDL wait
  pdl_wait();
  pdl_trigger();
  if (c < n) out[c] = ldg(src + k);
}


// NEXT-4 comparison smoothers (reading R13), on the color-permuted SELL layout.
// PJAC-NO: x_i = (b_i - sum_{j != i} a_ij xo_j) / a_ii for every row (xo: the values at
// the start of the sweep; LPR lanes per row as sell_row_kernel).
template <int LPR>
__global__ void __launch_bounds__(128) sell_jacobi_kernel(int s_first, int s_end,
                                                          const int* __restrict__ slice_row,
                                                          const int* __restrict__ slice_off,
                                                          const int* __restrict__ col,
                                                          const double* __restrict__ val,
                                                          const double* __restrict__ diag,
                                                          const double* __restrict__ b,
                                                          const double* __restrict__ xo,
                                                          double* __restrict__ x) {
  PDL_ENTRY();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = s_first + t / (kSell * LPR);
  if (s >= s_end) return;                      // whole warps (32*LPR threads per slice)
  const int rem = t % (kSell * LPR);
  const int l = rem / LPR, u = rem % LPR;
  const int row = ldg(slice_row + s) + l;
  const int o0 = ldg(slice_off + s), w = (ldg(slice_off + s + 1) - o0) / kSell;
  double acc = 0.0;
#pragma unroll 4
  for (int k = u; k < w; k += LPR) {
    const int o = o0 + k * kSell + l;
    acc = fma(ldg(val + o), ldg(xo + ldg(col + o)), acc);
  }
#pragma unroll
  for (int m = LPR / 2; m; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
  if (u == 0 && row < ldg(slice_row + s + 1)) x[row] = (ldg(b + row) - acc) / ldg(diag + row);
}

// PGS-NO (hybrid Jacobi/GS): one warp per chunk of K natural-order rows
// [cK, cK+K), relaxed in order (descending for the post-sweep); a coupling to a row of
// the same chunk relaxed earlier in this sweep uses its new value, every other coupling
// the start-of-sweep value xo.  The chunk is processed in groups of 32 rows, lane l
// holding the row at sweep position 32*g + l: each lane first sums, in parallel, its
// couplings to start-of-sweep values and to rows finished in earlier groups, and writes
// its couplings to earlier rows of the same group into a 32x32 shared tile; the group's
// triangle is then resolved in 32 steps (lane t finishes, broadcasts x_t by shuffle,
// later lanes add S[l][t] x_t).  perm/inv map natural <-> permuted rows;
// row_start/row_width locate a row's SELL entries.
// (K < 16: the thread-per-chunk variant below keeps the lanes busy.)
constexpr int kHgsWarps = 4;
__global__ void __launch_bounds__(32 * kHgsWarps) hybrid_gs_kernel(int n, int K, int asc,
                                                        const int* __restrict__ perm,
                                                        const int* __restrict__ inv,
                                                        const int* __restrict__ row_start,
                                                        const int* __restrict__ row_width,
                                                        const int* __restrict__ col,
                                                        const double* __restrict__ val,
                                                        const double* __restrict__ diag,
                                                        const double* __restrict__ b,
                                                        const double* __restrict__ xo, double* x) {
  __shared__ double S[kHgsWarps][32][33];
  PDL_ENTRY();
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * kHgsWarps + wi;
  const int q0 = c * K;
  if (q0 >= n) return;                                  // whole warp
  const int q1 = min(n, q0 + K);
  const int len = q1 - q0;
  double* Sw = &S[wi][lane][0];
  for (int g0 = 0; g0 < len; g0 += 32) {
    const int pos = g0 + lane;
    const bool active = pos < len;
    const int q = asc ? q0 + pos : q1 - 1 - pos;
#pragma unroll 4
    for (int t = 0; t < 32; ++t) Sw[t] = 0.0;
    double acc = 0.0, bv = 0.0, d = 1.0;
    int p = 0;
    if (active) {
      p = ldg(perm + q);
      const int o0 = ldg(row_start + p), w = ldg(row_width + p);
      for (int k = 0; k < w; ++k) {
        const int o = o0 + k * kSell;
        const int j = ldg(col + o);
        const int qj = ldg(inv + j);
        const double a = ldg(val + o);
        const int pj = asc ? qj - q0 : q1 - 1 - qj;     // sweep position of row j
        if (qj >= q0 && qj < q1 && pj < pos) {           // relaxed earlier in this sweep
          if (pj >= g0) Sw[pj - g0] = a;                 // same group: resolved below
          else acc = fma(a, x[j], acc);                  // earlier group: final
        } else {
          acc = fma(a, ldg(xo + j), acc);
        }
      }
      bv = ldg(b + p);
      d = 1.0 / ldg(diag + p);                          // one division per row, outside the chain
    }
    __syncwarp();
    double xi = 0.0;
    for (int t = 0; t < 32; ++t) {
      const double xt = __shfl_sync(0xffffffffu, (bv - acc) * d, t);
      if (lane == t) xi = xt;
      if (lane > t) acc = fma(Sw[t], xt, acc);
    }
    if (active) x[p] = xi;
    __syncwarp();                                       // x of this group final for the next
  }
}

// PGS-NO for small chunks (K < 16): one thread relaxes its chunk row by row.
__global__ void __launch_bounds__(128) hybrid_gs_thread_kernel(int n, int K, int asc, const int* __restrict__ perm,
                                                               const int* __restrict__ inv,
                                                               const int* __restrict__ row_start,
                                                               const int* __restrict__ row_width,
                                                               const int* __restrict__ col,
                                                               const double* __restrict__ val,
                                                               const double* __restrict__ diag,
                                                               const double* __restrict__ b,
                                                               const double* __restrict__ xo, double* x) {
  PDL_ENTRY();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int q0 = c * K;
  if (q0 >= n) return;
  const int q1 = min(n, q0 + K);
  for (int t = 0; t < q1 - q0; ++t) {
    const int q = asc ? q0 + t : q1 - 1 - t;
    const int p = ldg(perm + q);
    const int o0 = ldg(row_start + p), w = ldg(row_width + p);
    double acc = 0.0;
    for (int k = 0; k < w; ++k) {
      const int o = o0 + k * kSell;
      const int j = ldg(col + o);
      const int qj = ldg(inv + j);
      const bool fresh = qj >= q0 && qj < q1 && (asc ? qj < q : qj > q);
      acc = fma(ldg(val + o), fresh ? x[j] : ldg(xo + j), acc);
    }
    x[p] = (ldg(b + p) - acc) / ldg(diag + p);
  }
}

// First color of a pre-sweep from the zero initial guess: x_i = b_i / a_ii for the
// rows of color 1 and x_i = 0 elsewhere (one pass over the whole level).
__global__ void pgs_init_kernel(int n, int c1_end, const double* __restrict__ diag,
                                const double* __restrict__ b, double* __restrict__ x) {
  PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  x[i] = (i < c1_end) ? ldg(b + i) / ldg(diag + i) : 0.0;
}

// ---------------------------------------------------------------------------
// a4/a5 with LPR lanes per row (coarse levels: few rows per color, wide Galerkin
// rows -> the per-row dependent load chain, not bandwidth, sets the time).  Lane u of
// a row handles SELL entries k = u, u+LPR, ...; the LPR partial sums are combined by
// shuffles.  Slices (32 rows) map to 32*LPR consecutive threads (whole warps).
// WRITE_R: also write the residual of the updated row, r = (b - sum_{j!=i}) - a_ii x_i
// (rows of the LAST pre-sweep color: their neighbours are final, so this is exactly
// the a5 residual, fused).  MODE_RES: residual only (rows of the other colors).
// ---------------------------------------------------------------------------
template <int LPR, bool WRITE_R, bool MODE_RES>
__global__ void __launch_bounds__(512) sell_row_kernel(int s_first, int s_end,
                                                       const int* __restrict__ slice_row,
                                                       const int* __restrict__ slice_off,
                                                       const int* __restrict__ col,
                                                       const double* __restrict__ val,
                                                       const double* __restrict__ diag,
                                                       const double* __restrict__ b,
                                                       double* __restrict__ x,
                                                       double* __restrict__ r) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = s_first + t / (kSell * LPR);
  if (s >= s_end) return;                      // whole warps (32*LPR threads per slice)
  const int rem = t % (kSell * LPR);
  const int l = rem / LPR, u = rem % LPR;
  const int r0 = ldg(slice_row + s), r1 = ldg(slice_row + s + 1);
  const int row = r0 + l;
  const int o0 = ldg(slice_off + s), w = (ldg(slice_off + s + 1) - o0) / kSell;
  // prologue (overlaps the predecessor kernel): the first PF matrix entries of this
  // lane and the diagonal are immutable
  constexpr int PF = (LPR == 1) ? MSP_SELL_PF1 : MSP_SELL_PFL;
  int pc[PF];
  double pv[PF];
#pragma unroll
  for (int m = 0; m < PF; ++m) {
    const int k = u + m * LPR;
    const int o = o0 + k * kSell + l;
    pc[m] = (k < w) ? ldg(col + o) : row;
    pv[m] = (k < w) ? ldg(val + o) : 0.0;
  }
  const double d = (row < r1) ? ldg(diag + row) : 1.0;
  pdl_wait();
  pdl_trigger();
  double acc = 0.0;
#pragma unroll
  for (int m = 0; m < PF; ++m) acc = fma(pv[m], x[pc[m]], acc);
  for (int k = u + PF * LPR; k < w; k += LPR) {
    const int o = o0 + k * kSell + l;
    acc = fma(ldg(val + o), x[ldg(col + o)], acc);
  }
#pragma unroll
  for (int m = LPR / 2; m; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
  if (u != 0 || row >= r1) return;
  if (MODE_RES) {
    r[row] = ldg(b + row) - fma(d, x[row], acc);
  } else {
    const double bs = ldg(b + row) - acc;
    const double xi = bs / d;
    x[row] = xi;
    if (WRITE_R) r[row] = fma(-d, xi, bs);
  }
}

// Level-0 form of sell_row_kernel<1, ...> on a uniform-width SELL layout (every slice
// W <= 8 wide): row = row_first + 32 (s - s_first) + l and entry k at s*32*W + 32 k + l are
// arithmetic, so the PDL prologue loads all of the row's matrix entries and its diagonal
// with no slice-metadata round trip.  Same per-row arithmetic and summation order.
template <bool WRITE_R, bool MODE_RES>
__global__ void __launch_bounds__(MSP_UNI_TPB) sell_row_uniform_kernel(int s_first, int s_end, int row_first, int row_end,
                                                               int W, const int* __restrict__ col,
                                                               const double* __restrict__ val,
                                                               const double* __restrict__ diag,
                                                               const double* __restrict__ b,
                                                               double* __restrict__ x, double* __restrict__ r,
                                                               HaloPack pk) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = s_first + t / kSell;
  if (s >= s_end) return;
  const int l = t % kSell;
  const int row = row_first + (s - s_first) * kSell + l;
  const size_t o0 = (size_t)s * kSell * W + l;
  int pc[8];
  double pv[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    pc[m] = (m < W) ? ldg(col + o0 + (size_t)m * kSell) : row;
    pv[m] = (m < W) ? ldg(val + o0 + (size_t)m * kSell) : 0.0;
  }
  const bool valid = row < row_end;
  const double d = valid ? ldg(diag + row) : 1.0;
  pdl_wait();
  pdl_trigger();
  if (!valid) return;
  double acc = 0.0;
#pragma unroll
  for (int m = 0; m < 8; ++m) acc = fma(pv[m], x[pc[m]], acc);
  if (MODE_RES) {
    r[row] = ldg(b + row) - fma(d, x[row], acc);
  } else {
    const double bs = ldg(b + row) - acc;
    const double xi = bs / d;
    x[row] = xi;
    halo_pack(pk, row, xi);
    if (WRITE_R) r[row] = fma(-d, xi, bs);
  }
}

// Trailing colors c_first..c_last of one level in ONE CTA: every row of these colors is
// owned by this CTA, so consecutive colors are separated by __syncthreads (global
// writes of the CTA are visible to the CTA after the barrier) instead of kernel
// boundaries.  Same per-row arithmetic as sell_row_kernel (LPR lanes per row).
// Ascending (pre-sweep) order if asc, descending otherwise.  WRITE_R on the last color
// of an ascending sweep writes the residual of its rows (see sell_row_kernel).
template <int LPR>
__global__ void __launch_bounds__(1024) sell_tail_kernel(int c_first, int c_last, int asc, int write_r,
                                                         const int* __restrict__ color_slice,
                                                         const int* __restrict__ slice_row,
                                                         const int* __restrict__ slice_off,
                                                         const int* __restrict__ col,
                                                         const double* __restrict__ val,
                                                         const double* __restrict__ diag,
                                                         const double* __restrict__ b, double* x,
                                                         double* __restrict__ r) {
  PDL_ENTRY();
  const int nc = c_last - c_first + 1;
  for (int step = 0; step < nc; ++step) {
    const int c = asc ? c_first + step : c_last - step;
    const bool wr = write_r && asc && step == nc - 1;
    const int s0 = ldg(color_slice + c), s1 = ldg(color_slice + c + 1);
    const int items = (s1 - s0) * kSell * LPR;
    for (int t0 = 0; t0 < items; t0 += blockDim.x) {     // uniform trip count: shuffles safe
      const int t = t0 + threadIdx.x;
      const bool in = t < items;
      const int s = s0 + (in ? t / (kSell * LPR) : 0);
      const int rem = t % (kSell * LPR);
      const int l = rem / LPR, u = rem % LPR;
      const int row = ldg(slice_row + s) + l;
      const int o0 = ldg(slice_off + s), w = in ? (ldg(slice_off + s + 1) - o0) / kSell : 0;
      double acc = 0.0;
      for (int k = u; k < w; k += LPR) {
        const int o = o0 + k * kSell + l;
        acc = fma(ldg(val + o), x[ldg(col + o)], acc);
      }
#pragma unroll
      for (int m = LPR / 2; m; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
      if (in && u == 0 && row < ldg(slice_row + s + 1)) {
        const double d = ldg(diag + row);
        const double bs = ldg(b + row) - acc;
        const double xi = bs / d;
        x[row] = xi;
        if (wr) r[row] = fma(-d, xi, bs);
      }
    }
    __syncthreads();
  }
}




// a6 coarsest GEMV with W warps per row (one CTA per row): the row's 16-byte pairs are
// spread over 32*W lanes (stride 32*W, U pairs in flight per lane; the first U issued
// before the PDL wait), so the 4.4k-row inverse keeps every SM busy with ~4x more loads
// in flight than warp-per-row; warp sums, then the W partial sums added in warp order
// through shared memory (deterministic).
template <int W, int U>
__global__ void __launch_bounds__(32 * W) gemv_row_kernel(int n, int ld, const double* __restrict__ Ainv,
                                                          const double* __restrict__ b, double* __restrict__ x) {
  __shared__ double part[W];
  const int row = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const double2* a = reinterpret_cast<const double2*>(Ainv + (size_t)row * ld);
  const double2* bb = reinterpret_cast<const double2*>(b);
  const int n2 = n >> 1;
  constexpr int S = 32 * W;
  double2 pa[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int j = t + S * u;
    pa[u] = (j < n2) ? ldstream2(a + j) : make_double2(0.0, 0.0);
  }
  pdl_wait();
  pdl_trigger();
  double acc = 0.0;
  for (int j0 = 0; j0 < n2; j0 += S * U) {
    if (j0 > 0) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = j0 + t + S * u;
        pa[u] = (j < n2) ? ldstream2(a + j) : make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + t + S * u;
      if (j < n2) {
        const double2 bv = __ldg(bb + j);
        acc = fma(pa[u].x, bv.x, fma(pa[u].y, bv.y, acc));
      }
    }
  }
  if ((n & 1) && t == 0) acc = fma(ldg(Ainv + (size_t)row * ld + n - 1), ldg(b + n - 1), acc);
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) part[w] = acc;
  __syncthreads();
  if (t == 0) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < W; ++k) s += part[k];
    x[row] = s;
  }
}

// a5 part 2: restriction b_{l+1}[I] = sum_{i in I} r_i (P^T, piecewise-constant P).
// (fused: xc != null -> first color of the next level's pre-sweep from the zero guess)
__global__ void restrict_kernel(int nc, const int* __restrict__ pp, const int* __restrict__ pi,
                                const double* __restrict__ r, double* __restrict__ bc,
                                double* __restrict__ xc, const double* __restrict__ dc, int c1_end) {
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = I < nc;
  // PDL prologue: member lists (<= 4 members for 2-pass NPAIR) and diagonal are immutable
  const int e0 = live ? ldg(pp + I) : 0, e1 = live ? ldg(pp + I + 1) : 0;
  int m[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) m[k] = (e0 + k < e1) ? ldg(pi + e0 + k) : -1;
  const double d = (live && xc && I < c1_end) ? ldg(dc + I) : 1.0;
  pdl_wait();
  pdl_trigger();
  if (!live) return;
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (m[k] >= 0) s += ldg(r + m[k]);
  for (int e = e0 + 4; e < e1; ++e) s += ldg(r + ldg(pi + e));
  bc[I] = s;
  if (xc) xc[I] = (I < c1_end) ? s / d : 0.0;
}

// a7: prolongation and correction x_i += e[agg(i)].
__global__ void prolong_kernel(int n, const int* __restrict__ agg, const double* __restrict__ e,
                               double* __restrict__ x, HaloPack pk) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int a = (i < n) ? ldg(agg + i) : 0;      // immutable map: before the PDL wait
  pdl_wait();
  pdl_trigger();
  if (i < n) {
    const double xv = x[i] + ldg(e + a);
    x[i] = xv;
    halo_pack(pk, i, xv);
  }
}


__global__ void diag_solve_kernel(int n, const double* __restrict__ d, const double* __restrict__ b,
                                  double* __restrict__ x) {
  PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = ldg(b + i) / ldg(d + i);
}



// ---------------------------------------------------------------------------
// a9 (K4), general form for aggregate blocks of any size (pair_passes >= 3): BILU(0)
// substitution in ABMC order (R5).  One team of TS lanes per
// aggregate block (blocks of one color are independent); the <= 4 cells of a block
// are processed in order by the team.  Factors: rows in internal positions, L part
// = entries [rp[i], dg[i]), U part = (dg[i], rp[i+1]), slot dg[i] holds D~_i^-1;
// blocks column-major.
//   forward  (FWD):  y_i = r_i - sum_{k<i} L_ik y_k             (in place in v)
//   backward (BWD):  x_i = D~_i^-1 (y_i - sum_{j>i} U_ij x_j)   (in place in v),
//                    and z_i = x_i + (pressure slot) wp[i]  (Alg. 1 line 6: w += R r)
//   FUSED: forward then backward within the block (last color).
// ---------------------------------------------------------------------------
template <int B, bool FWD, bool BWD>
__global__ void __launch_bounds__(128) bilu_color_kernel(int b_first, int b_end,
                                                         const int* __restrict__ blk_ptr,
                                                         const int* __restrict__ rp,
                                                         const int* __restrict__ ci,
                                                         const int* __restrict__ dg,
                                                         const double* __restrict__ F,
                                                         double* v,
                                                         const double* __restrict__ wp,
                                                         double* __restrict__ z) {
  PDL_ENTRY();
  constexpr int TS = (B <= 4) ? 4 : 8;
  constexpr int BB = B * B;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int blk = b_first + gtid / TS;
  const int q = threadIdx.x % TS;
  const int lane = threadIdx.x & 31;
  const int base = lane - q;
  const unsigned mask = ((1u << TS) - 1u) << base;
  if (blk >= b_end) return;
  const int c0 = ldg(blk_ptr + blk), c1 = ldg(blk_ptr + blk + 1);
  if (FWD) {
    for (int i = c0; i < c1; ++i) {
      double acc = 0.0;
      const int d = ldg(dg + i);
      for (int e = ldg(rp + i); e < d; ++e) {
        const int k = ldg(ci + e);
        const double yq = (q < B) ? v[(size_t)k * B + q] : 0.0;
        const double* blkF = F + (size_t)e * BB;
#pragma unroll
        for (int t = 0; t < B; ++t) {
          const double yt = __shfl_sync(mask, yq, base + t);
          if (q < B) acc = fma(ldg(blkF + t * B + q), yt, acc);
        }
      }
      if (q < B) v[(size_t)i * B + q] -= acc;
      __syncwarp(mask);
    }
  }
  if (BWD) {
    for (int i = c1 - 1; i >= c0; --i) {
      double acc = 0.0;
      const int d = ldg(dg + i);
      const int e1 = ldg(rp + i + 1);
      for (int e = d + 1; e < e1; ++e) {
        const int j = ldg(ci + e);
        const double xq = (q < B) ? v[(size_t)j * B + q] : 0.0;
        const double* blkF = F + (size_t)e * BB;
#pragma unroll
        for (int t = 0; t < B; ++t) {
          const double xt = __shfl_sync(mask, xq, base + t);
          if (q < B) acc = fma(ldg(blkF + t * B + q), xt, acc);
        }
      }
      const double tq = (q < B) ? (v[(size_t)i * B + q] - acc) : 0.0;
      const double* Di = F + (size_t)d * BB;
      double xi = 0.0;
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const double tu = __shfl_sync(mask, tq, base + u);
        if (q < B) xi = fma(ldg(Di + u * B + q), tu, xi);
      }
      if (q < B) {
        v[(size_t)i * B + q] = xi;
        z[(size_t)i * B + q] = xi + ((q == 0) ? ldg(wp + i) : 0.0);
      }
      __syncwarp(mask);
    }
  }
}

// ---------------------------------------------------------------------------
// a9 v2: BILU(0) color phase with one lane group (TS lanes) per CELL of an aggregate
// block (<= MAXC cells): team = MAXC*TS lanes.  Phase 1 gathers, for every cell of
// the block in parallel, the EXTERNAL part of its L (forward) or U (backward) sum,
// whose operands are final (earlier / later colors).  Phase 2 resolves the intra-block
// triangle (<= MAXC-1 coupled predecessors) in order, passing the finished cell
// vectors through register shuffles.  Same arithmetic as bilu_color_kernel, only
// the summation order differs (external before intra-block terms).
// ---------------------------------------------------------------------------
template <int B, int MAXC, bool FWD, bool BWD, bool WFULL = false, bool PF = kBiluPrefetch>
__global__ void __launch_bounds__(128, (B <= 4) ? MSP_BILU_MINB : 8) bilu_block_kernel(int b_first, int b_end,
                                                         const int* __restrict__ blk_ptr,
                                                         const int* __restrict__ rp,
                                                         const int* __restrict__ ci,
                                                         const int* __restrict__ dg,
                                                         const int* __restrict__ cnt,
                                                         const int4* __restrict__ islot,
                                                         const double* __restrict__ F,
                                                         double* v,
                                                         const double* __restrict__ wp,
                                                         double* __restrict__ z,
                                                         const int2* __restrict__ slots,
                                                         double* __restrict__ sbuf) {
  constexpr int TS = (B <= 4) ? 4 : 8;
  constexpr int TM = MAXC * TS;
  static_assert(TM <= 32, "team must fit in a warp");
  constexpr int BB = B * B;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int blk = b_first + gtid / TM;
  const int lane = threadIdx.x & 31;
  const int tl = lane % TM;                 // lane within team
  const int cq = tl / TS, q = tl % TS;      // cell slot, row
  const int tbase = lane - tl;              // first lane of the team
  const int cbase = lane - q;               // first lane of this cell group
  const unsigned tmask = (TM == 32) ? 0xffffffffu : (((1u << TM) - 1u) << tbase);
  const unsigned cmask = ((1u << TS) - 1u) << cbase;
  if (blk >= b_end) return;
  const int c0 = ldg(blk_ptr + blk), c1 = ldg(blk_ptr + blk + 1);
  const int nc = c1 - c0;
  const bool valid = cq < nc;
  const int i = c0 + (valid ? cq : 0);
  const bool act = valid && q < B;
  double t = 0.0;                           // working value of row q of cell i
  // cnt[i] = (#external L entries) | (#intra-block U entries << 8), from setup
  const int cn = valid ? ldg(cnt + i) : 0;
  // intra-block slots: entry of (i, c0 + s) (diagonal at s = cq), immutable: loaded and
  // the needed factor blocks prefetched into L1 before the PDL wait, so the triangle
  // steps below never wait on a column search
  int sl[4] = {-1, -1, -1, -1};
  if (MAXC > 1 && valid) {
    const int4 s4 = __ldg(islot + i);
    sl[0] = s4.x; sl[1] = s4.y; sl[2] = s4.z; sl[3] = s4.w;
#pragma unroll
    for (int sidx = 0; sidx < MAXC; ++sidx) {
      const bool need = (FWD && sidx < cq) || (BWD && sidx >= cq);
      if (need && sl[sidx] >= 0 && q * 4 < BB)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(F + (size_t)sl[sidx] * BB + q * 4));
    }
  }
  // distributed mode: send positions of this cell (the halo of this color phase is packed
  // here, not by a separate kernel)
  const int2 sl2 = (slots && valid) ? __ldg(slots + i) : make_int2(-1, -1);
  // PDL prologue (4x4 blocks): indices and factor columns of the first PFE external
  // entries are immutable -> issued before the wait, overlapping the previous kernel
  constexpr int PFE = (B == 4 && PF) ? MSP_BILU_PFE : 0;
  int pk[PFE > 0 ? PFE : 1];
  double2 plo[PFE > 0 ? PFE : 1], phi[PFE > 0 ? PFE : 1];
  int px0 = 0, px1 = 0;
  if constexpr (PFE > 0) {
    if (FWD) {
      px0 = valid ? ldg(rp + i) : 0;
      px1 = px0 + (cn & 0xff);
    } else {
      px0 = (valid ? ldg(dg + i) : 0) + 1 + (cn >> 8);
      px1 = valid ? ldg(rp + i + 1) : 0;
    }
#pragma unroll
    for (int m = 0; m < PFE; ++m) {
      const int e = px0 + m;
      pk[m] = (e < px1) ? ldg(ci + e) : -1;
      if (e < px1) {
        const double2* cp = reinterpret_cast<const double2*>(F + (size_t)e * 16 + q * 4);
        plo[m] = ldstream2(cp);
        phi[m] = ldstream2(cp + 1);
      } else {
        plo[m] = make_double2(0.0, 0.0);
        phi[m] = plo[m];
      }
    }
  }
  pdl_wait();
  pdl_trigger();
  if (FWD) {
    const int e0 = valid ? ldg(rp + i) : 0;
    const int d = valid ? ldg(dg + i) : 0;
    const int eext = e0 + (cn & 0xff);       // [e0, eext): external L; [eext, d): intra L
    double acc = 0.0;
    if constexpr (B == 4) {                 // column-per-lane: 2 x 16 B loads, own y_q
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int estart = e0;
      if constexpr (PFE > 0) {
#pragma unroll
        for (int m = 0; m < PFE; ++m) {
          if (pk[m] < 0) break;
          const double yq = ldg(v + (size_t)pk[m] * 4 + q);
          a0 = fma(plo[m].x, yq, a0);
          a1 = fma(plo[m].y, yq, a1);
          a2 = fma(phi[m].x, yq, a2);
          a3 = fma(phi[m].y, yq, a3);
        }
        estart = min(eext, e0 + PFE);
      }
#pragma unroll 2
      for (int ee = estart; ee < eext; ++ee) {
        const double yq = ldg(v + (size_t)ldg(ci + ee) * 4 + q);
        const double2* cp = reinterpret_cast<const double2*>(F + (size_t)ee * 16 + q * 4);
        const double2 lo = ldstream2(cp), hi = ldstream2(cp + 1);
        a0 = fma(lo.x, yq, a0);
        a1 = fma(lo.y, yq, a1);
        a2 = fma(hi.x, yq, a2);
        a3 = fma(hi.y, yq, a3);
      }
      acc = reduce_scatter4(a0, a1, a2, a3, q, cmask);
    } else if constexpr (B >= 5) {          // 8-lane column-per-lane
      double a8[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) a8[r] = 0.0;
      for (int ee = e0; ee < eext; ++ee) {
        const double yq = (q < B) ? ldg(v + (size_t)ldg(ci + ee) * B + q) : 0.0;
        col_accum8<B>(F + (size_t)ee * BB, yq, q, a8);
      }
      acc = reduce_scatter8(a8, q, cmask);
    } else {
#pragma unroll 2
      for (int ee = e0; ee < eext; ++ee) {  // external L part: columns before the block
        const int k = ldg(ci + ee);
        const double yq = (q < B) ? ldg(v + (size_t)k * B + q) : 0.0;
        const double* blkF = F + (size_t)ee * BB;
#pragma unroll
        for (int u = 0; u < B; ++u) {
          const double yu = __shfl_sync(cmask, yq, cbase + u);
          if (q < B) acc = fma(ldg(blkF + u * B + q), yu, acc);
        }
      }
    }
    t = act ? (v[(size_t)i * B + q] - acc) : 0.0;
    // intra-block triangle, cells in ascending order
#pragma unroll
    for (int sidx = 0; sidx < MAXC - 1; ++sidx) {
      // cell sidx is final: broadcast its vector, later cells subtract L_{i,sidx} y_sidx
      double contrib = 0.0;
      const bool use = valid && cq > sidx && sl[sidx] >= 0;
      const double* blkF = F + (size_t)(use ? sl[sidx] : 0) * BB;
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const double yu = __shfl_sync(tmask, t, tbase + sidx * TS + u);
        if (use && q < B) contrib = fma(ldg(blkF + u * B + q), yu, contrib);
      }
      if (use) t -= contrib;
    }
    if (act) {
      v[(size_t)i * B + q] = t;
      if (!BWD) {
        if (sl2.x >= 0) sbuf[(size_t)sl2.x * B + q] = t;
        if (sl2.y >= 0) sbuf[(size_t)sl2.y * B + q] = t;
      }
    }
    __syncwarp(tmask);
  }
  if (BWD) {
    if (!FWD) t = act ? v[(size_t)i * B + q] : 0.0;
    const int d = valid ? ldg(dg + i) : 0;
    const int e1 = valid ? ldg(rp + i + 1) : 0;
    const int ei = d + 1 + (cn >> 8);        // (d, ei): intra U; [ei, e1): external U
    double acc = 0.0;
    if constexpr (B == 4) {                  // column-per-lane (see the forward part)
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int estart = ei;
      if constexpr (PFE > 0) {
        if (!FWD) {                              // (fused colors: no external U)
#pragma unroll
          for (int m = 0; m < PFE; ++m) {
            if (pk[m] < 0) break;
            const double xq = ldg(v + (size_t)pk[m] * 4 + q);
            a0 = fma(plo[m].x, xq, a0);
            a1 = fma(plo[m].y, xq, a1);
            a2 = fma(phi[m].x, xq, a2);
            a3 = fma(phi[m].y, xq, a3);
          }
          estart = min(e1, ei + PFE);
        }
      }
#pragma unroll 2
      for (int e = estart; e < e1; ++e) {
        const double xq = ldg(v + (size_t)ldg(ci + e) * 4 + q);
        const double2* cp = reinterpret_cast<const double2*>(F + (size_t)e * 16 + q * 4);
        const double2 lo = ldstream2(cp), hi = ldstream2(cp + 1);
        a0 = fma(lo.x, xq, a0);
        a1 = fma(lo.y, xq, a1);
        a2 = fma(hi.x, xq, a2);
        a3 = fma(hi.y, xq, a3);
      }
      acc = reduce_scatter4(a0, a1, a2, a3, q, cmask);
    } else if constexpr (B >= 5) {           // 8-lane column-per-lane
      double a8[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) a8[r] = 0.0;
      for (int e = ei; e < e1; ++e) {
        const double xq = (q < B) ? ldg(v + (size_t)ldg(ci + e) * B + q) : 0.0;
        col_accum8<B>(F + (size_t)e * BB, xq, q, a8);
      }
      acc = reduce_scatter8(a8, q, cmask);
    } else {
#pragma unroll 2
      for (int e = ei; e < e1; ++e) {        // external U part: columns after the block
        const int j = ldg(ci + e);
        const double xq = (q < B) ? ldg(v + (size_t)j * B + q) : 0.0;
        const double* blkF = F + (size_t)e * BB;
#pragma unroll
        for (int u = 0; u < B; ++u) {
          const double xu = __shfl_sync(cmask, xq, cbase + u);
          if (q < B) acc = fma(ldg(blkF + u * B + q), xu, acc);
        }
      }
    }
    t -= acc;
    const double* Dg = F + (size_t)(valid ? d : 0) * BB;
    double x = 0.0;
#pragma unroll
    for (int sidx = MAXC - 1; sidx >= 0; --sidx) {
      // cell sidx: x = D~^-1 t (its t is complete once all later cells were applied)
      double xs = 0.0;
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const double tu = __shfl_sync(tmask, t, tbase + sidx * TS + u);
        if (cq == sidx && act) xs = fma(ldg(Dg + u * B + q), tu, xs);
      }
      if (cq == sidx) x = xs;
      if (sidx == 0) break;
      // earlier cells subtract U_{i,sidx} x_sidx
      const bool use = valid && cq < sidx && sl[sidx] >= 0;
      const double* blkF = F + (size_t)(use ? sl[sidx] : 0) * BB;
      double contrib = 0.0;
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const double xu = __shfl_sync(tmask, xs, tbase + sidx * TS + u);
        if (use && q < B) contrib = fma(ldg(blkF + u * B + q), xu, contrib);
      }
      if (use) t -= contrib;
    }
    if (act) {
      v[(size_t)i * B + q] = x;
      if (sl2.x >= 0) sbuf[(size_t)sl2.x * B + q] = x;
      if (sl2.y >= 0) sbuf[(size_t)sl2.y * B + q] = x;
      // z = w + R r: WFULL -> w is a full cell vector (stages NPR), else only the
      // pressure correction wp (stages PR)
      z[(size_t)i * B + q] = x + (WFULL ? ldg(wp + (size_t)i * B + q) : ((q == 0) ? ldg(wp + i) : 0.0));
    }
  }
}

// ---------------------------------------------------------------------------
// NEXT-1: B_N stage (Alg. 1 line 2): one forward block Gauss-Seidel sweep on
// A_NN = Π_N^T A Π_N in the BILU (ABMC) order, zero initial guess (R12):
//   w_i = D_NN,i^-1 (r_N,i - sum_{k before i} A_NN,ik w_k).
// One launch per block color; team per aggregate block as bilu_block_kernel (lane q
// = row q of the cell; rows 1..B-1 are the N rows).  A's blocks are column-major; the
// N-N diagonal inverses Dn are (B-1)x(B-1) column-major per cell.  Output w is the full
// cell-interleaved vector with w_i[0] = 0 (pressure slot).
// ---------------------------------------------------------------------------
template <int B, int MAXC>
__global__ void __launch_bounds__(128) bgs_block_kernel(int b_first, int b_end,
                                                        const int* __restrict__ blk_ptr,
                                                        const int* __restrict__ rp,
                                                        const int* __restrict__ ci,
                                                        const int* __restrict__ dg,
                                                        const int* __restrict__ cnt,
                                                        const double* __restrict__ A,
                                                        const double* __restrict__ Dn,
                                                        const double* __restrict__ r,
                                                        double* __restrict__ w) {
  PDL_ENTRY();
  constexpr int TS = (B <= 4) ? 4 : 8;
  constexpr int TM = MAXC * TS;
  constexpr int BB = B * B;
  constexpr int NC = B - 1;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int blk = b_first + gtid / TM;
  const int lane = threadIdx.x & 31;
  const int tl = lane % TM;
  const int cq = tl / TS, q = tl % TS;
  const int tbase = lane - tl, cbase = lane - q;
  const unsigned tmask = (TM == 32) ? 0xffffffffu : (((1u << TM) - 1u) << tbase);
  const unsigned cmask = ((1u << TS) - 1u) << cbase;
  if (blk >= b_end) return;
  const int c0 = ldg(blk_ptr + blk), c1 = ldg(blk_ptr + blk + 1);
  const int nc = c1 - c0;
  const bool valid = cq < nc;
  const int i = c0 + (valid ? cq : 0);
  const bool act = valid && q >= 1 && q < B;       // N rows
  const int cn = valid ? ldg(cnt + i) : 0;
  const int e0 = valid ? ldg(rp + i) : 0;
  const int d = valid ? ldg(dg + i) : 0;
  const int eext = e0 + (cn & 0xff);
  double acc = 0.0;
  for (int e = e0; e < eext; ++e) {                 // external part (earlier colors)
    const int k = ldg(ci + e);
    const double wq = (q >= 1 && q < B) ? w[(size_t)k * B + q] : 0.0;
    const double* blkA = A + (size_t)e * BB;
#pragma unroll
    for (int u = 1; u < B; ++u) {
      const double wu = __shfl_sync(cmask, wq, cbase + u);
      if (act) acc = fma(ldg(blkA + u * B + q), wu, acc);
    }
  }
  double t = act ? (ldg(r + (size_t)i * B + q) - acc) : 0.0;
  double wi = 0.0;
  int e = eext;                                     // intra-block entries (earlier cells)
  const double* Di = Dn + (size_t)(valid ? i : 0) * NC * NC;
#pragma unroll
  for (int sidx = 0; sidx < MAXC; ++sidx) {
    // cell sidx is complete: w_sidx = Dn^-1 t_sidx
    double ws = 0.0;
#pragma unroll
    for (int u = 1; u < B; ++u) {
      const double tu = __shfl_sync(tmask, t, tbase + sidx * TS + u);
      if (cq == sidx && act) ws = fma(ldg(Di + (u - 1) * NC + (q - 1)), tu, ws);
    }
    if (cq == sidx) wi = ws;
    if (sidx == MAXC - 1) break;
    const bool use = valid && cq > sidx && e < d && ldg(ci + e) == c0 + sidx;
    const double* blkA = A + (size_t)(use ? e : 0) * BB;
    double contrib = 0.0;
#pragma unroll
    for (int u = 1; u < B; ++u) {
      const double wu = __shfl_sync(tmask, ws, tbase + sidx * TS + u);
      if (use && act) contrib = fma(ldg(blkA + u * B + q), wu, contrib);
    }
    if (use) { t -= contrib; ++e; }
  }
  if (valid && q < B) w[(size_t)i * B + q] = (q == 0) ? 0.0 : wi;
}

// w_i[0] = wp_i (adds the pressure correction into the pressure slots of a full vector)
__global__ void set_pressure_kernel(int n, int B, const double* __restrict__ wp, double* __restrict__ w) {
  PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) w[(size_t)i * B] = ldg(wp + i);
}

// ---------------------------------------------------------------------------
// SETUP on the GPU (NEXT-2): BILU(0) factorization (R5) of one ABMC block color, one
// thread per aggregate block (its cells in order), on row-major blocks in the internal
// order: for every L entry (i,k): A_ik <- A_ik D~_k^-1, then A_ij -= A_ik A_kj over the
// U entries (k,j) of row k that lie in row i's pattern; finally D~_i^-1 replaces the
// diagonal block (Gauss-Jordan, partial pivoting).  Exactly the host/oracle operation
// order with explicitly rounded multiplies and adds (no FMA contraction), so the
// factors are bit-identical to the host factorization (tests/test_gpu.py).
// ---------------------------------------------------------------------------
template <int B>
__device__ bool gj_invert(double* D) {           // in place, row-major B x B
  double a[B][B], r[B][B];
  for (int i = 0; i < B; ++i)
    for (int j = 0; j < B; ++j) { a[i][j] = D[i * B + j]; r[i][j] = (i == j) ? 1.0 : 0.0; }
  for (int k = 0; k < B; ++k) {
    int p = k;
    for (int i = k + 1; i < B; ++i) if (fabs(a[i][k]) > fabs(a[p][k])) p = i;
    if (a[p][k] == 0.0) return false;
    if (p != k)
      for (int j = 0; j < B; ++j) {
        const double t1 = a[k][j]; a[k][j] = a[p][j]; a[p][j] = t1;
        const double t2 = r[k][j]; r[k][j] = r[p][j]; r[p][j] = t2;
      }
    const double piv = a[k][k];                   // row divided by the pivot (IEEE division)
    for (int j = 0; j < B; ++j) { a[k][j] = __ddiv_rn(a[k][j], piv); r[k][j] = __ddiv_rn(r[k][j], piv); }
    for (int i = 0; i < B; ++i) {
      if (i == k) continue;
      const double f = a[i][k];
      if (f == 0.0) continue;
      for (int j = 0; j < B; ++j) {
        a[i][j] = __dsub_rn(a[i][j], __dmul_rn(f, a[k][j]));
        r[i][j] = __dsub_rn(r[i][j], __dmul_rn(f, r[k][j]));
      }
    }
  }
  for (int i = 0; i < B; ++i) for (int j = 0; j < B; ++j) D[i * B + j] = r[i][j];
  return true;
}

template <int B>
__global__ void bilu_factor_kernel(int b_first, int b_end, const int* __restrict__ blk_ptr,
                                   const int* __restrict__ rp, const int* __restrict__ ci,
                                   const int* __restrict__ dg, double* F, int* bad) {
  constexpr int BB = B * B;
  const int k = b_first + blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= b_end) return;
  double T[BB];
  for (int i = blk_ptr[k]; i < blk_ptr[k + 1]; ++i) {
    const int r0 = rp[i], r1 = rp[i + 1];
    for (int e = r0; e < dg[i]; ++e) {
      const int kk = ci[e];
      double* Lik = F + (size_t)e * BB;
      const double* Dk = F + (size_t)dg[kk] * BB;        // holds D~_k^-1
      for (int r = 0; r < B; ++r)
        for (int c = 0; c < B; ++c) {
          double sum = 0.0;
          for (int t = 0; t < B; ++t) sum = __dadd_rn(sum, __dmul_rn(Lik[r * B + t], Dk[t * B + c]));
          T[r * B + c] = sum;
        }
      for (int t = 0; t < BB; ++t) Lik[t] = T[t];
      int m = r0;                                         // row i's entries, ascending columns
      for (int f = dg[kk] + 1; f < rp[kk + 1]; ++f) {
        const int cj = ci[f];
        while (m < r1 && ci[m] < cj) ++m;
        if (m >= r1) break;
        if (ci[m] != cj) continue;
        const double* Ukj = F + (size_t)f * BB;
        double* Aij = F + (size_t)m * BB;
        for (int r = 0; r < B; ++r)
          for (int c = 0; c < B; ++c) {
            double sum = 0.0;
            for (int t = 0; t < B; ++t) sum = __dadd_rn(sum, __dmul_rn(Lik[r * B + t], Ukj[t * B + c]));
            Aij[r * B + c] = __dsub_rn(Aij[r * B + c], sum);
          }
      }
    }
    if (!gj_invert<B>(F + (size_t)dg[i] * BB)) atomicMax(bad, i);
  }
}

// internal-order row-major blocks from the caller's natural order: out[e] = in[src[e]]
template <int B>
__global__ void gather_blocks_kernel(int64_t nnzb, const int* __restrict__ src, const double* __restrict__ in,
                                     double* __restrict__ out) {
  constexpr int BB = B * B;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nnzb * BB) return;
  const int64_t e = t / BB;
  out[t] = ldg(in + (size_t)ldg(src + e) * BB + (t - e * BB));
}

// setup upload: row-major b x b blocks -> column-major (out[e][c*B + r] = in[e][r*B + c])
template <int B>
__global__ void transpose_blocks_kernel(int64_t nnzb, const double* __restrict__ in, double* __restrict__ out) {
  constexpr int BB = B * B;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nnzb * BB) return;
  const int64_t e = t / BB;
  const int k = (int)(t - e * BB);
  const int c = k / B, r = k - c * B;
  out[t] = ldg(in + (size_t)e * BB + r * B + c);
}

// ASMSP reuse: refresh A in the internal layout from the caller's
// natural-order row-major values: A_cm[e] = transpose(A_nat[src[e]]), Pcol[e] = column 0.
template <int B>
__global__ void refresh_values_kernel(int64_t nnzb, const int* __restrict__ src, const double* __restrict__ nat,
                                      double* __restrict__ Acm, double* __restrict__ Pcol) {
  PDL_ENTRY();
  constexpr int BB = B * B;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nnzb * BB) return;
  const int64_t e = t / BB;
  const int k = (int)(t - e * BB);          // destination index (column-major): k = c*B + r
  const int c = k / B, r = k - c * B;
  const double v = ldg(nat + (size_t)ldg(src + e) * BB + r * B + c);
  Acm[t] = v;
  if (c == 0) Pcol[e * B + r] = v;
}

// Distributed mode: scatter the allgathered level-1 right-hand side of every rank's owned
// aggregates into the replicated level-1 vector (fused: first color of the level-1
// pre-sweep from the zero guess when x1 != null).
__global__ void scatter_l1_kernel(int count, const int* __restrict__ idx, const double* __restrict__ recv,
                                  double* __restrict__ b1, double* __restrict__ x1, const double* __restrict__ d1,
                                  int c1_end) {
  PDL_ENTRY();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const int I = ldg(idx + t);
  if (I < 0) return;
  const double v = recv[t];
  b1[I] = v;
  if (x1) x1[I] = (I < c1_end) ? v / ldg(d1 + I) : 0.0;
}

__global__ void add_vec_kernel(int n, const double* __restrict__ a, const double* __restrict__ b,
                               double* __restrict__ out) {
  PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] + b[i];
}

__global__ void sqrt_kernel(const double* __restrict__ in, double* __restrict__ out) {
  PDL_ENTRY();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = sqrt(in[0]);
}

// ---------------------------------------------------------------------------
// a10 (K8): GMRES vector kernels with deterministic two-stage reductions.
// multidot: part[blk][i] = sum over this block's elements of V_i . w, i = 0..nv-1.
// ---------------------------------------------------------------------------
#ifndef MSP_RED_BLOCKS
#define MSP_RED_BLOCKS 592
#endif
#ifndef MSP_RED_THREADS
#define MSP_RED_THREADS 256
#endif
constexpr int kRedBlocks = MSP_RED_BLOCKS;     // 4 x 148 SMs
constexpr int kRedThreads = MSP_RED_THREADS;
constexpr int kMaxV = 32;

template <int NV>
__global__ void __launch_bounds__(kRedThreads) multidot_kernel(size_t N, int nv,
                                                               const double* __restrict__ V,
                                                               size_t ldv,
                                                               const double* __restrict__ w,
                                                               double* __restrict__ part) {
  PDL_ENTRY();
  double acc[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) acc[i] = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += stride) {
    const double wt = ldg(w + t);
#pragma unroll
    for (int i = 0; i < NV; ++i)
      if (i < nv) acc[i] = fma(ldg(V + i * ldv + t), wt, acc[i]);
  }
  __shared__ double sh[kRedThreads / 32][NV];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    if (i >= nv) break;
    double a = acc[i];
#pragma unroll
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) sh[wid][i] = a;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    double a = 0.0;
    for (int k = 0; k < kRedThreads / 32; ++k) a += sh[k][i];
    part[(size_t)blockIdx.x * kMaxV + i] = a;
  }
}

// second stage: out[i] = (accumulate ? out[i] : 0) + sum_blk part[blk][i]; if
// sqrt_last, out[nv-1] = sqrt(sum).  One block, one warp per output.
__global__ void reduce_parts_kernel(int nblk, int nv, const double* __restrict__ part,
                                    double* __restrict__ out, const double* __restrict__ addend,
                                    int sqrt_index) {
  PDL_ENTRY();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = wid; i < nv; i += nw) {
    double a = 0.0;
    for (int k = lane; k < nblk; k += 32) a += part[(size_t)k * kMaxV + i];
#pragma unroll
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) {
      if (i == sqrt_index) a = sqrt(a);
      out[i] = addend ? addend[i] + a : a;
    }
  }
}

// multi-axpy: w -= sum_i h[i] V_i  (or, with from_zero, w = sum_i h[i] V_i), with
// optional per-block partial of ||w||^2 into part[blk][slot].
template <int NV>
__global__ void __launch_bounds__(kRedThreads) multiaxpy_kernel(size_t N, int nv,
                                                                const double* __restrict__ V,
                                                                size_t ldv,
                                                                const double* __restrict__ h,
                                                                double* __restrict__ w,
                                                                int from_zero, double* part,
                                                                int slot) {
  PDL_ENTRY();
  __shared__ double hs[NV];
  for (int i = threadIdx.x; i < NV; i += blockDim.x) hs[i] = (i < nv) ? h[i] : 0.0;
  __syncthreads();
  double nrm = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += stride) {
    double a = from_zero ? 0.0 : w[t];
    if (from_zero) {
#pragma unroll
      for (int i = 0; i < NV; ++i)
        if (i < nv) a = fma(hs[i], ldg(V + i * ldv + t), a);
    } else {
#pragma unroll
      for (int i = 0; i < NV; ++i)
        if (i < nv) a = fma(-hs[i], ldg(V + i * ldv + t), a);
    }
    w[t] = a;
    nrm = fma(a, a, nrm);
  }
  if (part) {
    __shared__ double sh[kRedThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
    if (lane == 0) sh[wid] = nrm;
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = 0.0;
      for (int k = 0; k < kRedThreads / 32; ++k) a += sh[k];
      part[(size_t)blockIdx.x * kMaxV + slot] = a;
    }
  }
}

// ---------------------------------------------------------------------------
// a10 v2: fused CGS2 passes with in-kernel deterministic finalisation.
// Every block writes its partial sums to part[blk][0..nv); the last block to finish
// (atomic ticket) sums the partials in fixed block order 0..nblk-1 (deterministic
// for a fixed grid) and writes out[i] = addend[i] + sum (addend may be null),
// raw[i] = sum (optional), sqrt applied to out[sqrt_index].  ticket is reset for the
// next graph replay.
// ---------------------------------------------------------------------------
// partial sums of this CTA for vector slots [off, off + nv) -> part[blockIdx.x][off + i]
template <int NV>
__device__ __forceinline__ void block_partials(const double (&acc)[NV], int nv, double* part, int off = 0) {
  __shared__ double sh[32][NV];                  // up to 32 warps (1024-thread CTAs)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    if (i >= nv) break;
    double a = acc[i];
#pragma unroll
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) sh[wid][i] = a;
  }
  __syncthreads();
  const int nw = blockDim.x >> 5;               // (<= kRedThreads / 32 warps)
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    double a = 0.0;
    for (int k = 0; k < nw; ++k) a += sh[k][i];
    part[(size_t)blockIdx.x * kMaxV + off + i] = a;
  }
}

// The last CTA of the grid (all gridDim.x * gridDim.y CTAs) sums the partial rows
// 0..gridDim.x-1 for slots [0, nv) in fixed order.
__device__ __forceinline__ void finalize_partials(int nv, const double* part, double* out,
                                                  const double* addend, double* raw, int sqrt_index,
                                                  unsigned* ticket) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(ticket, 1u) == gridDim.x * gridDim.y - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = wid; i < nv; i += nw) {
    double a = 0.0;
    for (int k = lane; k < (int)gridDim.x; k += 32) a += __ldcg(part + (size_t)k * kMaxV + i);
#pragma unroll
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) {
      if (raw) raw[i] = a;
      double v = addend ? addend[i] + a : a;
      if (i == sqrt_index) v = sqrt(v);
      out[i] = v;
    }
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

// vector of EW doubles (EW = 2: one 16-byte load; EW = 1: 8-byte load)
template <int EW> struct VecT;
template <> struct VecT<1> {
  double x;
  __device__ static VecT ldre(const double* p, size_t t) {
    double v;
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p + t));
    return {v};
  }
  __device__ static VecT ld(const double* p, size_t t) { return {__ldg(p + t)}; }
  __device__ static VecT ldcg(const double* p, size_t t) { return {__ldcg(p + t)}; }
};
__device__ __forceinline__ double2 ld_nc_v2_volatile(const double* p) {   // L1-cached, never merged
  double2 v;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
template <> struct VecT<2> {
  double x, y;
  __device__ static VecT ldre(const double* p, size_t t) {
    const double2 v = ld_nc_v2_volatile(p + 2 * t);
    return {v.x, v.y};
  }
  __device__ static VecT ld(const double* p, size_t t) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(p) + t);
    return {v.x, v.y};
  }
  __device__ static VecT ldcg(const double* p, size_t t) {
    const double2 v = __ldcg(reinterpret_cast<const double2*>(p) + t);
    return {v.x, v.y};
  }
};
template <int EW> __device__ __forceinline__ double vdot(const VecT<EW>& a, const VecT<EW>& b, double acc);
template <> __device__ __forceinline__ double vdot<1>(const VecT<1>& a, const VecT<1>& b, double acc) {
  return fma(a.x, b.x, acc);
}
template <> __device__ __forceinline__ double vdot<2>(const VecT<2>& a, const VecT<2>& b, double acc) {
  return fma(a.x, b.x, fma(a.y, b.y, acc));
}
template <int EW> __device__ __forceinline__ void vaxpy(double c, const VecT<EW>& v, VecT<EW>& a);
template <> __device__ __forceinline__ void vaxpy<1>(double c, const VecT<1>& v, VecT<1>& a) { a.x = fma(c, v.x, a.x); }
template <> __device__ __forceinline__ void vaxpy<2>(double c, const VecT<2>& v, VecT<2>& a) {
  a.x = fma(c, v.x, a.x);
  a.y = fma(c, v.y, a.y);
}

// pass A: h = V^T w (nv vectors); NE = N / EW elements of EW doubles
template <int NV, int EW, int MINB = 2>
__global__ void __launch_bounds__(kRedThreads, MINB) cgs_dot_kernel(size_t NE, int nv, const double* __restrict__ V,
                                                                 size_t ldv, const double* __restrict__ w,
                                                                 double* part, double* out, const double* addend,
                                                                 double* raw, int sqrt_index, unsigned* ticket) {
  PDL_ENTRY();
  using T = VecT<EW>;
  // gridDim.y > 1: CTA row y handles vectors [y*NV, min(nv, (y+1)*NV))
  const int vbase = blockIdx.y * NV;
  const int nvl = min(NV, nv - vbase);
  const double* Vb = V + (size_t)vbase * ldv;
  double acc[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) acc[i] = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < NE; t += stride) {
    const T wt = T::ld(w, t);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      if (i < nvl) acc[i] = vdot<EW>(T::ld(Vb + i * ldv, t), wt, acc[i]);
      if (i % 16 == 15) asm volatile("" ::: "memory");   // <= 16 loads in flight (registers)
    }
  }
  block_partials<NV>(acc, nvl, part, vbase);
  finalize_partials(nv, part, out, addend, raw, sqrt_index, ticket);
}

// pass B (DOT=true): w <- w - V h and h2 = V^T w; pass C (DOT=false): w <- w - V h and
// ||w||^2.  16-byte loads (two elements per thread and step).  In pass B the basis is
// read twice per element pair by the same thread (axpy, then dot); the second read is
// an L1 hit, which keeps registers low (full occupancy) instead of holding NV values.
// NVD: the dot part covers only the first min(nv, NVD) vectors (the rest by a
// separate cgs_dot pass), so that NV=32 axpys stay register-light.
template <int NV, int EW, bool DOT, int NVD = NV, int MINB = 2>
__global__ void __launch_bounds__(kRedThreads, MINB) cgs_axpy_kernel(size_t NE, int nv, const double* __restrict__ V,
                                                                  size_t ldv, const double* __restrict__ h,
                                                                  double* __restrict__ w, double* part,
                                                                  double* out, const double* addend,
                                                                  double* raw, int sqrt_index, unsigned* ticket) {
  PDL_ENTRY();
  using T = VecT<EW>;
  __shared__ double hs[NV];
  for (int i = threadIdx.x; i < NV; i += blockDim.x) hs[i] = (i < nv) ? h[i] : 0.0;
  __syncthreads();
  double acc[DOT ? NVD : 1];
#pragma unroll
  for (int i = 0; i < (DOT ? NVD : 1); ++i) acc[i] = 0.0;
  const int nvd = nv < NVD ? nv : NVD;
  T* wT = reinterpret_cast<T*>(w);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < NE; t += stride) {
    T a = wT[t];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      if (i < nv) vaxpy<EW>(-hs[i], T::ld(V + i * ldv, t), a);
      if (i % 16 == 15) asm volatile("" ::: "memory");
    }
    wT[t] = a;
    if constexpr (DOT) {
#pragma unroll
      for (int i = 0; i < NVD; ++i) {  // re-read through L2 (.cg): not merged with the first read
        if (i < nvd) acc[i] = vdot<EW>(T::ldcg(V + i * ldv, t), a, acc[i]);
        if (i % 16 == 15) asm volatile("" ::: "memory");
      }
    } else {
      acc[0] = vdot<EW>(a, a, acc[0]);
    }
  }
  if constexpr (DOT) {
    block_partials<NVD>(acc, nvd, part);
    finalize_partials(nvd, part, out, addend, raw, sqrt_index, ticket);
  } else {
    block_partials<1>(acc, 1, part);
    finalize_partials(1, part, out, addend, raw, sqrt_index, ticket);
  }
}

// ---------------------------------------------------------------------------
// DCGS2 Arnoldi (orth = 2, reading R14): delayed re-orthogonalisation, two passes over
// the basis per step instead of CGS2's three.  Step k holds V[0..k) final and V[k]
// provisional = the previous step's once-projected vector u_{k-1}, stored UNnormalised
// (the method only needs it up to a factor, so no scaling pass), with its second-
// projection coefficients h2 = V[0..k)^T u_{k-1} and rho = ||u_{k-1} - V h2|| in the
// state st: st[0..k) = h2, st[kMaxV] = nu = 1, st[kMaxV+1] = rho; k = 0: V[0] final,
// nu = rho = 1.  w = A B V[k].
// Pass 1 (cgs_dot): a = V[0..k]^T w.  Pass 2 (this kernel), per element:
//   v_k = (nu V[k] - V[0..k) h2) / rho          (V[k] finalised in place)
//   u   = w - V[0..k) a[0..k) - c_k v_k,  c_k = (nu a_k - h2^T a[0..k)) / rho
// and, when DOT, the sums V[0..k)^T u, v_k^T u, u^T u (slots 0..k-1, k, k+1); without
// DOT the caller gets them from cgs_dot over V[0..k+1] (u is stored in the slot V[k+1]).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dcgs_scalars(int k, const double* a, const double* st, double& nu, double& rho,
                                             double& ck) {
  nu = k ? st[kMaxV] : 1.0;
  rho = k ? st[kMaxV + 1] : 1.0;
  double c = nu * a[k];
  for (int i = 0; i < k; ++i) c -= st[i] * a[i];
  ck = c / rho;
}

#ifndef MSP_DCGS_MINB
#define MSP_DCGS_MINB 4                  // 64 registers: 4 CTAs/SM (2: 128 regs, 18% slower)
#endif
#ifndef MSP_DCGS_L1RE
#define MSP_DCGS_L1RE 0
#endif
#ifndef MSP_DCGS_GROUP
#define MSP_DCGS_GROUP 16
#endif
template <int NV, int EW, bool DOT>
__global__ void __launch_bounds__(kRedThreads, MSP_DCGS_MINB) dcgs_update_kernel(size_t NE, int k, const double* __restrict__ V,
                                                                    size_t ldv, double* vk, double* w,
                                                                    const double* __restrict__ a,
                                                                    const double* __restrict__ st, double* part,
                                                                    double* out, unsigned* ticket) {
  PDL_ENTRY();
  using T = VecT<EW>;
  __shared__ double h2s[NV], as[NV], sc[4];
  for (int i = threadIdx.x; i < NV; i += blockDim.x) {
    h2s[i] = (i < k) ? st[i] : 0.0;
    as[i] = (i < k) ? a[i] : 0.0;
  }
  if (threadIdx.x == 0) {
    dcgs_scalars(k, a, st, sc[0], sc[1], sc[2]);
    sc[3] = 1.0 / sc[1];
  }
  __syncthreads();
  const double nu = sc[0], rinv = sc[3], ck = sc[2];
  double acc[DOT ? NV : 1];
#pragma unroll
  for (int i = 0; i < (DOT ? NV : 1); ++i) acc[i] = 0.0;
  double accv = 0.0, accu = 0.0;
  T* vT = reinterpret_cast<T*>(vk);
  T* wT = reinterpret_cast<T*>(w);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < NE; t += stride) {
    T vf = vT[t], u = wT[t];                           // issued before the basis loads
    T s1, s2;
    if constexpr (EW == 2) { s1 = {0.0, 0.0}; s2 = {0.0, 0.0}; } else { s1 = {0.0}; s2 = {0.0}; }
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      if (i < k) {
        const T vi = T::ld(V + i * ldv, t);
        vaxpy<EW>(h2s[i], vi, s1);
        vaxpy<EW>(as[i], vi, s2);
      }
      if (i % MSP_DCGS_GROUP == MSP_DCGS_GROUP - 1) asm volatile("" ::: "memory");
    }
    vf.x = (nu * vf.x - s1.x) * rinv;                   // (one division per CTA, not per element)
    u.x = u.x - s2.x - ck * vf.x;
    if constexpr (EW == 2) {
      vf.y = (nu * vf.y - s1.y) * rinv;
      u.y = u.y - s2.y - ck * vf.y;
    }
    vT[t] = vf;
    wT[t] = u;
    if constexpr (DOT) {
#pragma unroll
      for (int i = 0; i < NV; ++i) {
#if MSP_DCGS_L1RE
        if (i < k) acc[i] = vdot<EW>(T::ldre(V + i * ldv, t), u, acc[i]);
#else
        if (i < k) acc[i] = vdot<EW>(T::ldcg(V + i * ldv, t), u, acc[i]);
#endif
        if (i % MSP_DCGS_GROUP == MSP_DCGS_GROUP - 1) asm volatile("" ::: "memory");
      }
      accv = vdot<EW>(vf, u, accv);
      accu = vdot<EW>(u, u, accu);
    }
  }
  if constexpr (DOT) {
    block_partials<NV>(acc, k, part, 0);
    const double tail[2] = {accv, accu};
    block_partials<2>(tail, 2, part, k);
    finalize_partials(k + 2, part, out, nullptr, nullptr, -1, ticket);
  }
}

// DCGS2 pass 2, staged variant (DOT, 16-byte pairs, k <= NV): every thread streams its own
// element pair of the k+2 vectors (V[0..k), V[k], w) into a private shared-memory slot
// with cp.async (NBUF = 2: one tile ahead; NBUF = 1: the current tile), so k+2 16-byte
// loads per thread are in flight without holding registers, and the dot phase re-reads
// shared memory instead of L2.  Each thread reads only the slots it filled: no block
// barriers in the stream.  Same per-element arithmetic as dcgs_update_kernel; also
// covers k > 16 in ONE pass (the register kernel needs a separate dot pass there).
constexpr int kDcgsStThreads = 256;        // default CTA size (the launches choose per NV)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(NPEND)); }

template <int NV, int TPB = kDcgsStThreads, int NBUF = 2>
__global__ void __launch_bounds__(TPB, 1) dcgs_update_staged_kernel(size_t NE, int k, const double* __restrict__ V,
                                                                              size_t ldv, double* vk, double* w,
                                                                              const double* __restrict__ a,
                                                                              const double* __restrict__ st, double* part,
                                                                              double* out, unsigned* ticket) {
  extern __shared__ double2 stage[];            // [NBUF][NV + 2][TPB]
  __shared__ double h2s[NV], as[NV], sc[4];
  PDL_ENTRY();
  for (int i = threadIdx.x; i < NV; i += blockDim.x) {
    h2s[i] = (i < k) ? st[i] : 0.0;
    as[i] = (i < k) ? a[i] : 0.0;
  }
  if (threadIdx.x == 0) {
    dcgs_scalars(k, a, st, sc[0], sc[1], sc[2]);
    sc[3] = 1.0 / sc[1];
  }
  __syncthreads();
  const double nu = sc[0], rinv = sc[3], ck = sc[2];
  const int nvec = k + 2;                        // V[0..k), V[k], w
  auto slot = [&](int buf, int i) -> double2* { return stage + ((size_t)buf * (NV + 2) + i) * TPB + threadIdx.x; };
  auto src = [&](int i, size_t t) -> const double2* {
    const double* base = (i < k) ? V + (size_t)i * ldv : (i == k ? vk : w);
    return reinterpret_cast<const double2*>(base) + t;
  };
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (NBUF == 2 && t < NE)
    for (int i = 0; i < nvec; ++i) cp_async16(slot(0, i), src(i, t));
  if (NBUF == 2) cp_async_commit();
  double acc[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) acc[i] = 0.0;
  double accv = 0.0, accu = 0.0;
  int buf = 0;
  for (; t < NE; t += stride, buf ^= (NBUF - 1)) {
    if (NBUF == 2) {
      const size_t tn = t + stride;
      if (tn < NE)
        for (int i = 0; i < nvec; ++i) cp_async16(slot(buf ^ 1, i), src(i, tn));
      cp_async_commit();
      cp_async_wait<1>();                        // this tile's copies are complete
    } else {                                     // single buffer: this tile only
      for (int i = 0; i < nvec; ++i) cp_async16(slot(0, i), src(i, t));
      cp_async_commit();
      cp_async_wait<0>();
    }
    double2 s1 = make_double2(0.0, 0.0), s2 = s1;
#pragma unroll
    for (int i = 0; i < NV; ++i)
      if (i < k) {
        const double2 vi = *slot(buf, i);
        s1.x = fma(h2s[i], vi.x, s1.x); s1.y = fma(h2s[i], vi.y, s1.y);
        s2.x = fma(as[i], vi.x, s2.x); s2.y = fma(as[i], vi.y, s2.y);
      }
    double2 vf = *slot(buf, k), u = *slot(buf, k + 1);
    vf.x = (nu * vf.x - s1.x) * rinv;
    vf.y = (nu * vf.y - s1.y) * rinv;
    u.x = u.x - s2.x - ck * vf.x;
    u.y = u.y - s2.y - ck * vf.y;
    reinterpret_cast<double2*>(vk)[t] = vf;
    reinterpret_cast<double2*>(w)[t] = u;
#pragma unroll
    for (int i = 0; i < NV; ++i)
      if (i < k) {
        const double2 vi = *slot(buf, i);
        acc[i] = fma(vi.x, u.x, fma(vi.y, u.y, acc[i]));
      }
    accv = fma(vf.x, u.x, fma(vf.y, u.y, accv));
    accu = fma(u.x, u.x, fma(u.y, u.y, accu));
  }
  cp_async_wait<0>();
  block_partials<NV>(acc, k, part, 0);
  const double tail[2] = {accv, accu};
  block_partials<2>(tail, 2, part, k);
  finalize_partials(k + 2, part, out, nullptr, nullptr, -1, ticket);
}

// One CTA: from a = V[0..k]^T w, the old state and the sums s (V[0..k)^T u, v_k^T u,
// u^T u) -> new state (h2' = s[0..k], nu' = 1 (u kept unnormalised),
// rho' = sqrt(u^T u - ||h2'||^2)) and the host record rec[0..k] = c + h2',
// rec[k+1] = rho', rec[k+2] = nu', rec[k+3 .. 2k+3] = h2' (the host applies the
// Hessenberg correction, R14).
__global__ void dcgs_finish_kernel(int k, const double* __restrict__ a, const double* __restrict__ st_in,
                                   const double* __restrict__ s, double* __restrict__ st_out,
                                   double* __restrict__ rec) {
  PDL_ENTRY();
  if (threadIdx.x != 0) return;
  double nu, rho, ck;
  dcgs_scalars(k, a, st_in, nu, rho, ck);
  const double uu = s[k + 1];
  double ss = 0.0;
  for (int i = 0; i <= k; ++i) ss += s[i] * s[i];
  const double nun = 1.0;
  const double rhon = sqrt(fmax(uu - ss, 0.0));
  for (int i = 0; i <= k; ++i) {
    const double ci = (i < k) ? a[i] : ck;
    rec[i] = ci + s[i];
    rec[k + 3 + i] = s[i];
    st_out[i] = s[i];
  }
  rec[k + 1] = rhon;
  rec[k + 2] = nun;
  st_out[kMaxV] = nun;
  st_out[kMaxV + 1] = rhon;
}

// v = w * (1/s[0])   (Arnoldi normalisation; s on device)
__global__ void scale_kernel(size_t N, const double* __restrict__ w, const double* __restrict__ s,
                             double* __restrict__ v) {
  PDL_ENTRY();
  const double inv = 1.0 / s[0];
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += stride) v[t] = w[t] * inv;
}

// y = x + alpha*z  (x += z with alpha = 1)
__global__ void axpy_kernel(size_t N, double alpha, const double* __restrict__ z, double* __restrict__ x) {
  PDL_ENTRY();
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += stride)
    x[t] = fma(alpha, z[t], x[t]);
}

// permutations between the caller's natural cell order and the internal order
template <int B>
__global__ void perm_gather_kernel(int n, const int* __restrict__ order, const double* __restrict__ src,
                                   double* __restrict__ dst) {
  PDL_ENTRY();   // dst[p] = src[order[p]]
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * B) return;
  const int p = t / B, q = t - p * B;
  dst[t] = ldg(src + (size_t)ldg(order + p) * B + q);
}
template <int B>
__global__ void perm_scatter_kernel(int n, const int* __restrict__ order, const double* __restrict__ src,
                                    double* __restrict__ dst) {
  PDL_ENTRY();  // dst[order[p]] = src[p]
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * B) return;
  const int p = t / B, q = t - p * B;
  dst[(size_t)ldg(order + p) * B + q] = src[t];
}

// L2 flush for the per-kernel timings (msp_time_kernel): read a buffer twice the L2 size
// (clean lines only); *sink keeps the loads live.
__global__ void flush_read_kernel(size_t n, const double* __restrict__ buf, double* sink) {
  double acc = 0.0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    acc += __ldcg(buf + i);
  if (acc == 12345.678) *sink = acc;               // never true for the zero-filled buffer
}

__global__ void scalar_perm_kernel(int n, const int* __restrict__ idx, const double* __restrict__ src,
                                   double* __restrict__ dst, int scatter) {
  PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (scatter) dst[ldg(idx + i)] = src[i];
  else dst[i] = ldg(src + ldg(idx + i));
}

// ---------------------------------------------------------------------------
// a10/a11 on the device (one restart cycle = one CUDA graph): the Givens update of the
// Hessenberg column of step j and the convergence test of the host loop in gmres(),
// run by one thread after the step's kernels; it sets the conditional handle of step
// j+1 when the cycle goes on (no host round trip per Arnoldi step).  Same operation
// order as the host loop (explicitly rounded; hypot for the rotation).
// State g (ld kGv = 32): H[33*32] rotated, Hraw[33*32] (DCGS2 unrotated columns),
// cs[32], sn[32], gam[33], h2p[32], hist[32], scal[8] = {||b||, tol, nu, rho, k, broke,
// it0, maxit}.
constexpr int kGv = 32;
constexpr int kGvH = 0, kGvHraw = kGvH + (kGv + 1) * kGv, kGvCs = kGvHraw + (kGv + 1) * kGv, kGvSn = kGvCs + kGv,
              kGvGam = kGvSn + kGv, kGvH2 = kGvGam + kGv + 1, kGvHist = kGvH2 + kGv, kGvScal = kGvHist + kGv,
              kGvSize = kGvScal + 8;

__global__ void givens_init_kernel(double* g, const double* beta, double bnorm, double tol, double it0, double maxit) {
  for (int i = threadIdx.x; i < kGvSize; i += blockDim.x) g[i] = 0.0;
  __syncthreads();
  if (threadIdx.x == 0) {
    g[kGvGam] = beta[0];
    double* sc = g + kGvScal;
    sc[0] = bnorm; sc[1] = tol; sc[2] = 1.0; sc[3] = 1.0; sc[4] = 0.0; sc[5] = 0.0; sc[6] = it0; sc[7] = maxit;
  }
}

template <bool DCGS>
__global__ void givens_kernel(int j, int m, const double* __restrict__ rec, double* g,
                              cudaGraphConditionalHandle next, int has_next) {
  if (threadIdx.x != 0) return;
  pdl_wait();
  double* H = g + kGvH;
  double* Hraw = g + kGvHraw;
  double* cs = g + kGvCs;
  double* sn = g + kGvSn;
  double* gam = g + kGvGam;
  double* h2p = g + kGvH2;
  double* sc = g + kGvScal;
  auto Hc = [&](int i) -> double& { return H[i * kGv + j]; };
  if (DCGS) {
    const double nup = sc[2], rhop = sc[3];
    for (int i = 0; i <= j + 1; ++i) {
      double v = __dmul_rn(nup, (i <= j) ? rec[i] : rec[j + 1]);
      for (int l = 0; l < j; ++l) v = __dsub_rn(v, __dmul_rn(h2p[l], Hraw[i * kGv + l]));
      Hraw[i * kGv + j] = __ddiv_rn(v, rhop);
      Hc(i) = Hraw[i * kGv + j];
    }
    for (int l = 0; l <= j; ++l) h2p[l] = rec[j + 3 + l];
    sc[2] = rec[j + 2];
    sc[3] = rec[j + 1];
  } else {
    for (int i = 0; i <= j + 1; ++i) Hc(i) = rec[i];
  }
  const double hn = Hc(j + 1);
  for (int i = 0; i < j; ++i) {
    const double a = Hc(i), c = Hc(i + 1);
    Hc(i) = __dadd_rn(__dmul_rn(cs[i], a), __dmul_rn(sn[i], c));
    Hc(i + 1) = __dadd_rn(__dmul_rn(-sn[i], a), __dmul_rn(cs[i], c));
  }
  const double rho = hypot(Hc(j), Hc(j + 1));
  cs[j] = __ddiv_rn(Hc(j), rho);
  sn[j] = __ddiv_rn(Hc(j + 1), rho);
  Hc(j) = rho;
  Hc(j + 1) = 0.0;
  gam[j + 1] = __dmul_rn(-sn[j], gam[j]);
  gam[j] = __dmul_rn(cs[j], gam[j]);
  const double bnorm = sc[0];
  const double est = __ddiv_rn(fabs(gam[j + 1]), bnorm);
  g[kGvHist + j] = est;
  sc[4] = (double)(j + 1);
  const bool broke = hn < __dmul_rn(1e-14, bnorm);
  sc[5] = broke ? 1.0 : 0.0;
  const bool stop = est <= sc[1] || broke || sc[6] + (double)(j + 1) >= sc[7];
  if (!stop && has_next && j + 1 < m) cudaGraphSetConditional(next, 1);
}

}  // namespace mspk
