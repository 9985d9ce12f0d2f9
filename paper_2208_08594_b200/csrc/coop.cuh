// Persistent cooperative V-cycle (B_P of Alg. 1 line 4; UA-AMG V-cycle with PGS-MC
// smoothing): the whole V-cycle in ONE launch.  Each phase of the
// multi-launch path (a color of a PGS-MC sweep, residual/restriction, the coarsest
// GEMV, a prolongation) becomes a grid-stride loop over the same work items,
// separated by grid-wide barriers (cooperative launch, all CTAs co-resident).  This
// removes ~70 dependent launches per V-cycle whose coarse-level work is too small to
// amortise a launch (round-1 ncu launch list: 2668 pgs_color launches = 27% of solve
// time).  Arithmetic per row is identical to kernels.cuh (same summation order).
#pragma once
#include <cooperative_groups.h>

#include "kernels.cuh"

namespace mspk {

namespace cg = cooperative_groups;

constexpr int kMaxLevels = 20;

struct LevelDev {
  int n, ncolor, nslices, fuse_rr, n_next;
  const int* color_row;    // [ncolor+1] device
  const int* color_slice;  // [ncolor+1] device
  const int* slice_row;
  const int* slice_off;
  const int* col;
  const double* val;
  const double* diag;
  const int* agg;          // row -> next-level row
  const int* pt_ptr;       // next-level row -> member rows
  const int* pt_idx;
  const int* row_start;    // SELL offset of (slice, lane) of each row (fused residual)
  const int* row_width;    // SELL width of the row's slice
  double* b;
  double* x;
  double* r;
};

struct VParams {
  int L, pre, post, nL, ldA, coarse_diag;
  const double* Ainv;
  const double* cdiag;
  double* bL;
  double* xL;
  LevelDev lv[kMaxLevels];
};

__device__ __forceinline__ void coop_color(const LevelDev& D, int c, int tid, int nth) {
  const int s0 = __ldg(D.color_slice + c), s1 = __ldg(D.color_slice + c + 1);
  const int items = (s1 - s0) * kSell;
  for (int t = tid; t < items; t += nth) {
    const int s = s0 + t / kSell, l = t % kSell;
    const int row = __ldg(D.slice_row + s) + l;
    if (row >= __ldg(D.slice_row + s + 1)) continue;
    const int o0 = __ldg(D.slice_off + s), w = (__ldg(D.slice_off + s + 1) - o0) / kSell;
    double acc = 0.0;
    int o = o0 + l;
    for (int k = 0; k < w; ++k, o += kSell) acc = fma(__ldg(D.val + o), D.x[__ldg(D.col + o)], acc);
    D.x[row] = (D.b[row] - acc) / __ldg(D.diag + row);
  }
}

__device__ __forceinline__ double coop_row_residual(const LevelDev& D, int p) {
  const int rs = __ldg(D.row_start + p), w = __ldg(D.row_width + p);
  double acc = __ldg(D.diag + p) * D.x[p];
  int o = rs;
  for (int k = 0; k < w; ++k, o += kSell) acc = fma(__ldg(D.val + o), D.x[__ldg(D.col + o)], acc);
  return D.b[p] - acc;
}

template <int TPB>
__global__ void __launch_bounds__(TPB) vcycle_coop_kernel(const VParams* __restrict__ P) {
  cg::grid_group grid = cg::this_grid();
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nth = gridDim.x * blockDim.x;
  const int L = P->L;
  for (int l = 0; l < L; ++l) {
    const LevelDev& D = P->lv[l];
    double* bn = (l + 1 < L) ? P->lv[l + 1].b : P->bL;
    for (int sw = 0; sw < P->pre; ++sw) {
      int c = 0;
      if (sw == 0) {                                  // color 1 from the zero guess
        const int c1 = __ldg(D.color_row + 1);
        for (int i = tid; i < D.n; i += nth) D.x[i] = (i < c1) ? D.b[i] / __ldg(D.diag + i) : 0.0;
        grid.sync();
        c = 1;
      }
      for (; c < D.ncolor; ++c) {
        coop_color(D, c, tid, nth);
        grid.sync();
      }
    }
    if (D.fuse_rr) {                                  // b_{l+1} = P^T (b - A x)
      for (int I = tid; I < D.n_next; I += nth) {
        double s = 0.0;
        for (int e = __ldg(D.pt_ptr + I); e < __ldg(D.pt_ptr + I + 1); ++e)
          s += coop_row_residual(D, __ldg(D.pt_idx + e));
        bn[I] = s;
      }
      grid.sync();
    } else {
      const int items = D.nslices * kSell;
      for (int t = tid; t < items; t += nth) {
        const int s = t / kSell, lq = t % kSell;
        const int row = __ldg(D.slice_row + s) + lq;
        if (row >= __ldg(D.slice_row + s + 1)) continue;
        const int o0 = __ldg(D.slice_off + s), w = (__ldg(D.slice_off + s + 1) - o0) / kSell;
        double acc = __ldg(D.diag + row) * D.x[row];
        int o = o0 + lq;
        for (int k = 0; k < w; ++k, o += kSell) acc = fma(__ldg(D.val + o), D.x[__ldg(D.col + o)], acc);
        D.r[row] = D.b[row] - acc;
      }
      grid.sync();
      for (int I = tid; I < D.n_next; I += nth) {
        double s = 0.0;
        for (int e = __ldg(D.pt_ptr + I); e < __ldg(D.pt_ptr + I + 1); ++e) s += D.r[__ldg(D.pt_idx + e)];
        bn[I] = s;
      }
      grid.sync();
    }
  }
  // coarsest direct solve (a6)
  if (P->coarse_diag) {
    for (int i = tid; i < P->nL; i += nth) P->xL[i] = P->bL[i] / __ldg(P->cdiag + i);
  } else {
    const int lane = threadIdx.x & 31;
    const int nw = nth >> 5;
    const int n = P->nL;
    for (int row = tid >> 5; row < n; row += nw) {
      const double* a = P->Ainv + (size_t)row * P->ldA;
      double acc = 0.0;
      const int n2 = n & ~1;
      for (int j = 2 * lane; j < n2; j += 64) {
        const double2 av = __ldg(reinterpret_cast<const double2*>(a + j));
        acc = fma(av.x, P->bL[j], acc);
        acc = fma(av.y, P->bL[j + 1], acc);
      }
      if ((n & 1) && lane == 0) acc = fma(__ldg(a + n - 1), P->bL[n - 1], acc);
#pragma unroll
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) P->xL[row] = acc;
    }
  }
  grid.sync();
  for (int l = L - 1; l >= 0; --l) {
    const LevelDev& D = P->lv[l];
    const double* xn = (l + 1 < L) ? P->lv[l + 1].x : P->xL;
    for (int i = tid; i < D.n; i += nth) D.x[i] += xn[__ldg(D.agg + i)];
    grid.sync();
    for (int sw = 0; sw < P->post; ++sw)
      for (int c = D.ncolor - 1; c >= 0; --c) {
        coop_color(D, c, tid, nth);
        if (l > 0 || sw + 1 < P->post || c > 0) grid.sync();
      }
  }
}

}  // namespace mspk
