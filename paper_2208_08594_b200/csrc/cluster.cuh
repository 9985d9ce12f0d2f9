// Coarse V-cycle legs in ONE thread-block cluster (B_P of Alg. 1 line 4; UA-AMG V-cycle
// with PGS-MC smoothing, Alg. 4).
//
// Below level 1 every PGS-MC color phase touches a few thousand rows (C3: level 2
// 70 k rows / 10 colors, level 3 17.5 k rows / 11 colors): each costs a dependent
// kernel node (~3 us) while the data it moves takes well under 1 us.  Here the color
// phases, residuals, restrictions and prolongations of levels [lc, L) run inside one
// cluster of CS CTAs (one per SM of one GPC) separated by hardware cluster barriers
// (barrier.cluster arrive.release / wait.acquire, a few hundred cycles; the acquire
// side invalidates L1 so the next phase reads the other CTAs' x from L2).  Before each
// barrier every thread already loads the immutable matrix entries of its first row of
// the NEXT phase (the same prologue the multi-launch kernels run before griddepcontrol
// .wait), so a phase after the barrier only waits for the x gathers.
//
// Two kernels per V-cycle: the down leg (pre-sweeps, residual, restriction of every
// level in [lc, L), ending with the coarsest right-hand side) and the up leg
// (prolongation and post-sweeps back to level lc); the coarsest GEMV between them is
// bandwidth-bound (154 MB at C3) and stays a full-GPU kernel.
//
// Per-row arithmetic and summation order are exactly those of sell_row_kernel /
// restrict_kernel / prolong_kernel (PF = 4 prefetched entries first, zero-padded), so
// the cluster path reproduces the multi-launch path bit for bit.
#pragma once
#include "kernels.cuh"

namespace mspk {

constexpr int kClMaxLevels = 8;
constexpr int kClThreads = 1024;

struct ClLevel {
  int n, ncolor, lpr, n_next, c1_next;   // c1_next: end of color 1 of the next level (fused init)
  const int* color_slice;                // [ncolor+1] device
  const int* slice_row;
  const int* slice_off;
  const int* col;
  const double* val;
  const double* diag;
  const int* agg;
  const int* pt_ptr;
  const int* pt_idx;
  double* b;
  double* x;
  double* r;
  double* bn;                            // next level's b (or the coarsest b)
  double* xn;                            // next level's x (or the coarsest x)
  const double* dn;                      // next level's diagonal (null: coarsest, no fused init)
};

struct ClParams {
  int nlev, pre, post;
  ClLevel lv[kClMaxLevels];
};

__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// prefetched first row of a phase (matrix entries are immutable)
struct ClPf {
  int pc[4];
  double pv[4];
  double d;
};

// mode 0: GS update; 1: GS update + residual of the updated row (last pre-sweep color);
// 2: residual only
__device__ __forceinline__ void cl_prefetch(const ClLevel& D, int s0, int t, ClPf& pf) {
  const int lpr = D.lpr;
  const int per = kSell * lpr;
  const int s = s0 + t / per;
  const int rem = t % per;
  const int l = rem / lpr, u = rem % lpr;
  const int r0 = ldg(D.slice_row + s), r1 = ldg(D.slice_row + s + 1);
  const int row = r0 + l;
  const int o0 = ldg(D.slice_off + s), w = (ldg(D.slice_off + s + 1) - o0) / kSell;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int k = u + m * lpr;
    const int o = o0 + k * kSell + l;
    pf.pc[m] = (k < w) ? ldg(D.col + o) : row;
    pf.pv[m] = (k < w) ? ldg(D.val + o) : 0.0;
  }
  pf.d = (row < r1) ? ldg(D.diag + row) : 1.0;
}

// one SELL color range [s0, s1) of level D; the synchronisation separating it from the
// previous phase (sync: 0 none, 1 cluster barrier, 2 griddepcontrol wait on the previous
// kernel) is taken after the prefetch of the thread's first work item
__device__ __forceinline__ void cl_rows(const ClLevel& D, int s0, int s1, int mode, int tid, int nth,
                                        int sync) {
  const int lpr = D.lpr;
  const int per = kSell * lpr;
  const int items = (s1 - s0) * per;
  ClPf pf;
  const bool have = tid < items;
  if (have) cl_prefetch(D, s0, tid, pf);
  __syncwarp();
  if (sync == 1) cluster_barrier();
  else if (sync == 2) { pdl_wait(); pdl_trigger(); }
  for (int t = tid; t < items; t += nth) {       // items % 32 == 0: warps stay converged
    if (t != tid) cl_prefetch(D, s0, t, pf);
    const int s = s0 + t / per;
    const int rem = t % per;
    const int l = rem / lpr, u = rem % lpr;
    const int r0 = ldg(D.slice_row + s), r1 = ldg(D.slice_row + s + 1);
    const int row = r0 + l;
    const int o0 = ldg(D.slice_off + s), w = (ldg(D.slice_off + s + 1) - o0) / kSell;
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < 4; ++m) acc = fma(pf.pv[m], D.x[pf.pc[m]], acc);
    for (int k = u + 4 * lpr; k < w; k += lpr) {
      const int o = o0 + k * kSell + l;
      acc = fma(ldg(D.val + o), D.x[ldg(D.col + o)], acc);
    }
    for (int m = lpr / 2; m; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
    if (u == 0 && row < r1) {
      const double d = pf.d;
      if (mode == 2) {
        D.r[row] = D.b[row] - fma(d, D.x[row], acc);
      } else {
        const double bs = D.b[row] - acc;
        const double xi = bs / d;
        D.x[row] = xi;
        if (mode == 1) D.r[row] = fma(-d, xi, bs);
      }
    }
  }
}

// down leg: for l in [0, nlev): pre-sweeps (the zero-guess first color of level 0 was
// fused into the producer of its b; deeper levels get it from the restriction phase),
// residual, restriction b_{l+1} = P^T r (+ fused zero-guess first color of level l+1)
__global__ void __launch_bounds__(kClThreads, 1) vcycle_cluster_down_kernel(const __grid_constant__ ClParams P) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nth = gridDim.x * blockDim.x;        // the grid is exactly one cluster
  bool first = true;                             // first phase: ordered by griddepcontrol
  for (int li = 0; li < P.nlev; ++li) {
    const ClLevel& D = P.lv[li];
    const int g = D.ncolor;
    for (int sw = 0; sw < P.pre; ++sw) {
      const bool wr = (sw + 1 == P.pre);
      int c = (sw == 0) ? 1 : 0;
      if (sw == 0 && g == 1 && wr) {             // single color: residual of all rows
        cl_rows(D, 0, ldg(D.color_slice + g), 2, tid, nth, first ? 2 : 1);
        first = false;
        continue;
      }
      for (; c < g; ++c) {
        const bool last = (c == g - 1);
        cl_rows(D, ldg(D.color_slice + c), ldg(D.color_slice + c + 1), (last && wr) ? 1 : 0, tid, nth,
                first ? 2 : 1);
        first = false;
      }
      if (wr && g > 1) cl_rows(D, 0, ldg(D.color_slice + g - 1), 2, tid, nth, 1);
    }
    if (first) { pdl_wait(); pdl_trigger(); first = false; }
    cluster_barrier();
    for (int I = tid; I < D.n_next; I += nth) {  // restriction (restrict_kernel order)
      double s = 0.0;
      for (int e = ldg(D.pt_ptr + I); e < ldg(D.pt_ptr + I + 1); ++e) s += D.r[ldg(D.pt_idx + e)];
      D.bn[I] = s;
      if (D.dn) D.xn[I] = (I < D.c1_next) ? s / ldg(D.dn + I) : 0.0;
    }
  }
}

// up leg: for l = nlev-1 .. 0: x_l += x_{l+1}[agg] (x_{nlev} = coarsest x), post-sweeps in
// descending color order
__global__ void __launch_bounds__(kClThreads, 1) vcycle_cluster_up_kernel(const __grid_constant__ ClParams P) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nth = gridDim.x * blockDim.x;
  pdl_wait();
  pdl_trigger();
  for (int li = P.nlev - 1; li >= 0; --li) {
    const ClLevel& D = P.lv[li];
    if (li < P.nlev - 1) cluster_barrier();      // x_{l+1} final
    for (int i = tid; i < D.n; i += nth) D.x[i] += D.xn[ldg(D.agg + i)];
    for (int sw = 0; sw < P.post; ++sw)
      for (int c = D.ncolor - 1; c >= 0; --c)
        cl_rows(D, ldg(D.color_slice + c), ldg(D.color_slice + c + 1), 0, tid, nth, 1);
  }
}

}  // namespace mspk
