// a9 (K4) for 4x4 blocks with per-slot metadata: the BILU(0) substitution of
// bilu_block_kernel (same arithmetic and summation order: external couplings column-per-
// lane in entry order, one reduce-scatter, the intra-block triangle by shuffles), with a
// shorter dependent load chain per CTA.
//
// bilu_block_kernel walks blk_ptr -> (rp, dg, cnt, islot of the cell) -> (ci, F) -> y:
// four dependent global-memory round trips before the first FMA, paid by every CTA after
// the first wave (only the first wave hides them under the previous kernel's PDL tail).
// Here every (block, cell slot) has its metadata at a fixed index s = blk*MAXC + slot:
//   mf[s] = {cell, e0, e_ext, -} (forward: external L entries [e0, e_ext)),
//   mb[s] = {cell, d, e_i, e1}   (backward: D~^-1 at d, external U entries [e_i, e1)),
//   cf[s] / cb[s] = the columns of the first four external entries, sl[s] = intra-block
//   entries per slot (as islot),
// so the chain is (metadata) -> (factor columns, y / x gathers) -> FMAs: two round trips.
#pragma once
#include "kernels.cuh"

#ifndef MSP_BILU_META_PRE
#define MSP_BILU_META_PRE 2                  // external factor columns loaded before the PDL wait (<= 4)
#endif
#ifndef MSP_BILU_META_TPB
#define MSP_BILU_META_TPB 64                 // 64-thread CTAs (24 per SM): C3 apply 311.2 -> 308.2 us vs 128
#endif
#ifndef MSP_BILU_META_MINB
#define MSP_BILU_META_MINB (1536 / MSP_BILU_META_TPB)
#endif

namespace mspk {

template <int MAXC, bool FWD, bool BWD>
__global__ void __launch_bounds__(MSP_BILU_META_TPB, MSP_BILU_META_MINB) bilu_meta4_kernel(
    int b_first, int b_end, const int4* __restrict__ mf, const int4* __restrict__ cf, const int4* __restrict__ mb,
    const int4* __restrict__ cb, const int4* __restrict__ slt, const int* __restrict__ ci,
    const double* __restrict__ F, double* v, const double* __restrict__ wp, double* __restrict__ z) {
  constexpr int TS = 4;
  constexpr int TM = MAXC * TS;
  static_assert(TM <= 32, "team must fit in a warp");
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int blk = b_first + gtid / TM;
  const int lane = threadIdx.x & 31;
  const int tl = lane % TM;
  const int cq = tl / TS, q = tl % TS;
  const int tbase = lane - tl, cbase = lane - q;
  const unsigned tmask = (TM == 32) ? 0xffffffffu : (((1u << TM) - 1u) << tbase);
  const unsigned cmask = 0xfu << cbase;
  if (blk >= b_end) return;
  const size_t s = (size_t)blk * MAXC + cq;
  // ---- level 1: metadata of this slot (no dependency)
  const int4 m1 = FWD ? __ldg(mf + s) : __ldg(mb + s);
  const int4 c1 = FWD ? __ldg(cf + s) : __ldg(cb + s);
  const int4 m2 = (FWD && BWD) ? __ldg(mb + s) : make_int4(0, 0, 0, 0);
  int sl[4] = {-1, -1, -1, -1};
  if (MAXC > 1) {
    const int4 s4 = __ldg(slt + s);
    sl[0] = s4.x; sl[1] = s4.y; sl[2] = s4.z; sl[3] = s4.w;
  }
  const int i = m1.x;
  const bool valid = i >= 0;
  const int ir = valid ? i : 0;
  // ---- level 2, immutable part before the PDL wait: the first two external factor columns
  // (and an L1 prefetch of the intra-block factor blocks used by the triangle)
  const int xa = FWD ? m1.y : m1.z;                 // external range of the first phase
  const int xb = FWD ? m1.z : m1.w;
  double2 plo[MSP_BILU_META_PRE], phi[MSP_BILU_META_PRE];
#pragma unroll
  for (int u = 0; u < MSP_BILU_META_PRE; ++u) {
    const int e = xa + u;
    if (valid && e < xb) {
      const double2* cp = reinterpret_cast<const double2*>(F + (size_t)e * 16 + q * 4);
      plo[u] = ldstream2(cp);
      phi[u] = ldstream2(cp + 1);
    } else {
      plo[u] = make_double2(0.0, 0.0);
      phi[u] = plo[u];
    }
  }
  if (MAXC > 1 && valid) {
#pragma unroll
    for (int sidx = 0; sidx < MAXC; ++sidx) {
      const bool need = (FWD && sidx < cq) || (BWD && sidx >= cq);
      if (need && sl[sidx] >= 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(F + (size_t)sl[sidx] * 16 + q * 4));
    }
    if (BWD && !FWD) asm volatile("prefetch.global.L1 [%0];" ::"l"(F + (size_t)m1.y * 16 + q * 4));
  }
  pdl_wait();
  pdl_trigger();
  double t = 0.0;
  // external part of one phase over [ea, eb): entries 0,1 from the prefetched columns,
  // 2,3 with the columns from the metadata, the rest loading their columns
  auto ext = [&](int ea, int eb, const int4& cc, bool pre) -> double {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const int cs[4] = {cc.x, cc.y, cc.z, cc.w};
    double yq[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) yq[u] = (valid && ea + u < eb) ? ldg(v + (size_t)cs[u] * 4 + q) : 0.0;
    double2 lo[4], hi[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (pre && u < MSP_BILU_META_PRE) { lo[u] = plo[u]; hi[u] = phi[u]; continue; }
      const int e = ea + u;
      if (valid && e < eb) {
        const double2* cp = reinterpret_cast<const double2*>(F + (size_t)e * 16 + q * 4);
        lo[u] = ldstream2(cp);
        hi[u] = ldstream2(cp + 1);
      } else {
        lo[u] = make_double2(0.0, 0.0);
        hi[u] = lo[u];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a0 = fma(lo[u].x, yq[u], a0);
      a1 = fma(lo[u].y, yq[u], a1);
      a2 = fma(hi[u].x, yq[u], a2);
      a3 = fma(hi[u].y, yq[u], a3);
    }
    if (valid) {
#pragma unroll 2
      for (int e = ea + 4; e < eb; ++e) {
        const double yv = ldg(v + (size_t)ldg(ci + e) * 4 + q);
        const double2* cp = reinterpret_cast<const double2*>(F + (size_t)e * 16 + q * 4);
        const double2 l = ldstream2(cp), h = ldstream2(cp + 1);
        a0 = fma(l.x, yv, a0);
        a1 = fma(l.y, yv, a1);
        a2 = fma(h.x, yv, a2);
        a3 = fma(h.y, yv, a3);
      }
    }
    return reduce_scatter4(a0, a1, a2, a3, q, cmask);
  };
  if (FWD) {
    const double acc = ext(m1.y, m1.z, c1, true);
    t = valid ? (v[(size_t)ir * 4 + q] - acc) : 0.0;
#pragma unroll
    for (int sidx = 0; sidx < MAXC - 1; ++sidx) {
      double contrib = 0.0;
      const bool use = valid && cq > sidx && sl[sidx] >= 0;
      const double* blkF = F + (size_t)(use ? sl[sidx] : 0) * 16;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double yu = __shfl_sync(tmask, t, tbase + sidx * TS + u);
        if (use) contrib = fma(ldg(blkF + u * 4 + q), yu, contrib);
      }
      if (use) t -= contrib;
    }
    if (valid) v[(size_t)ir * 4 + q] = t;
    __syncwarp(tmask);
  }
  if (BWD) {
    const int4 mB = FWD ? m2 : m1;
    if (!FWD) t = valid ? v[(size_t)ir * 4 + q] : 0.0;
    const int4 cB = FWD ? __ldg(cb + s) : c1;
    t -= ext(mB.z, mB.w, cB, !FWD);
    const double* Dg = F + (size_t)(valid ? mB.y : 0) * 16;
    double x = 0.0;
#pragma unroll
    for (int sidx = MAXC - 1; sidx >= 0; --sidx) {
      double xs = 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double tu = __shfl_sync(tmask, t, tbase + sidx * TS + u);
        if (cq == sidx && valid) xs = fma(ldg(Dg + u * 4 + q), tu, xs);
      }
      if (cq == sidx) x = xs;
      if (sidx == 0) break;
      const bool use = valid && cq < sidx && sl[sidx] >= 0;
      const double* blkF = F + (size_t)(use ? sl[sidx] : 0) * 16;
      double contrib = 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double xu = __shfl_sync(tmask, xs, tbase + sidx * TS + u);
        if (use) contrib = fma(ldg(blkF + u * 4 + q), xu, contrib);
      }
      if (use) t -= contrib;
    }
    if (valid) {
      v[(size_t)ir * 4 + q] = x;
      z[(size_t)ir * 4 + q] = x + ((q == 0) ? ldg(wp + ir) : 0.0);
    }
  }
}

// 5x5 .. 8x8 blocks: the same metadata scheme with 8-lane cell groups (lane q < B owns
// row q; external couplings column-per-lane through col_accum8 and one reduce-scatter, as
// bilu_block_kernel's B >= 5 path; the columns of the first four external entries come
// from the metadata, so their gathers issue at once instead of one ci -> y chain each).
template <int B, int MAXC, bool FWD, bool BWD>
#ifndef MSP_BILU_META8_TPB
#define MSP_BILU_META8_TPB 64                // C4 apply 878 -> 857 us vs 128
#endif
__global__ void __launch_bounds__(MSP_BILU_META8_TPB, 1024 / MSP_BILU_META8_TPB) bilu_meta8_kernel(
    int b_first, int b_end, const int4* __restrict__ mf, const int4* __restrict__ cf, const int4* __restrict__ mb,
    const int4* __restrict__ cb, const int4* __restrict__ slt, const int* __restrict__ ci,
    const double* __restrict__ F, double* v, const double* __restrict__ wp, double* __restrict__ z) {
  constexpr int TS = 8;
  constexpr int TM = MAXC * TS;
  constexpr int BB = B * B;
  static_assert(B >= 5 && B <= 8 && TM <= 32, "8-lane groups");
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int blk = b_first + gtid / TM;
  const int lane = threadIdx.x & 31;
  const int tl = lane % TM;
  const int cq = tl / TS, q = tl % TS;
  const int tbase = lane - tl, cbase = lane - q;
  const unsigned tmask = (TM == 32) ? 0xffffffffu : (((1u << TM) - 1u) << tbase);
  const unsigned cmask = 0xffu << cbase;
  if (blk >= b_end) return;
  const size_t s = (size_t)blk * MAXC + cq;
  const int4 m1 = FWD ? __ldg(mf + s) : __ldg(mb + s);
  const int4 c1 = FWD ? __ldg(cf + s) : __ldg(cb + s);
  int sl[4] = {-1, -1, -1, -1};
  if (MAXC > 1) {
    const int4 s4 = __ldg(slt + s);
    sl[0] = s4.x; sl[1] = s4.y; sl[2] = s4.z; sl[3] = s4.w;
  }
  const int i = m1.x;
  const bool valid = i >= 0;
  const bool act = valid && q < B;
  const int ir = valid ? i : 0;
  if (MAXC > 1 && valid && q < B) {
#pragma unroll
    for (int sidx = 0; sidx < MAXC; ++sidx) {
      const bool need = (FWD && sidx < cq) || (BWD && sidx >= cq);
      if (need && sl[sidx] >= 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(F + (size_t)sl[sidx] * BB + q * B));
    }
  }
  pdl_wait();
  pdl_trigger();
  double t = 0.0;
  auto ext = [&](int ea, int eb, const int4& cc) -> double {
    double a8[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) a8[r] = 0.0;
    const int cs[4] = {cc.x, cc.y, cc.z, cc.w};
    double yq[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) yq[u] = (act && ea + u < eb) ? ldg(v + (size_t)cs[u] * B + q) : 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (valid && ea + u < eb) col_accum8<B>(F + (size_t)(ea + u) * BB, yq[u], q, a8);
    if (valid) {
      for (int e = ea + 4; e < eb; ++e) {
        const double yv = (q < B) ? ldg(v + (size_t)ldg(ci + e) * B + q) : 0.0;
        col_accum8<B>(F + (size_t)e * BB, yv, q, a8);
      }
    }
    return reduce_scatter8(a8, q, cmask);
  };
  if (FWD) {
    const double acc = ext(m1.y, m1.z, c1);
    t = act ? (v[(size_t)ir * B + q] - acc) : 0.0;
#pragma unroll
    for (int sidx = 0; sidx < MAXC - 1; ++sidx) {
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
    if (act) v[(size_t)ir * B + q] = t;
    __syncwarp(tmask);
  }
  if (BWD) {
    const int4 mB = FWD ? __ldg(mb + s) : m1;
    if (!FWD) t = act ? v[(size_t)ir * B + q] : 0.0;
    const int4 cB = FWD ? __ldg(cb + s) : c1;
    t -= ext(mB.z, mB.w, cB);
    const double* Dg = F + (size_t)(valid ? mB.y : 0) * BB;
    double x = 0.0;
#pragma unroll
    for (int sidx = MAXC - 1; sidx >= 0; --sidx) {
      double xs = 0.0;
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const double tu = __shfl_sync(tmask, t, tbase + sidx * TS + u);
        if (cq == sidx && act) xs = fma(ldg(Dg + u * B + q), tu, xs);
      }
      if (cq == sidx) x = xs;
      if (sidx == 0) break;
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
      v[(size_t)ir * B + q] = x;
      z[(size_t)ir * B + q] = x + ((q == 0) ? ldg(wp + ir) : 0.0);
    }
  }
}

}  // namespace mspk
