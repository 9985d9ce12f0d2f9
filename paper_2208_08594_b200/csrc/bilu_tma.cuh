// a9 (K4) for 4x4 blocks with the factor stream staged by TMA bulk copies.
//
// BILU(0) substitution in ABMC order (R5; Alg. 1 line 6), same arithmetic as
// bilu_block_kernel (kernels.cuh): one lane group of 4 lanes per cell of an aggregate block
// (<= MAXC cells, team = 4*MAXC lanes), lane q owns row q; external couplings summed
// column-per-lane and reduce-scattered, the intra-block triangle resolved by shuffles.
//
// What differs is where the factors come from.  The factors are kept in a SPLIT layout
// (setup): FL holds the L blocks of every row (external, then intra-block; positions
// ascending), FU holds D~^-1 followed by the U blocks (intra-block, then external), each
// with its own row pointers and columns.  The cells of a CTA are consecutive positions, so
// the L (forward) or U (backward) factor blocks a CTA needs form ONE contiguous range of
// FL / FU.  Thread 0 issues cp.async.bulk copies of that range (and of the matching
// column indices) into shared memory at kernel entry -- BEFORE the programmatic-dependent-
// launch wait, since factors are immutable -- so the whole factor stream of a color phase
// is in flight while the previous phase drains, and the per-cell dependent chain is left
// with only the L2 gathers of the neighbours' y / x values.  (The single-use factor stream
// is tagged evict-first in L2 so the gathered vector stays resident.)
#pragma once
#include "kernels.cuh"

namespace mspk {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// make the initialised barrier visible to the async (TMA) proxy
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// 1-D bulk copy global -> shared (16-byte aligned, size a multiple of 16), completion
// counted on `bar` (complete_tx)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
#ifdef MSP_TMA_NO_POLICY
  (void)pol;
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
  return;
#endif
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

#ifndef MSP_TMA_W
#define MSP_TMA_W 4                               // consumer warps per CTA
#endif
#ifndef MSP_TMA_D
#define MSP_TMA_D 3                               // pipeline stages per consumer warp
#endif
constexpr int kTmaW = MSP_TMA_W;
constexpr int kTmaStages = MSP_TMA_W * MSP_TMA_D;
constexpr int kTmaThreads = 32 * (kTmaW + 1);     // warp 0: producer
constexpr int kTmaHdr = 256 + 32 * kTmaStages;    // barriers (2 per stage) + chunk headers

// A chunk = the aggregate blocks one consumer warp handles per step (32 / (4*MAXC) blocks
// of one color; their cells, factor blocks and columns are contiguous).  Setup table:
//   a = {blk_lo, blk_hi, c_lo, c_hi},  b = {eL0, eL1, eU0, eU1}  (FL / FU entry ranges).
struct TmaChunk {
  int4 a, b;
};

// Byte layout of one pipeline stage for a chunk (all offsets 16-byte aligned):
//   [FL blocks][FU blocks][ciL window][ciU window][cell meta][islot][blk_ptr window]
struct TmaStageLayout {
  int nL, nU, ciL0, nciL, ciU0, nciU, ncell, bp0, nbp;
  int oFU, oCL, oCU, oCM, oIS, oBP, bytes;
  __host__ __device__ TmaStageLayout(const TmaChunk& k, bool fwd, bool bwd) {
    nL = fwd ? k.b.y - k.b.x : 0;
    nU = bwd ? k.b.w - k.b.z : 0;
    ciL0 = k.b.x & ~3;
    nciL = nL ? (((k.b.y + 3) & ~3) - ciL0) : 0;
    ciU0 = k.b.z & ~3;
    nciU = nU ? (((k.b.w + 3) & ~3) - ciU0) : 0;
    ncell = k.a.w - k.a.z;
    bp0 = k.a.x & ~3;
    nbp = ((k.a.y + 1 + 3) & ~3) - bp0;
    oFU = nL * 128;
    oCL = oFU + nU * 128;
    oCU = oCL + nciL * 4;
    oCM = oCU + nciU * 4;
    oIS = oCM + ncell * 16;
    oBP = oIS + ncell * 16;
    bytes = oBP + nbp * 4;
  }
};

// One color phase, persistent and warp-specialised: CTA b owns chunks chunk_first + b + m *
// gridDim.x (m = 0, 1, ...).  Warp 0 (producer) streams chunk m into ring stage m % S with
// cp.async.bulk (full[s]: transaction count; the first S chunks are issued BEFORE the PDL
// wait -- factors are immutable); consumer warp m % W waits full[s], computes the chunk
// from shared memory (only the neighbours' y / x values are gathered, from L2) and
// releases the stage (empty[s]).  Per cell (cell meta cm[i] = {rpL[i], rpU[i], rpU[i+1],
// cnt[i]}; cnt = #external L | #intra-block U << 8; islot[i]: per block slot s the FL
// entry of (i, c0+s) for s < own slot, the FU entry for s >= own slot (own slot = D~^-1)):
//   FWD: y_i = r_i - sum_{k before i} L_ik y_k (in place in v)
//   BWD: x_i = D~_i^-1 (y_i - sum_{j after i} U_ij x_j) (in place in v); z_i = x_i + wp[i]
//        on the pressure slot;  FWD && BWD: the last color (forward, then backward).
template <int MAXC, bool FWD, bool BWD>
__global__ void __launch_bounds__(kTmaThreads) bilu_tma4_kernel(
    int chunk_first, int chunk_end, int stage_bytes, const TmaChunk* __restrict__ chunks,
    const int* __restrict__ blk_ptr, const int* __restrict__ ciL, const double* __restrict__ FL,
    const int* __restrict__ ciU, const double* __restrict__ FU, const int4* __restrict__ cmeta,
    const int4* __restrict__ islot, double* v, const double* __restrict__ wp, double* __restrict__ z) {
  constexpr int TS = 4;
  constexpr int TM = MAXC * TS;
  static_assert(TM <= 32, "team must fit in a warp");
  constexpr int S = kTmaStages;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + S;
  TmaChunk* hdr = reinterpret_cast<TmaChunk*>(smem + 256);             // per-stage chunk entry
  unsigned char* stage0 = smem + kTmaHdr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nmine = (chunk_end - chunk_first - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init_fence();
  }
  __syncthreads();                                                     // barriers initialised
  if (warp == 0) {
    // ---------------- producer: table entries 32 at a time (one per lane), copies by lane 0
    const uint64_t pol = l2_evict_first_policy();
    for (int m0 = 0; m0 < nmine; m0 += 32) {
      TmaChunk mine;
      if (m0 + lane < nmine) mine = chunks[chunk_first + blockIdx.x + (m0 + lane) * gridDim.x];
      const int cnt = min(32, nmine - m0);
      for (int j = 0; j < cnt; ++j) {
        TmaChunk k;
        k.a.x = __shfl_sync(0xffffffffu, mine.a.x, j); k.a.y = __shfl_sync(0xffffffffu, mine.a.y, j);
        k.a.z = __shfl_sync(0xffffffffu, mine.a.z, j); k.a.w = __shfl_sync(0xffffffffu, mine.a.w, j);
        k.b.x = __shfl_sync(0xffffffffu, mine.b.x, j); k.b.y = __shfl_sync(0xffffffffu, mine.b.y, j);
        k.b.z = __shfl_sync(0xffffffffu, mine.b.z, j); k.b.w = __shfl_sync(0xffffffffu, mine.b.w, j);
        const int m = m0 + j;
        const int s = m % S;
        if (lane == 0) {
          if (m >= S) mbar_wait_parity(empty + s, (uint32_t)(((m / S) - 1) & 1));
          const TmaStageLayout Ly(k, FWD, BWD);
          hdr[s] = k;
          unsigned char* st = stage0 + (size_t)s * stage_bytes;
          uint64_t* bar = full + s;
          mbar_arrive_expect_tx(bar, (uint32_t)Ly.bytes);
          if (Ly.nL) {
            bulk_g2s(st, FL + (size_t)k.b.x * 16, (uint32_t)Ly.nL * 128, bar, pol);
            bulk_g2s(st + Ly.oCL, ciL + Ly.ciL0, (uint32_t)Ly.nciL * 4, bar, pol);
          }
          if (Ly.nU) {
            bulk_g2s(st + Ly.oFU, FU + (size_t)k.b.z * 16, (uint32_t)Ly.nU * 128, bar, pol);
            bulk_g2s(st + Ly.oCU, ciU + Ly.ciU0, (uint32_t)Ly.nciU * 4, bar, pol);
          }
          bulk_g2s(st + Ly.oCM, cmeta + k.a.z, (uint32_t)Ly.ncell * 16, bar, pol);
          bulk_g2s(st + Ly.oIS, islot + k.a.z, (uint32_t)Ly.ncell * 16, bar, pol);
          bulk_g2s(st + Ly.oBP, blk_ptr + Ly.bp0, (uint32_t)Ly.nbp * 4, bar, pol);
        }
        __syncwarp();
      }
    }
    pdl_trigger();
    return;
  }
  // ---------------- consumers
  const int cw = warp - 1;
  const int tl = lane % TM;
  const int cq = tl / TS, q = tl % TS;
  const int tbase = lane - tl, cbase = lane - q;
  const unsigned tmask = (TM == 32) ? 0xffffffffu : (((1u << TM) - 1u) << tbase);
  const unsigned cmask = 0xfu << cbase;
  const int team = lane / TM;
  pdl_wait();
  pdl_trigger();
  for (int m = cw; m < nmine; m += kTmaW) {
    const int s = m % S;
    mbar_wait_parity(full + s, (uint32_t)((m / S) & 1));
    const TmaChunk k = hdr[s];
    const TmaStageLayout Ly(k, FWD, BWD);
    const unsigned char* st = stage0 + (size_t)s * stage_bytes;
    const double* sFL = reinterpret_cast<const double*>(st);
    const double* sFU = reinterpret_cast<const double*>(st + Ly.oFU);
    const int* sCL = reinterpret_cast<const int*>(st + Ly.oCL);
    const int* sCU = reinterpret_cast<const int*>(st + Ly.oCU);
    const int4* sCM = reinterpret_cast<const int4*>(st + Ly.oCM);
    const int4* sIS = reinterpret_cast<const int4*>(st + Ly.oIS);
    const int* sBP = reinterpret_cast<const int*>(st + Ly.oBP);
    const int blk = k.a.x + team;
    if (blk < k.a.y) {
      const int c0 = sBP[blk - Ly.bp0], c1 = sBP[blk + 1 - Ly.bp0];
      const bool valid = cq < c1 - c0;
      const int i = c0 + (valid ? cq : 0);
      const int4 cm = sCM[i - k.a.z];
      const int cn = valid ? cm.w : 0;
      int sl[4] = {-1, -1, -1, -1};
      if (MAXC > 1 && valid) {
        const int4 s4 = sIS[i - k.a.z];
        sl[0] = s4.x; sl[1] = s4.y; sl[2] = s4.z; sl[3] = s4.w;
      }
      double t = 0.0;
      if (FWD) {
        const int li0 = valid ? cm.x - k.b.x : 0;                   // local FL range of cell i
        const int lx = li0 + (cn & 0xff);                            // [li0, lx): external L
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        for (int base = li0; base < lx; base += 4) {
          int kk[4];
          double yq[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) kk[u] = (base + u < lx) ? sCL[base + u + k.b.x - Ly.ciL0] : -1;
#pragma unroll
          for (int u = 0; u < 4; ++u) yq[u] = (kk[u] >= 0) ? ldg(v + (size_t)kk[u] * 4 + q) : 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (kk[u] >= 0) {
              const double2* cp = reinterpret_cast<const double2*>(sFL + (size_t)(base + u) * 16 + q * 4);
              const double2 lo = cp[0], hi = cp[1];
              a0 = fma(lo.x, yq[u], a0);
              a1 = fma(lo.y, yq[u], a1);
              a2 = fma(hi.x, yq[u], a2);
              a3 = fma(hi.y, yq[u], a3);
            }
          }
        }
        const double acc = reduce_scatter4(a0, a1, a2, a3, q, cmask);
        t = valid ? (v[(size_t)i * 4 + q] - acc) : 0.0;
#pragma unroll
        for (int sidx = 0; sidx < MAXC - 1; ++sidx) {
          // cell sidx is final: broadcast its vector, later cells subtract L_{i,sidx} y_sidx
          double contrib = 0.0;
          const bool use = valid && cq > sidx && sl[sidx] >= 0;
          const double* blkF = sFL + (size_t)(use ? sl[sidx] - k.b.x : 0) * 16;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double yu = __shfl_sync(tmask, t, tbase + sidx * TS + u);
            if (use) contrib = fma(blkF[u * 4 + q], yu, contrib);
          }
          if (use) t -= contrib;
        }
        if (valid) v[(size_t)i * 4 + q] = t;
        __syncwarp(tmask);
      }
      if (BWD) {
        if (!FWD) t = valid ? v[(size_t)i * 4 + q] : 0.0;
        const int ui0 = valid ? cm.y - k.b.z : 0;                   // local FU range (diag first)
        const int ui1 = valid ? cm.z - k.b.z : 0;
        const int ux = ui0 + 1 + (cn >> 8);                          // [ux, ui1): external U
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        for (int base = ux; base < ui1; base += 4) {
          int kk[4];
          double xq[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) kk[u] = (base + u < ui1) ? sCU[base + u + k.b.z - Ly.ciU0] : -1;
#pragma unroll
          for (int u = 0; u < 4; ++u) xq[u] = (kk[u] >= 0) ? ldg(v + (size_t)kk[u] * 4 + q) : 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (kk[u] >= 0) {
              const double2* cp = reinterpret_cast<const double2*>(sFU + (size_t)(base + u) * 16 + q * 4);
              const double2 lo = cp[0], hi = cp[1];
              a0 = fma(lo.x, xq[u], a0);
              a1 = fma(lo.y, xq[u], a1);
              a2 = fma(hi.x, xq[u], a2);
              a3 = fma(hi.y, xq[u], a3);
            }
          }
        }
        t -= reduce_scatter4(a0, a1, a2, a3, q, cmask);
        const double* Dg = sFU + (size_t)ui0 * 16;
        double x = 0.0;
#pragma unroll
        for (int sidx = MAXC - 1; sidx >= 0; --sidx) {
          // cell sidx: x = D~^-1 t (its t is complete once all later cells were applied)
          double xs = 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double tu = __shfl_sync(tmask, t, tbase + sidx * TS + u);
            if (cq == sidx && valid) xs = fma(Dg[u * 4 + q], tu, xs);
          }
          if (cq == sidx) x = xs;
          if (sidx == 0) break;
          // earlier cells subtract U_{i,sidx} x_sidx
          const bool use = valid && cq < sidx && sl[sidx] >= 0;
          const double* blkF = sFU + (size_t)(use ? sl[sidx] - k.b.z : 0) * 16;
          double contrib = 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double xu = __shfl_sync(tmask, xs, tbase + sidx * TS + u);
            if (use) contrib = fma(blkF[u * 4 + q], xu, contrib);
          }
          if (use) t -= contrib;
        }
        if (valid) {
          v[(size_t)i * 4 + q] = x;
          z[(size_t)i * 4 + q] = x + ((q == 0) ? ldg(wp + i) : 0.0);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);                            // stage s consumed
  }
}

}  // namespace mspk
