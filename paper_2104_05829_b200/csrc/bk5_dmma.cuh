// BK5 variant 7, "dmma": the six 1-D contractions on the FP64 tensor cores
// (mma.sync.m8n8k4.f64, SASS DMMA) for high orders (N + 1 = NQ >= 9).
//
// Why: at NQ >= 12 the register-pencil kernel (bk5_pencil.cuh) is issue- and
// latency-bound: ncu at NQ = 13 (profiles/r2o_*) counts ~2.5 instructions per
// DFMA (uniform constant loads of D-hat, address moves) at 12 warps per SM.
// One m8n8k4 DMMA does 256 FMAs per warp instruction, so the contractions
// cost ~8x fewer issue slots at the same FP64 rate (DMMA 37.1 vs DFMA 35.8
// TF/s measured, profiles/r1_fp64_pipes.json), at the price of padding the
// contracted and output extents to 16.
//
// A contraction along one axis is the GEMM  Y[m][n] = sum_kk A[m][kk] X[kk][n]
// with A = D-hat (forward) or D-hat^T (backward) held in registers as zero-
// padded 16 x 16 fragments, kk / m the contracted axis and n = (p, q) the two
// others.  Warp w owns p = w (NQ warps per element) and q in two 8-wide
// tiles [0, 8) and [8, 16): every fragment address is p*SP + q*SQ + kk*SK
// with no division, and each warp runs 2 n-tiles x 2 m-tiles x 4 k-steps =
// 16 DMMA per contraction (4 independent accumulators).  X reads with kk or q
// >= NQ land on finite data (the rest of the element, or the zeroed tail)
// and meet a zero row / column of A, so no predication is needed; outputs with
// m or q >= NQ are not stored.  Element buffers use row stride PJ = 20 and
// plane stride PK = 4 (mod 16) doubles: fragment reads are bank-conflict
// free along every axis.
//
// Per element (persistent CTA, NQ warps; shared U, R, S), with the warp's
// ownership making most phases warp-private (4 block barriers per element):
//   u -> U (warp = k plane);  F1 Di U -> R, F2 Dj U -> S (warp = k plane)
//   | F3 Dk U -> U in place (warp = j column)
//   | G: R, S, U <- G (R, S, U) (warp = k plane; G coalesced, L2-prefetched)
//   | B3 Dk^T U -> U in place (warp = j column)
//   | B2 U += Dj^T S, B1 w = lam0 (Di^T R + U) [+ mass, mask, u.w] (warp = k)
// HBM per point: u 8 + G 48 + w 8 B (the BK5 roofline).  The next element's
// u and G are bulk-prefetched into L2 at the start of each element.
#pragma once
#include "bk5_pencil.cuh"

namespace nk {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int NQ>
struct DmmaCfg {
  static_assert(NQ >= 9 && NQ <= 16, "dmma BK5: NQ in [9, 16] (two 8-row m tiles)");
  static constexpr int PJ = 20;                                   // = 4 mod 16
  static constexpr int PK = NQ * PJ + ((4 - (NQ * PJ) % 16) + 16) % 16;
  static constexpr int VOL = NQ * PK;
  static constexpr int NQ2 = NQ * NQ, NQ3 = NQ2 * NQ;
  static constexpr int THREADS = NQ * 32;
  static constexpr int TAIL = 3 * PK;   // zeroed: reads past the last buffer stay finite
  static size_t smem_bytes() { return sizeof(double) * (3 * (size_t)VOL + TAIL + 32); }
  __device__ __forceinline__ static int idx(int k, int j, int i) { return k * PK + j * PJ + i; }
};

// Y = A X along the axis of stride SK for the warp's p (stride SP); the
// lane's accumulators c[t][mt][0..1] hold rows m = mt*8 + lane/4, columns
// q = t*8 + 2*(lane%4) + {0, 1}.
template <int NQ, int SK, int SP, int SQ>
__device__ __forceinline__ void dmma_contract(const double* __restrict__ X,
                                              const double (&A)[2][4], int p, int lane,
                                              double (&c)[2][2][2]) {
  const double* xb = X + p * SP + (lane >> 2) * SQ + (lane & 3) * SK;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const double b0 = xb[ks * 4 * SK];
    const double b1 = xb[ks * 4 * SK + 8 * SQ];
    if (ks == 0) {
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) c[t][mt][0] = c[t][mt][1] = 0.0;
    }
    dmma884(c[0][0][0], c[0][0][1], A[0][ks], b0);
    dmma884(c[0][1][0], c[0][1][1], A[1][ks], b0);
    dmma884(c[1][0][0], c[1][0][1], A[0][ks], b1);
    dmma884(c[1][1][0], c[1][1][1], A[1][ks], b1);
  }
}

// f(c, m, q) for the lane's stored entries (m, q < NQ).
template <int NQ, typename F>
__device__ __forceinline__ void dmma_foreach(int lane, const double (&c)[2][2][2], F&& f) {
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int m = mt * 8 + (lane >> 2);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int q = t * 8 + 2 * (lane & 3) + h;
        if (m < NQ && q < NQ) f(c[t][mt][h], m, q);
      }
    }
}

template <int NQ, int MINB>
__global__ void __launch_bounds__(NQ * 32, MINB)
bk5_dmma(int64_t nlist, const int32_t* __restrict__ elist, const __grid_constant__ DParam<NQ> D,
         const double* __restrict__ G, const double* __restrict__ u, double* __restrict__ w,
         double lam0, const double* __restrict__ B, double lam1,
         const uint8_t* __restrict__ mask, nk_cg_state* st, double* __restrict__ partials,
         int64_t part_base, int64_t reduce_count) {
  using C = DmmaCfg<NQ>;
  constexpr int NQ2 = C::NQ2, NQ3 = C::NQ3, PK = C::PK, PJ = C::PJ, VOL = C::VOL;
  extern __shared__ __align__(16) double smem[];
  double* U = smem;
  double* R = U + VOL;
  double* S = R + VOL;
  double* red = S + VOL + C::TAIL;
  const int t = threadIdx.x, lane = t & 31, wq = t >> 5;   // warp = its k plane / j column
  auto elem_of = [&](int64_t slot) -> int64_t { return elist ? (int64_t)elist[slot] : slot; };
  // zero-padded A fragments: row m = mt*8 + lane/4, column kk = ks*4 + lane%4
  double Af[2][4], Ab[2][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int m = mt * 8 + (lane >> 2), kk = ks * 4 + (lane & 3);
      const bool ok = m < NQ && kk < NQ;
      Af[mt][ks] = ok ? D.d[m * NQ + kk] : 0.0;    // forward: D[m][kk]
      Ab[mt][ks] = ok ? D.d[kk * NQ + m] : 0.0;    // backward: D^T
    }
  }
  for (int q = t; q < 3 * VOL + C::TAIL; q += C::THREADS) smem[q] = 0.0;
  __syncthreads();   // padding reads of other warps' regions must see finite data
  if ((int64_t)blockIdx.x < nlist && t == 0)
    prefetch_l2(G + elem_of(blockIdx.x) * 6 * NQ3, 6 * NQ3 * (int64_t)sizeof(double));
  pdl_wait();
  pdl_trigger();
  if (st != nullptr && st->done) return;
  // the warp's (j, i) points of its k plane: idx = lane + 32 r
  constexpr int PR = (NQ2 + 31) / 32;
  double dot = 0.0;
  double c[2][2][2];
  for (int64_t slot = blockIdx.x; slot < nlist; slot += gridDim.x) {
    const int64_t e = elem_of(slot);
    if (t == 0 && slot + gridDim.x < nlist) {   // next element's operands into L2
      const int64_t en = elem_of(slot + gridDim.x);
      prefetch_l2(G + en * 6 * NQ3, 6 * NQ3 * (int64_t)sizeof(double));
      prefetch_l2(u + en * NQ3, NQ3 * (int64_t)sizeof(double));
    }
    const double* ue = u + e * NQ3 + wq * NQ2;
    // ---- u plane k = wq -> U (warp-private: only this warp reads it before
    // the first barrier)
    {
      double v[PR];
#pragma unroll
      for (int r = 0; r < PR; ++r) {
        const int q = lane + 32 * r;
        v[r] = q < NQ2 ? __ldg(ue + q) : 0.0;
      }
#pragma unroll
      for (int r = 0; r < PR; ++r) {
        const int q = lane + 32 * r;
        if (q < NQ2) U[wq * PK + (q / NQ) * PJ + (q % NQ)] = v[r];
      }
    }
    __syncwarp();
    // ---- F1: Di (contract i; p = k, q = j) -> R ;  F2: Dj (contract j; q = i) -> S
    dmma_contract<NQ, 1, PK, PJ>(U, Af, wq, lane, c);
    dmma_foreach<NQ>(lane, c, [&](double v, int m, int q) { R[C::idx(wq, q, m)] = v; });
    dmma_contract<NQ, PJ, PK, 1>(U, Af, wq, lane, c);
    dmma_foreach<NQ>(lane, c, [&](double v, int m, int q) { S[C::idx(wq, m, q)] = v; });
    __syncthreads();
    // ---- F3: Dk (contract k; p = j, q = i), in place in the warp's j column
    dmma_contract<NQ, PK, PJ, 1>(U, Af, wq, lane, c);
    __syncwarp();
    dmma_foreach<NQ>(lane, c, [&](double v, int m, int q) { U[C::idx(m, wq, q)] = v; });
    __syncthreads();
    // ---- G: pointwise symmetric 3x3 on the warp's k plane (G coalesced)
    {
      const double* ge = G + e * 6 * NQ3 + wq * NQ2;
#pragma unroll
      for (int r0 = 0; r0 < PR; r0 += 2) {
        double g[2][6];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int q = lane + 32 * (r0 + r);
#pragma unroll
          for (int cc = 0; cc < 6; ++cc)
            g[r][cc] = (r0 + r < PR && q < NQ2) ? __ldg(ge + cc * NQ3 + q) : 0.0;
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int q = lane + 32 * (r0 + r);
          if (r0 + r < PR && q < NQ2) {
            const int x = wq * PK + (q / NQ) * PJ + (q % NQ);
            const double ur = R[x], us = S[x], ut = U[x];
            R[x] = g[r][0] * ur + g[r][1] * us + g[r][2] * ut;
            S[x] = g[r][1] * ur + g[r][3] * us + g[r][4] * ut;
            U[x] = g[r][2] * ur + g[r][4] * us + g[r][5] * ut;
          }
        }
      }
    }
    __syncthreads();
    // ---- B3: Dk^T gt, in place in the warp's j column
    dmma_contract<NQ, PK, PJ, 1>(U, Ab, wq, lane, c);
    __syncwarp();
    dmma_foreach<NQ>(lane, c, [&](double v, int m, int q) { U[C::idx(m, wq, q)] = v; });
    __syncthreads();
    // ---- B2: U += Dj^T gs (warp = k plane, private from here on)
    dmma_contract<NQ, PJ, PK, 1>(S, Ab, wq, lane, c);
    dmma_foreach<NQ>(lane, c, [&](double v, int m, int q) { U[C::idx(wq, m, q)] += v; });
    __syncwarp();
    // ---- B1: w = lam0 (Di^T gr + U) [+ lam1 B u] [mask] -> HBM; fused u.w
    dmma_contract<NQ, 1, PK, PJ>(R, Ab, wq, lane, c);
    const int64_t gb = e * NQ3 + wq * NQ2;   // (k = wq, j = q, i = m)
    dmma_foreach<NQ>(lane, c, [&](double v, int m, int q) {
      const int g = q * NQ + m;
      double r = lam0 * (v + U[C::idx(wq, q, m)]);
      if (B != nullptr || st != nullptr) {
        const double uv = __ldg(u + gb + g);
        if (B != nullptr) r = fma(lam1 * __ldg(B + gb + g), uv, r);
        if (mask != nullptr) r = mask[gb + g] ? r : 0.0;
        dot = fma(uv, r, dot);
      } else if (mask != nullptr) {
        r = mask[gb + g] ? r : 0.0;
      }
      w[gb + g] = r;
    });
    __syncwarp();   // the next element's u load rewrites this warp's plane
  }
  if (st != nullptr) {
    double vv[1] = {dot};
    block_sum<1>(vv, red);
    if (t == 0) partials[part_base + blockIdx.x] = vv[0];
    if (reduce_count > 0 && last_block(&st->ticket[0], gridDim.x)) {
      double sres[1];
      reduce_partials<1>(partials, reduce_count, 0, sres, red);
      if (t == 0) st->pAp = sres[0];
    }
  }
}

template <int NQ, int MINB>
static int64_t dmma_grid(int64_t nlist) {
  static int64_t resident = -1;
  if (resident < 0) {
    using C = DmmaCfg<NQ>;
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(bk5_dmma<NQ, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::smem_bytes());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bk5_dmma<NQ, MINB>, C::THREADS,
                                                  C::smem_bytes());
    resident = (int64_t)sms * (per > 0 ? per : 1);
  }
  return nlist < resident ? nlist : resident;
}

template <int NQ, int MINB>
static int launch_dmma(int64_t nlist, const int32_t* elist, const double* Dhost, const double* G,
                       const double* u, double* w, double lam0, const double* B, double lam1,
                       const uint8_t* mask, nk_cg_state* st, double* partials, int64_t part_base,
                       int64_t reduce_count, cudaStream_t s) {
  using C = DmmaCfg<NQ>;
  const int64_t grid = dmma_grid<NQ, MINB>(nlist);
  if (grid == 0) return NK_OK;
  DParam<NQ> D;
  D.set(Dhost);
  launch_ex(st != nullptr ? kPdlStep : 0, bk5_dmma<NQ, MINB>, dim3((unsigned)grid),
            dim3(C::THREADS), C::smem_bytes(), s, nlist, elist, D, G, u, w, lam0, B, lam1, mask,
            st, partials, part_base, reduce_count);
  return check_launch("bk5_dmma");
}

}  // namespace nk
