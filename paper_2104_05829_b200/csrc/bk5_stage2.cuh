// BK5 variant 9, "stage2": the stage kernel (bk5_stage.cuh) with TWO threads
// per pencil, for the high orders where one CTA (6-8 warps) per SM is all the
// shared memory allows.
//
// Why: ncu of bk5_stage at N = 12 (profiles/r2y_stage13_phase_stalls.txt)
// shows no memory stall left -- 0 excess shared wavefronts, issue active 38%
// -- but one 6-warp CTA per SM: every contraction phase is a short, barrier-
// delimited burst whose dependency chains (shared-load -> DFMA chain ->
// shared-store) 1.5 warps per scheduler cannot hide.  Here the CTA has two
// halves of ceil(NQ^2 / 32) warps each (h = warp-uniform half index); both
// halves load the same pencil (16 distinct addresses per warp instruction =
// the same wavefront count per distinct line, broadcast within the pair is
// not needed because the halves are different warps), form the even-odd
// sums, and each computes the outputs of its own pair range of the even-odd
// split (half 0: pairs [0, K0), half 1: pairs [K0, N/2) and the middle row
// at odd N+1).  Per output the FMA sequence is exactly matvec's, so results
// are bit-identical to pencil2 / stage.
//
// Per element (two u buffers, G staged, R and S as in stage):
//   F1 i-pencils  u row     -> my ur outputs -> R
//   F2 j-pencils  u column  -> my us outputs -> S
//   F3 k-pencils  u column  -> my ut outputs (registers)         ; sync (A)
//   G  k-pencils  my points: R, S <- gr, gs ; gt -> the spent u buffer ; sync (B)
//   B2 j-pencils  S column -> registers ; sync ; my D^T gs outputs -> S ; sync
//   B3 k-pencils  gt column (u buffer) -> my D^T gt outputs, S += ; sync
//   B1 i-pencils  R row, S row -> my w outputs -> u buffer rows   ; sync (C)
//   bulk store of w (as stage)
// Six block barriers per element (stage: five) -- the in-place B2 needs
// its reads complete before either half writes.
#pragma once
#include <type_traits>

#include "bk5_stage.cuh"

namespace nk {

// Pair ranges of the even-odd split per half.
template <int NQ, int HALF>
struct HalfSet {
  static constexpr int H = NQ / 2, ODD = NQ & 1;
  static constexpr int K0 = (H + 1) / 2;
  static constexpr int P0 = HALF == 0 ? 0 : K0, P1 = HALF == 0 ? K0 : H;
  static constexpr int MID = (HALF == 1 && ODD) ? 1 : 0;
  static constexpr int CNT = 2 * (P1 - P0) + MID;
  // output index (along the pencil) of slot j
  __host__ __device__ static constexpr int idx(int j) {
    return j < 2 * (P1 - P0) ? ((j & 1) ? NQ - 1 - (P0 + j / 2) : P0 + j / 2) : H;
  }
};
template <int NQ>
struct HalfMax {
  static constexpr int CNT =
      HalfSet<NQ, 0>::CNT > HalfSet<NQ, 1>::CNT ? HalfSet<NQ, 0>::CNT : HalfSet<NQ, 1>::CNT;
};

// matvec restricted to this half's outputs: out[j] = (D v)[HalfSet::idx(j)]
// (TRANS: D^T), the same FMA order as matvec (bk5_pencil.cuh).
template <int NQ, bool TRANS, int HALF>
__device__ __forceinline__ void matvec_half(const DParam<NQ>& D, const double (&v)[NQ],
                                            double (&out)[HalfMax<NQ>::CNT]) {
  using HS = HalfSet<NQ, HALF>;
  constexpr int H = NQ / 2, ODD = NQ & 1, HE = H + ODD;
  constexpr int OFF = TRANS ? DParam<NQ>::EOF_ : 0;
  double s[H > 0 ? H : 1], d[H > 0 ? H : 1];
#pragma unroll
  for (int m = 0; m < H; ++m) {
    s[m] = v[m] + v[NQ - 1 - m];
    d[m] = v[m] - v[NQ - 1 - m];
  }
#pragma unroll
  for (int q = HS::P0; q < HS::P1; ++q) {
    double e = 0.0, o = 0.0;
#pragma unroll
    for (int m = 0; m < H; ++m) {
      e = fma(D.eo[OFF + DParam<NQ>::ei(q, m)], s[m], e);
      o = fma(D.eo[OFF + DParam<NQ>::oi(q, m)], d[m], o);
    }
    if (ODD) e = fma(D.eo[OFF + DParam<NQ>::ei(q, H)], v[H], e);
    out[2 * (q - HS::P0)] = o + e;
    out[2 * (q - HS::P0) + 1] = o - e;
  }
  if (HS::MID) {
    double mm = 0.0;
#pragma unroll
    for (int m = 0; m < H; ++m) mm = fma(D.eo[OFF + DParam<NQ>::mi(m)], d[m], mm);
    out[HS::CNT - 1] = mm;
  }
}

template <int NQ, int NGS>
struct Stage2Cfg {
  static constexpr int NQ2 = NQ * NQ, NQ3 = NQ2 * NQ;
  static constexpr int HALF_T = (NQ2 + 31) / 32 * 32;   // threads per half (whole warps)
  static constexpr int THREADS = 2 * HALF_T;
  using SC = StageCfg<NQ, NGS, 2>;
  static size_t smem_bytes() { return SC::smem_bytes(); }
};

template <int NQ, int NGS, int MINB>
__global__ void __launch_bounds__(Stage2Cfg<NQ, NGS>::THREADS, MINB)
bk5_stage2(int64_t nlist, const int32_t* __restrict__ elist, const __grid_constant__ DParam<NQ> D,
           const double* __restrict__ G, const double* __restrict__ u, double* __restrict__ w,
           double lam0, const double* __restrict__ B, double lam1,
           const uint8_t* __restrict__ mask, nk_cg_state* st, double* __restrict__ partials,
           int64_t part_base, int64_t reduce_count, int64_t u_len) {
  using L = PencilLayout<NQ>;
  using C2 = Stage2Cfg<NQ, NGS>;
  using C = typename C2::SC;
  constexpr int NQ2 = C::NQ2, NQ3 = C::NQ3, VOL = C::VOL, CM = HalfMax<NQ>::CNT;
  extern __shared__ __align__(128) double smem[];
  if (st != nullptr && st->done) return;
  double* Ub0 = smem;
  double* Gb = Ub0 + 2 * C::UB;
  double* Rr = Gb + C::GBUF;
  double* Ss = Rr + VOL;
  double* red = Ss + VOL;
  uint64_t* ubar = reinterpret_cast<uint64_t*>(red + 32);   // [2]
  uint64_t* gbar = ubar + 2;

  const int t = threadIdx.x;
  const int h = t / C2::HALF_T;            // warp-uniform
  const int tt = t - h * C2::HALF_T;
  const bool act = tt < NQ2;
  const int a = act ? tt % NQ : 0, b = act ? tt / NQ : 0;
  const int64_t stride = gridDim.x;
  const bool bulkw = ((reinterpret_cast<uintptr_t>(u) ^ reinterpret_cast<uintptr_t>(w)) & 15) == 0;
  auto elem_of = [&](int64_t slot) -> int64_t { return elist ? (int64_t)elist[slot] : slot; };
  auto phase_of = [&](int64_t e) -> int {
    return (int)((reinterpret_cast<uintptr_t>(u + e * NQ3) >> 3) & 1);
  };
  auto issue_u = [&](int64_t slot, int bi) {   // thread 0 (as bk5_stage)
    const int64_t s0 = elem_of(slot) * NQ3;
    const int sh = phase_of(s0 / NQ3);
    int64_t cnt = (NQ3 + sh + 1) & ~int64_t(1);
    const bool tail = s0 - sh + cnt > u_len;
    if (tail) cnt -= 2;
    double* dst = Ub0 + bi * C::UB;
    mbar_expect_tx(&ubar[bi], (uint32_t)(cnt * sizeof(double)));
    tma_load_1d(dst, u + s0 - sh, (uint32_t)(cnt * sizeof(double)), &ubar[bi]);
    if (tail) {
      dst[cnt] = u[s0 - sh + cnt];
      fence_proxy_async();
    }
  };
  auto issue_g = [&](int64_t slot) {
    const double* src = G + elem_of(slot) * 6 * NQ3;
    constexpr uint32_t GBYTES = (uint32_t)(((NGS * NQ3 + 1) & ~1) * sizeof(double));
    mbar_expect_tx(gbar, GBYTES);
    tma_load_1d(Gb, src, GBYTES, gbar);
    if (NGS < 6) prefetch_l2(src + NGS * NQ3, (int64_t)(6 - NGS) * NQ3 * sizeof(double));
  };

  if (t == 0) {
    mbar_init(&ubar[0], 1);
    mbar_init(&ubar[1], 1);
    mbar_init(gbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t == 0 && (int64_t)blockIdx.x < nlist) {
    issue_u(blockIdx.x, 0);
    issue_g(blockIdx.x);
  }
  __syncthreads();

  using H0 = std::integral_constant<int, 0>;
  using H1 = std::integral_constant<int, 1>;
  double dot = 0.0;
  int it = 0;
  for (int64_t slot = blockIdx.x; slot < nlist; slot += stride, ++it) {
    const int64_t e = elem_of(slot);
    const int sh = phase_of(e);
    const int bi = it & 1;
    double* uS = Ub0 + bi * C::UB + sh;
    if (t == 0 && slot + stride < nlist) {
      bulk_wait_read0();
      issue_u(slot + stride, bi ^ 1);
    }
    mbar_wait(&ubar[bi], (it >> 1) & 1);
    double ut[CM];
    auto fwd = [&](auto hc) {
      constexpr int HF = decltype(hc)::value;
      using HS = HalfSet<NQ, HF>;
      double v[NQ], o[CM];
      // F1: i-pencil (j = a, k = b)
      const double* row = uS + b * NQ2 + a * NQ;
      if (NQ % 2 == 0 && sh == 0) {
#pragma unroll
        for (int m = 0; m < NQ; m += 2) {
          const double2 p = *reinterpret_cast<const double2*>(row + m);
          v[m] = p.x;
          v[m + 1] = p.y;
        }
      } else {
#pragma unroll
        for (int m = 0; m < NQ; ++m) v[m] = row[m];
      }
      matvec_half<NQ, false, HF>(D, v, o);
#pragma unroll
      for (int j = 0; j < HS::CNT; ++j) Rr[L::idx(b, a, HS::idx(j))] = o[j];
      // F2: j-pencil (i = a, k = b)
#pragma unroll
      for (int m = 0; m < NQ; ++m) v[m] = uS[b * NQ2 + m * NQ + a];
      matvec_half<NQ, false, HF>(D, v, o);
#pragma unroll
      for (int j = 0; j < HS::CNT; ++j) Ss[L::idx(b, HS::idx(j), a)] = o[j];
      // F3: k-pencil (i = a, j = b) -> ut
#pragma unroll
      for (int m = 0; m < NQ; ++m) v[m] = uS[m * NQ2 + b * NQ + a];
      matvec_half<NQ, false, HF>(D, v, ut);
    };
    if (act) {
      if (h == 0) fwd(H0{}); else fwd(H1{});
    }
    __syncthreads();   // (A) u read for the last time: the buffer takes gt
    mbar_wait(gbar, it & 1);
    auto gph = [&](auto hc) {
      constexpr int HF = decltype(hc)::value;
      using HS = HalfSet<NQ, HF>;
      const double* gp = G + e * 6 * NQ3 + b * NQ + a;
#pragma unroll
      for (int j = 0; j < HS::CNT; ++j) {
        const int k = HS::idx(j);
        const int p = k * NQ2 + b * NQ + a;
        double g[6];
#pragma unroll
        for (int c = 0; c < 6; ++c)
          g[c] = c < NGS ? Gb[c * NQ3 + p] : __ldg(gp + c * NQ3 + k * NQ2);
        const int q = L::idx(k, b, a);
        const double ur = Rr[q], us = Ss[q];
        Rr[q] = g[0] * ur + g[1] * us + g[2] * ut[j];
        Ss[q] = g[1] * ur + g[3] * us + g[4] * ut[j];
        uS[p] = g[2] * ur + g[4] * us + g[5] * ut[j];   // gt, dense (k, j, i)
      }
    };
    if (act) {
      if (h == 0) gph(H0{}); else gph(H1{});
    }
    __syncthreads();   // (B) G buffer read for the last time
    if (t == 0 && slot + stride < nlist) issue_g(slot + stride);
    {  // B2: j-pencils, in place on S: all reads, barrier, then each half writes
      double v[NQ];
      if (act) {
#pragma unroll
        for (int m = 0; m < NQ; ++m) v[m] = Ss[L::idx(b, m, a)];
      }
      __syncthreads();
      auto b2 = [&](auto hc) {
        constexpr int HF = decltype(hc)::value;
        using HS = HalfSet<NQ, HF>;
        double o[CM];
        matvec_half<NQ, true, HF>(D, v, o);
#pragma unroll
        for (int j = 0; j < HS::CNT; ++j) Ss[L::idx(b, HS::idx(j), a)] = o[j];
      };
      if (act) {
        if (h == 0) b2(H0{}); else b2(H1{});
      }
    }
    __syncthreads();
    auto b3 = [&](auto hc) {   // B3: k-pencils, S += D^T gt (gt column from the u buffer)
      constexpr int HF = decltype(hc)::value;
      using HS = HalfSet<NQ, HF>;
      double v[NQ], o[CM];
#pragma unroll
      for (int m = 0; m < NQ; ++m) v[m] = uS[m * NQ2 + b * NQ + a];
      matvec_half<NQ, true, HF>(D, v, o);
#pragma unroll
      for (int j = 0; j < HS::CNT; ++j) {
        const int q = L::idx(HS::idx(j), b, a);
        Ss[q] = o[j] + Ss[q];
      }
    };
    if (act) {
      if (h == 0) b3(H0{}); else b3(H1{});
    }
    __syncthreads();
    auto b1 = [&](auto hc) {   // B1: i-pencils + epilogue, w outputs into the u buffer rows
      constexpr int HF = decltype(hc)::value;
      using HS = HalfSet<NQ, HF>;
      double v[NQ], o[CM];
#pragma unroll
      for (int m = 0; m < NQ; ++m) v[m] = Rr[L::idx(b, a, m)];
      matvec_half<NQ, true, HF>(D, v, o);
      const int64_t off = e * NQ3 + b * NQ2 + a * NQ;
      double* urow = uS + b * NQ2 + a * NQ;
#pragma unroll
      for (int j = 0; j < HS::CNT; ++j) {
        const int i = HS::idx(j);
        double r = lam0 * (o[j] + Ss[L::idx(b, a, i)]);
        if (B != nullptr || st != nullptr) {
          const double uu = __ldg(u + off + i);
          if (B != nullptr) r = fma(lam1 * __ldg(B + off + i), uu, r);
          if (mask != nullptr) r = mask[off + i] ? r : 0.0;
          dot = fma(uu, r, dot);
        } else if (mask != nullptr) {
          r = mask[off + i] ? r : 0.0;
        }
        if (bulkw) {
          urow[i] = r;
          if (i == 0 && tt == 0 && sh) w[e * NQ3] = r;
          if (i == NQ - 1 && tt == NQ2 - 1 && ((NQ3 - sh) & 1)) w[e * NQ3 + NQ3 - 1] = r;
        } else {
          w[off + i] = r;
        }
      }
      if (bulkw) fence_proxy_async();
    };
    if (act) {
      if (h == 0) b1(H0{}); else b1(H1{});
    }
    __syncthreads();   // (C) R, S free; w rows in shared
    if (bulkw && t == 0) {
      const int64_t cnt = (NQ3 - sh) & ~int64_t(1);
      bulk_store(w + e * NQ3 + sh, uS + sh, (uint32_t)(cnt * sizeof(double)));
      bulk_commit();
    }
  }
  if (t == 0) bulk_wait0();

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

template <int NQ, int NGS, int MINB>
static int64_t stage2_grid(int64_t nlist) {
  static int64_t resident = -1;
  if (resident < 0) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    using C2 = Stage2Cfg<NQ, NGS>;
    cudaFuncSetAttribute(bk5_stage2<NQ, NGS, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C2::smem_bytes());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bk5_stage2<NQ, NGS, MINB>, C2::THREADS,
                                                  C2::smem_bytes());
    resident = (int64_t)sms * (per > 0 ? per : 1);
  }
  return nlist < resident ? nlist : resident;
}

template <int NQ, int NGS, int MINB>
static int launch_stage2(int64_t nlist, const int32_t* elist, const double* Dhost,
                         const double* G, const double* u, double* w, double lam0,
                         const double* B, double lam1, const uint8_t* mask, nk_cg_state* st,
                         double* partials, int64_t part_base, int64_t reduce_count,
                         int64_t u_len, cudaStream_t s) {
  using C2 = Stage2Cfg<NQ, NGS>;
  const int64_t grid = stage2_grid<NQ, NGS, MINB>(nlist);
  if (grid == 0) return NK_OK;
  if ((reinterpret_cast<uintptr_t>(u) & 7) || (reinterpret_cast<uintptr_t>(G) & 15)) {
    set_error("bk5_stage2: u must be 8-byte and G 16-byte aligned");
    return NK_ERR_INVALID;
  }
  DParam<NQ> D;
  D.set(Dhost);
  bk5_stage2<NQ, NGS, MINB><<<(unsigned)grid, C2::THREADS, C2::smem_bytes(), s>>>(
      nlist, elist, D, G, u, w, lam0, B, lam1, mask, st, partials, part_base, reduce_count, u_len);
  return check_launch("bk5_stage2");
}

}  // namespace nk
