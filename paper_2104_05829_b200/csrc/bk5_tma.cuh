// BK5 variant 4, "pencil-TMA": persistent CTAs; the element stream (u and the
// six G factors, contiguous per element) is moved HBM -> shared memory by the
// TMA engine (cp.async.bulk, SASS UBLKCP) into a 2-stage ring with mbarrier
// transaction counts, so DRAM traffic for element e+2 is in flight while the
// CTA computes element e+1 -- memory-level parallelism no longer depends on
// registers or occupancy.  Compute is the pencil scheme of bk5_pencil.cuh
// (register 1-D contractions, D in the constant bank, swizzled transposes),
// reordered so the first pass reads u from the stage in the conflict-free
// k-pencil orientation.
//
// Per element (NQ^2 threads; t = a + NQ*b):
//   F3  k-pencils (i=a,j=b): u column from stage -> ut = D u (regs); U <- u
//   F1  i-pencils (j=a,k=b): U row   -> ur -> R ;  F2 j-pencils: U col -> us -> S
//   G   k-pencils: G from stage, R,S,ut -> gr,gs (in place), gt (regs); wt -> U
//   B2  j-pencils: U += D^T gs ;  B1 i-pencils: w = D^T gr + U -> epilogue -> HBM
// Requirements: NQ even (16-byte bulk-copy granularity of u and G).
#pragma once
#include "bk5_pencil.cuh"

namespace nk {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// expected-transaction bytes without an arrival (the arrival comes later)
__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_1d_hint(void* dst, const void* src, uint32_t bytes,
                                                 uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

template <int NQ, int MINB>
struct TmaCfg {
  static constexpr int NQ2 = NQ * NQ, NQ3 = NQ2 * NQ;
  static constexpr int THREADS = NQ2;
  static constexpr int STAGE = 7 * NQ3;  // doubles: u then G[6]
  static constexpr int VOL = PencilLayout<NQ>::VOL;
  // layout (doubles): stage[2] | U R S | red[32] ; mbarriers after
  static size_t smem_bytes() { return sizeof(double) * (2 * STAGE + 3 * VOL + 32) + 2 * 8; }
};

template <int NQ, int MINB>
__global__ void __launch_bounds__(NQ * NQ, MINB)
bk5_pencil_tma(int64_t nlist, const int32_t* __restrict__ elist,
               const __grid_constant__ DParam<NQ> D, const double* __restrict__ G,
               const double* __restrict__ u, double* __restrict__ w, double lam0,
               const double* __restrict__ B, double lam1, const uint8_t* __restrict__ mask,
               nk_cg_state* st, double* __restrict__ partials, int64_t part_base,
               int64_t reduce_count) {
  static_assert(NQ % 2 == 0, "bulk copies need 16-byte multiples");
  using L = PencilLayout<NQ>;
  using C = TmaCfg<NQ, MINB>;
  constexpr int NQ2 = C::NQ2, NQ3 = C::NQ3, VOL = C::VOL, STAGE = C::STAGE;
  extern __shared__ __align__(128) double smem[];
  if (st != nullptr && st->done) return;

  double* stage0 = smem;
  double* U = smem + 2 * STAGE;
  double* Rr = U + VOL;
  double* Ss = Rr + VOL;
  double* red = Ss + VOL;
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + 32);

  const int t = threadIdx.x;
  const int a = t % NQ, b = t / NQ;
  const int64_t stride = gridDim.x;
  constexpr uint32_t UB = NQ3 * sizeof(double), GB = 6 * NQ3 * sizeof(double);

  auto elem_of = [&](int64_t slot) -> int64_t { return elist ? (int64_t)elist[slot] : slot; };
  auto issue = [&](int64_t slot, int s) {
    const int64_t e = elem_of(slot);
    double* dst = stage0 + s * STAGE;
    mbar_expect_tx(&bar[s], UB + GB);
    tma_load_1d(dst, u + e * NQ3, UB, &bar[s]);
    tma_load_1d(dst + NQ3, G + e * 6 * NQ3, GB, &bar[s]);
  };

  if (t == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t == 0) {
    if ((int64_t)blockIdx.x < nlist) issue(blockIdx.x, 0);
    if ((int64_t)blockIdx.x + stride < nlist) issue(blockIdx.x + stride, 1);
  }

  double dot = 0.0;
  int it = 0;
  for (int64_t slot = blockIdx.x; slot < nlist; slot += stride, ++it) {
    const int s = it & 1;
    const double* su = stage0 + s * STAGE;
    const double* sg = su + NQ3;
    const int64_t e = elem_of(slot);
    mbar_wait(&bar[s], (it >> 1) & 1);

    // ---- F3: k-pencils (i = a, j = b) from the stage: ut in registers; U <- u
    double ut[NQ];
    {
      double v[NQ];
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        v[k] = su[k * NQ2 + b * NQ + a];
        U[L::idx(k, b, a)] = v[k];
      }
      matvec<NQ, false>(D, v, ut);
    }
    __syncthreads();
    // ---- F1: i-pencils (j = a, k = b) -> R ; F2: j-pencils (i = a, k = b) -> S
    {
      double v[NQ], o[NQ];
#pragma unroll
      for (int m = 0; m < NQ; ++m) v[m] = U[L::idx(b, a, m)];
      matvec<NQ, false>(D, v, o);
#pragma unroll
      for (int i = 0; i < NQ; ++i) Rr[L::idx(b, a, i)] = o[i];
#pragma unroll
      for (int m = 0; m < NQ; ++m) v[m] = U[L::idx(b, m, a)];
      matvec<NQ, false>(D, v, o);
#pragma unroll
      for (int j = 0; j < NQ; ++j) Ss[L::idx(b, j, a)] = o[j];
    }
    __syncthreads();
    // ---- G: k-pencils; then wt = D^T gt -> U (U's u copy is no longer read)
    {
      double gt[NQ];
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        const int p = k * NQ2 + b * NQ + a;
        const double g0 = sg[0 * NQ3 + p], g1 = sg[1 * NQ3 + p], g2 = sg[2 * NQ3 + p];
        const double g3 = sg[3 * NQ3 + p], g4 = sg[4 * NQ3 + p], g5 = sg[5 * NQ3 + p];
        const int q = L::idx(k, b, a);
        const double ur = Rr[q], us = Ss[q];
        Rr[q] = g0 * ur + g1 * us + g2 * ut[k];
        Ss[q] = g1 * ur + g3 * us + g4 * ut[k];
        gt[k] = g2 * ur + g4 * us + g5 * ut[k];
      }
      double o[NQ];
      matvec<NQ, true>(D, gt, o);
#pragma unroll
      for (int k = 0; k < NQ; ++k) U[L::idx(k, b, a)] = o[k];
    }
    __syncthreads();
    // ---- B2: j-pencils: U <- D^T gs + wt
    {
      double v[NQ], o[NQ];
#pragma unroll
      for (int m = 0; m < NQ; ++m) v[m] = Ss[L::idx(b, m, a)];
      matvec<NQ, true>(D, v, o);
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        const int q = L::idx(b, j, a);
        U[q] = o[j] + U[q];
      }
    }
    __syncthreads();
    // ---- B1: i-pencils (j = a, k = b): w = D^T gr + U, epilogue, store
    {
      double v[NQ], o[NQ];
#pragma unroll
      for (int m = 0; m < NQ; ++m) v[m] = Rr[L::idx(b, a, m)];
      matvec<NQ, true>(D, v, o);
      const int64_t off = e * NQ3 + b * NQ2 + a * NQ;
      const double* urow = su + b * NQ2 + a * NQ;
      double res[NQ];
#pragma unroll
      for (int i = 0; i < NQ; ++i) res[i] = lam0 * (o[i] + U[L::idx(b, a, i)]);
      if (B != nullptr) {
#pragma unroll
        for (int i = 0; i < NQ; ++i) res[i] = fma(lam1 * __ldg(B + off + i), urow[i], res[i]);
      }
      if (mask != nullptr) {
#pragma unroll
        for (int i = 0; i < NQ; ++i) res[i] = mask[off + i] ? res[i] : 0.0;
      }
      if (st != nullptr) {
#pragma unroll
        for (int i = 0; i < NQ; ++i) dot = fma(urow[i], res[i], dot);
      }
      double* wr = w + off;
#pragma unroll
      for (int i = 0; i < NQ; i += 2)
        *reinterpret_cast<double2*>(wr + i) = make_double2(res[i], res[i + 1]);
    }
    __syncthreads();  // stage s and U/R/S free
    if (t == 0 && slot + 2 * stride < nlist) issue(slot + 2 * stride, s);
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

// Grid: persistent, min(nlist, SMs * resident CTAs per SM).
template <int NQ, int MINB>
static int64_t tma_grid(int64_t nlist) {
  static int64_t resident = -1;
  if (resident < 0) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    using C = TmaCfg<NQ, MINB>;
    cudaFuncSetAttribute(bk5_pencil_tma<NQ, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::smem_bytes());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bk5_pencil_tma<NQ, MINB>, C::THREADS,
                                                  C::smem_bytes());
    resident = (int64_t)sms * (per > 0 ? per : 1);
  }
  return nlist < resident ? nlist : resident;
}

template <int NQ, int MINB>
static int launch_pencil_tma(int64_t nlist, const int32_t* elist, const double* Dhost,
                             const double* G, const double* u, double* w, double lam0,
                             const double* B, double lam1, const uint8_t* mask, nk_cg_state* st,
                             double* partials, int64_t part_base, int64_t reduce_count,
                             cudaStream_t s) {
  using C = TmaCfg<NQ, MINB>;
  const int64_t grid = tma_grid<NQ, MINB>(nlist);
  if (grid == 0) return NK_OK;
  if ((reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(G)) & 15) {
    set_error("bk5_pencil_tma: u and G must be 16-byte aligned");
    return NK_ERR_INVALID;
  }
  DParam<NQ> D;
  D.set(Dhost);
  bk5_pencil_tma<NQ, MINB><<<(unsigned)grid, C::THREADS, C::smem_bytes(), s>>>(
      nlist, elist, D, G, u, w, lam0, B, lam1, mask, st, partials, part_base, reduce_count);
  return check_launch("bk5_pencil_tma");
}

}  // namespace nk

namespace nk {

// ---------------------------------------------------------------------------
// Fused BP5 operator step on the TMA pipeline (see bk5_pcg.cuh for the math):
// the stage carries p_{k-1}, r_k, invD and G of an element (9 NQ^3 doubles);
// F3 (k-pencils, coalesced) forms p_k = invD r + beta p_{k-1}, writes it to HBM
// and back into the stage, and applies the deferred x += alpha_{k-1} p_{k-1}
// with x read/written directly (coalesced planes).  On the stop iteration only
// the x update runs (no TMA traffic).
// SB (single buffers, the stage-kernel scheme, bk5_stage.cuh): ONE p buffer
// and ONE G buffer instead of the 2-stage (p, G) ring -- p(next) is issued as
// soon as F3 has read the current p, G(next) as soon as the G phase is done
// -- so a CTA needs 42 KB of shared memory instead of 71 KB and four or five
// CTAs fit on an SM instead of three (NK_KNOB_TMA; four is the default:
// 0.1080 -> 0.1068 ms per BP5 iteration, profiles/r2zo_bp5_tma_knob.jsonl).
template <int NQ, int MINB, bool SB = false>
struct TmaPcgCfg {
  static constexpr int NQ2 = NQ * NQ, NQ3 = NQ2 * NQ;
  static constexpr int THREADS = NQ2;
  static constexpr int STAGE = 7 * NQ3;  // p, G[6]  (r, invD, x: plain loads)
  static constexpr int NST = SB ? 1 : 2;
  static constexpr int VOL = PencilLayout<NQ>::VOL;
  static size_t smem_bytes() { return sizeof(double) * (NST * STAGE + 3 * VOL + 32) + 2 * 8; }
};

template <int NQ, int MINB, bool SB, bool TAIL>
__device__ __forceinline__ void tma_pcg_body(int64_t nlist, const int32_t* __restrict__ elist,
                   const DParam<NQ>& D, const double* __restrict__ G,
                   double* __restrict__ p, double* __restrict__ w, double lam0,
                   const double* __restrict__ B, double lam1, const uint8_t* __restrict__ mask,
                   double* __restrict__ x, const double* __restrict__ r,
                   const double* __restrict__ invD, nk_cg_state* st,
                   double* __restrict__ partials, int64_t part_base, int64_t reduce_count,
                   double* __restrict__ hist, int pdl_flags, int l2_flags,
                   const GsTail& tail) {
  static_assert(NQ % 2 == 0, "bulk copies need 16-byte multiples");
  using L = PencilLayout<NQ>;
  using C = TmaPcgCfg<NQ, MINB, SB>;
  constexpr int NQ2 = C::NQ2, NQ3 = C::NQ3, VOL = C::VOL, STAGE = C::STAGE;
  extern __shared__ __align__(128) double smem[];
  double* stage0 = smem;   // SB: [p | G], bar[0] = p, bar[1] = G
  double* U = smem + C::NST * STAGE;
  double* Rr = U + VOL;
  double* Ss = Rr + VOL;
  double* red = Ss + VOL;
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + 32);

  const int t = threadIdx.x;
  const int a = t % NQ, b = t / NQ;
  const int64_t stride = gridDim.x;
  constexpr uint32_t UB = NQ3 * sizeof(double), GB = 6 * NQ3 * sizeof(double);
  auto elem_of = [&](int64_t slot) -> int64_t { return elist ? (int64_t)elist[slot] : slot; };
  // L2 policies (NK_KNOB_L2): streamed once per iteration (G, p, x, mask)
  // vs reused by the iteration's update kernel (r, w) and invD
  const uint64_t pol_s = l2_policy(l2_flags & kL2StreamFirst ? 1 : 0);
  const uint64_t pol_r = l2_policy(l2_flags & kL2ReuseLast ? 2 : 0);
  const uint64_t pol_d = l2_policy(l2_flags & kL2InvDLast ? 2 : 0);

  // PDL prologue: G (static) of this CTA's first two elements starts moving
  // while the predecessor kernel drains.  The stage's mbarrier gets the G
  // bytes as expected transactions but no arrival, so its phase cannot
  // complete before the p copy (or the drain below) arrives.  The done read
  // is a racy hint only (done is monotonic within a graph-replayed chunk).
  __shared__ int s_pre;
  if (t == 0) {
    s_pre = !(pdl_flags & kPdlNoPrologue) &&
            *reinterpret_cast<volatile const int*>(&st->done) == 0;
    const bool pre = s_pre;
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (pre) {
      for (int s = 0; s < C::NST; ++s) {
        const int64_t slot = blockIdx.x + s * stride;
        if (slot < nlist) {
          uint64_t* gb = SB ? &bar[1] : &bar[s];
          mbar_expect_tx_only(gb, GB);
          tma_load_1d_hint(stage0 + s * STAGE + NQ3, G + elem_of(slot) * 6 * NQ3, GB, gb, pol_s);
        }
      }
    }
  }
  __syncthreads();
  const bool pre = s_pre;
  pdl_wait();
  if (!(pdl_flags & kPdlLateTrigger)) pdl_trigger();
  const bool done = st->done != 0;
  const int it = st->iter;
  const bool conv = it > 0 && st->rr <= st->thresh2;
  const bool stop = it > 0 && (conv || it >= st->max_iter);
  if (pre && (done || stop)) {  // drain the prologue copies before smem is released
    for (int s = 0; s < C::NST; ++s) {
      if (blockIdx.x + s * stride < nlist) {
        uint64_t* gb = SB ? &bar[1] : &bar[s];
        if (t == 0) mbar_arrive(gb);
        mbar_wait(gb, 0);
      }
    }
  }
  if (done) return;
  const double alpha_prev = st->alpha;
  const double rz = st->rz;
  const double beta =
      it == 0 ? 0.0 : (st->flexible ? (-alpha_prev * st->zap) / rz : st->rz_new / rz);
  double dot = 0.0;

  if (stop) {  // final deferred x update only
    for (int64_t slot = blockIdx.x; slot < nlist; slot += stride) {
      const int64_t e = elem_of(slot);
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        const int64_t q = e * NQ3 + k * NQ2 + t;
        st_hint(x + q, fma(alpha_prev, ld_hint(p + q, pol_s), ld_hint(x + q, pol_s)), pol_s);
      }
    }
  } else {
    // g: whether the stage's G copy is already in flight (the prologue)
    auto issue = [&](int64_t slot, int s, bool g) {
      const int64_t e = elem_of(slot);
      double* dst = stage0 + s * STAGE;
      mbar_expect_tx(&bar[s], g ? UB : UB + GB);
      tma_load_1d_hint(dst, p + e * NQ3, UB, &bar[s], pol_s);
      if (!g) tma_load_1d_hint(dst + NQ3, G + e * 6 * NQ3, GB, &bar[s], pol_s);
      // r, invD, x and mask of the same element are read with plain
      // (coalesced) loads: start them towards L2 now, two elements ahead
      if (it > 0) {
        prefetch_l2_hint(r + e * NQ3, UB, pol_r);
        prefetch_l2_hint(invD + e * NQ3, UB, pol_d);
        prefetch_l2_hint(x + e * NQ3, UB, pol_s);
      }
      if (mask != nullptr) prefetch_l2_hint(mask + e * NQ3, NQ3, pol_s);
    };
    // SB: p and G travel separately (bar[0] p, bar[1] G)
    auto issue_p = [&](int64_t slot) {
      const int64_t e = elem_of(slot);
      mbar_expect_tx(&bar[0], UB);
      tma_load_1d_hint(stage0, p + e * NQ3, UB, &bar[0], pol_s);
      if (it > 0) {
        prefetch_l2_hint(r + e * NQ3, UB, pol_r);
        prefetch_l2_hint(invD + e * NQ3, UB, pol_d);
        prefetch_l2_hint(x + e * NQ3, UB, pol_s);
      }
      if (mask != nullptr) prefetch_l2_hint(mask + e * NQ3, NQ3, pol_s);
    };
    auto issue_g = [&](int64_t slot, bool arrive) {
      const int64_t e = elem_of(slot);
      if (arrive) mbar_expect_tx(&bar[1], GB);
      tma_load_1d_hint(stage0 + NQ3, G + e * 6 * NQ3, GB, &bar[1], pol_s);
    };
    if (t == 0) {
      if (SB) {
        if ((int64_t)blockIdx.x < nlist) {
          issue_p(blockIdx.x);
          if (pre) mbar_arrive(&bar[1]);      // the prologue's G copy: its arrival
          else issue_g(blockIdx.x, true);
        }
      } else {
        if ((int64_t)blockIdx.x < nlist) issue(blockIdx.x, 0, pre);
        if ((int64_t)blockIdx.x + stride < nlist) issue(blockIdx.x + stride, 1, pre);
      }
    }
    // x, r, invD columns (k-pencil, coalesced planes) and the mask row of
    // an element are loaded into registers one element AHEAD (software
    // pipelined across the persistent loop), so their L2 latency overlaps
    // a whole element's contractions instead of the F3 prologue (ncu phase
    // attribution, profiles/r2zc_*: F3 long-scoreboard 56%).
    double xv[NQ], rv[NQ], dv[NQ];
    uint64_t mk = ~0ull;
    const bool mask8 = NQ == 8 && mask != nullptr && (reinterpret_cast<uintptr_t>(mask) & 7) == 0;
    auto load_vec = [&](int64_t slot, double (&xo)[NQ], double (&ro)[NQ], double (&dvo)[NQ],
                        uint64_t& mo) {
      const int64_t e = elem_of(slot);
      if (it > 0) {
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
          const int64_t q = e * NQ3 + k * NQ2 + t;
          xo[k] = ld_hint(x + q, pol_s);
          ro[k] = ldg_hint(r + q, pol_r);
          dvo[k] = ldg_hint(invD + q, pol_d);
        }
      }
      if (mask8)   // the B1 row (j = a, k = b): 8 bytes
        mo = __ldg(reinterpret_cast<const unsigned long long*>(mask + e * NQ3 + b * NQ2 +
                                                               a * NQ));
    };
    if ((int64_t)blockIdx.x < nlist) load_vec(blockIdx.x, xv, rv, dv, mk);
    int itl = 0;
    for (int64_t slot = blockIdx.x; slot < nlist; slot += stride, ++itl) {
      const int s = SB ? 0 : (itl & 1);
      double* su = stage0 + s * STAGE;
      const double* sg = su + NQ3;
      const int64_t e = elem_of(slot);
      mbar_wait(&bar[s], SB ? (itl & 1) : ((itl >> 1) & 1));

      // ---- F3 + prologue: k-pencils (i = a, j = b)
      double ut[NQ];
      {
        double v[NQ];
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
          const int pp = k * NQ2 + t;
          double pv = su[pp];
          if (it > 0) {
            st_hint(x + e * NQ3 + pp, fma(alpha_prev, pv, xv[k]), pol_s);
            pv = fma(beta, pv, dv[k] * rv[k]);
            st_hint(p + e * NQ3 + pp, pv, pol_s);
          }
          v[k] = pv;
          U[L::idx(k, b, a)] = pv;
        }
        matvec<NQ, false>(D, v, ut);
      }
      // the next element's vectors: in flight for the rest of this element
      uint64_t mk_next = ~0ull;
      if (slot + stride < nlist) load_vec(slot + stride, xv, rv, dv, mk_next);
      __syncthreads();
      // SB: the p buffer has been read (it lives on in U): p(next) may land
      if (SB && t == 0 && slot + stride < nlist) issue_p(slot + stride);
      double prow[NQ];   // p row (j = a, k = b): F1's input, B1's dot and mass term
      {  // F1 (i-pencils) -> R ; F2 (j-pencils) -> S
        double v[NQ], o[NQ];
#pragma unroll
        for (int m = 0; m < NQ; ++m) prow[m] = U[L::idx(b, a, m)];
        matvec<NQ, false>(D, prow, o);
#pragma unroll
        for (int i = 0; i < NQ; ++i) Rr[L::idx(b, a, i)] = o[i];
#pragma unroll
        for (int m = 0; m < NQ; ++m) v[m] = U[L::idx(b, m, a)];
        matvec<NQ, false>(D, v, o);
#pragma unroll
        for (int j = 0; j < NQ; ++j) Ss[L::idx(b, j, a)] = o[j];
      }
      __syncthreads();
      if (SB) mbar_wait(&bar[1], itl & 1);
      {  // G (k-pencils), wt -> U
        double gt[NQ];
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
          const int pp = k * NQ2 + t;
          const double g0 = sg[0 * NQ3 + pp], g1 = sg[1 * NQ3 + pp], g2 = sg[2 * NQ3 + pp];
          const double g3 = sg[3 * NQ3 + pp], g4 = sg[4 * NQ3 + pp], g5 = sg[5 * NQ3 + pp];
          const int q = L::idx(k, b, a);
          const double ur = Rr[q], us = Ss[q];
          Rr[q] = g0 * ur + g1 * us + g2 * ut[k];
          Ss[q] = g1 * ur + g3 * us + g4 * ut[k];
          gt[k] = g2 * ur + g4 * us + g5 * ut[k];
        }
        double o[NQ];
        matvec<NQ, true>(D, gt, o);
#pragma unroll
        for (int k = 0; k < NQ; ++k) U[L::idx(k, b, a)] = o[k];
      }
      __syncthreads();
      // SB: the G buffer has been read: G(next) may land
      if (SB && t == 0 && slot + stride < nlist) issue_g(slot + stride, true);
      {  // B2 (j-pencils)
        double v[NQ], o[NQ];
#pragma unroll
        for (int m = 0; m < NQ; ++m) v[m] = Ss[L::idx(b, m, a)];
        matvec<NQ, true>(D, v, o);
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
          const int q = L::idx(b, j, a);
          U[q] = o[j] + U[q];
        }
      }
      __syncthreads();
      {  // B1 (i-pencils) + epilogue
        double v[NQ], o[NQ];
#pragma unroll
        for (int m = 0; m < NQ; ++m) v[m] = Rr[L::idx(b, a, m)];
        matvec<NQ, true>(D, v, o);
        const int64_t off = e * NQ3 + b * NQ2 + a * NQ;
        double res[NQ];
#pragma unroll
        for (int i = 0; i < NQ; ++i) {
          double vv = lam0 * (o[i] + U[L::idx(b, a, i)]);
          if (B != nullptr) vv = fma(lam1 * __ldg(B + off + i), prow[i], vv);
          if (mask != nullptr) {
            const bool keep = mask8 ? ((mk >> (8 * i)) & 0xff) != 0
                                    : ldg_u8_hint(mask + off + i, pol_s) != 0;
            vv = keep ? vv : 0.0;
          }
          res[i] = vv;
          dot = fma(prow[i], vv, dot);
        }
        double* wr = w + off;
#pragma unroll
        for (int i = 0; i < NQ; i += 2)
          st2_hint(wr + i, make_double2(res[i], res[i + 1]), pol_r);
      }
      __syncthreads();
      mk = mk_next;
      if (!SB && t == 0 && slot + 2 * stride < nlist) issue(slot + 2 * stride, s, false);
    }
  }

  if (pdl_flags & kPdlLateTrigger) pdl_trigger();
  double vv[1] = {dot};
  block_sum<1>(vv, red);
  if (t == 0) partials[part_base + blockIdx.x] = vv[0];
  auto finish = [&]() {
    double sres[1];
    reduce_partials<1>(partials, reduce_count, 0, sres, red);
    if (t == 0) {
      if (it > 0 && hist) hist[it] = sqrt(st->rr);
      if (stop) {
        st->converged = conv ? 1 : 0;
        st->done = 1;
      } else {
        st->pAp = sres[0];
        if (it > 0) st->rz = st->rz_new;
      }
    }
  };
  if (TAIL && tail.n > 0 && !stop) {  // every CTA of the grid takes this branch
    const int lane = t & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (t >> 5);
    const int64_t W = tail.wstart[tail.n];
    int idx[kTailU], cls[kTailU];
    gs_tail_idx(tail, gw, nw, lane, idx, cls);  // plan data: in flight across the barrier
    const bool last = grid_barrier(st);
    if (last && reduce_count > 0) finish();
    for (int64_t v0 = gw; v0 < W; v0 += (int64_t)kTailU * nw) {
      if (v0 != gw) gs_tail_idx(tail, v0, nw, lane, idx, cls);
      gs_tail_fold(tail, w, lane, idx, cls);
    }
    return;
  }
  if (reduce_count > 0 && last_block(&st->ticket[0], gridDim.x)) finish();
}

template <int NQ, int MINB, bool SB = false, bool TAIL = false>
__global__ void __launch_bounds__(NQ * NQ, MINB)
bk5_pencil_tma_pcg(int64_t nlist, const int32_t* __restrict__ elist,
                   const __grid_constant__ DParam<NQ> D, const double* __restrict__ G,
                   double* __restrict__ p, double* __restrict__ w, double lam0,
                   const double* __restrict__ B, double lam1, const uint8_t* __restrict__ mask,
                   double* __restrict__ x, const double* __restrict__ r,
                   const double* __restrict__ invD, nk_cg_state* st,
                   double* __restrict__ partials, int64_t part_base, int64_t reduce_count,
                   double* __restrict__ hist, int pdl_flags, int l2_flags,
                   const __grid_constant__ GsTail tail) {
  tma_pcg_body<NQ, MINB, SB, TAIL>(nlist, elist, D, G, p, w, lam0, B, lam1, mask, x, r, invD, st, partials, part_base, reduce_count, hist, pdl_flags, l2_flags, tail);
}

// the same kernel with an explicit register cap (MINB = 5 under
// __launch_bounds__ makes ptxas cap at 168 registers and spill; 200 x 64
// threads x 5 CTAs still fits the 64 K register file)
template <int NQ, int MINB, bool SB, int NREG>
__global__ void __maxnreg__(NREG)
bk5_pencil_tma_pcg_nreg(int64_t nlist, const int32_t* __restrict__ elist,
                   const __grid_constant__ DParam<NQ> D, const double* __restrict__ G,
                   double* __restrict__ p, double* __restrict__ w, double lam0,
                   const double* __restrict__ B, double lam1, const uint8_t* __restrict__ mask,
                   double* __restrict__ x, const double* __restrict__ r,
                   const double* __restrict__ invD, nk_cg_state* st,
                   double* __restrict__ partials, int64_t part_base, int64_t reduce_count,
                   double* __restrict__ hist, int pdl_flags, int l2_flags,
                   const __grid_constant__ GsTail tail) {
  tma_pcg_body<NQ, MINB, SB, false>(nlist, elist, D, G, p, w, lam0, B, lam1, mask, x, r, invD, st, partials, part_base, reduce_count, hist, pdl_flags, l2_flags, tail);
}

template <int NQ, int MINB, bool SB, bool TAIL = false>
static auto tma_pcg_kernel() {
  if constexpr (SB && MINB == 5 && !TAIL) return bk5_pencil_tma_pcg_nreg<NQ, MINB, SB, 200>;
  else return bk5_pencil_tma_pcg<NQ, MINB, SB, TAIL>;
}

template <int NQ, int MINB, bool SB = false, bool TAIL = false>
static int64_t tma_pcg_grid(int64_t nlist) {
  static int64_t resident = -1;
  if (resident < 0) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    using C = TmaPcgCfg<NQ, MINB, SB>;
    cudaFuncSetAttribute(tma_pcg_kernel<NQ, MINB, SB, TAIL>(),
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, tma_pcg_kernel<NQ, MINB, SB, TAIL>(), C::THREADS,
                                                  C::smem_bytes());
    resident = (int64_t)sms * (per > 0 ? per : 1);
  }
  return nlist < resident ? nlist : resident;
}

template <int NQ, int MINB, bool SB = false>
static int launch_pencil_tma_pcg(int64_t nlist, const int32_t* elist, const double* Dhost,
                                 const double* G, double* p, double* w, double lam0,
                                 const double* B, double lam1, const uint8_t* mask, double* x,
                                 const double* r, const double* invD, nk_cg_state* st,
                                 double* partials, int64_t part_base, int64_t reduce_count,
                                 double* hist, cudaStream_t s) {
  using C = TmaPcgCfg<NQ, MINB, SB>;
  const int64_t grid = tma_pcg_grid<NQ, MINB, SB>(nlist);
  if (grid == 0) return NK_OK;
  if ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(G)) & 15) {
    set_error("bk5_pencil_tma_pcg: p and G must be 16-byte aligned");
    return NK_ERR_INVALID;
  }
  DParam<NQ> D;
  D.set(Dhost);
  GsTail tail{};
  // the tail variant (its own instantiation: the plain step keeps its
  // register count) needs the same grid, all of it resident, for the barrier
  if (const GsTail* off = gs_tail_offer();
      off != nullptr && elist == nullptr && tma_pcg_grid<NQ, MINB, SB, true>(nlist) == grid) {
    tail = *off;
    gs_tail_mark_used();
    launch_ex(kPdlStep, tma_pcg_kernel<NQ, MINB, SB, true>(), dim3((unsigned)grid),
              dim3(C::THREADS), C::smem_bytes(), s, nlist, elist, D, G, p, w, lam0, B, lam1,
              mask, x, r, invD, st, partials, part_base, reduce_count, hist, knob(NK_KNOB_PDL),
              knob(NK_KNOB_L2), tail);
    return check_launch("bk5_pencil_tma_pcg(gs tail)");
  }
  launch_ex(kPdlStep, tma_pcg_kernel<NQ, MINB, SB>(), dim3((unsigned)grid), dim3(C::THREADS),
            C::smem_bytes(), s, nlist, elist, D, G, p, w, lam0, B, lam1, mask, x, r, invD, st,
            partials, part_base, reduce_count, hist, knob(NK_KNOB_PDL), knob(NK_KNOB_L2), tail);
  return check_launch("bk5_pencil_tma_pcg");
}

}  // namespace nk
