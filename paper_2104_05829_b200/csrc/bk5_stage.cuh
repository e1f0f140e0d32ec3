// BK5 variant 8, "stage": persistent CTAs whose element operands are staged
// in shared memory by the TMA engine (auto at N = 6, 8, 9, 10, 12, 13, 14;
// serves N + 1 = NQ in 3, 5..16).
//
// Why: ncu source-level stall sampling of the register-pencil kernels at
// N = 12 (bk5_pencil<13>) and N = 15 (bk5_pencil2<16>) puts 48-56% of the
// warp stalls on two phases that wait for L2: the u rows of F1 (long
// scoreboard 62%) and the 6 x NQ G loads per thread of the G phase (long
// scoreboard 35-52%, LSU throttle) -- with only 2 CTAs (12-16 warps) per SM
// nothing covers them, and a hot-L2 run (profiles/r2u_bk5_hot.jsonl) is no
// faster than a cold one: the limiter is L2 -> SM latency, not HBM.  Here a
// single thread moves the NEXT element's u and G into shared memory with
// cp.async.bulk (SASS UBLKCP, mbarrier transaction counts) while the CTA
// computes the current one, so every phase reads shared memory:
//
//   (start)      issue u(next) into the other u buffer (NUB = 2)
//   wait u_bar   F1 i-pencils  u row (shared)     -> ur -> R
//                F2 j-pencils  u column (shared)  -> us -> S
//                F3 k-pencils  u column (shared)  -> ut (registers)
//   sync (A)
//   wait g_bar   G  k-pencils  G (shared; components >= NGS from L2) -> gr, gs
//                   in place in R, S; gt (registers)
//   sync (B)     G buffer free: issue G(next)
//   B2 j-pencils S column  -> D^T gs in place      ; sync
//   B3 k-pencils S column += D^T gt                 ; sync
//   B1 i-pencils w = lam0 (D^T R row + S row) [+ lam1 B u, mask, u.w]
//                -> the element's spent u buffer
//   sync (C)     one bulk store (cp.async.bulk.global.shared) of w -> HBM (or,
//                through the UVA, pinned host memory: the e2e direct path)
//
// The contractions are the register pencils of bk5_pencil.cuh (even-odd D-hat
// in the constant bank, 12 shared accesses per point as in pencil2).  The
// u buffer is the element's dense HBM image (i fastest): conflict-free for
// the column passes and, for F1's rows, with 8-byte reads at odd NQ (row
// stride NQ odd) and 16-byte reads at even NQ (row stride NQ/2 chunks: 5 and
// 7 are conflict-free, 6 two-way).  At odd NQ an element starts 8 bytes off
// a 16-byte boundary every other element: the copy then starts one double
// early (the buffer pointer shifts by one); the array's very last double,
// when a copy would run past the allocation, is stored by a plain load.
// NGS of the six G components are staged (all six when the CTA fits); the
// rest are read from global memory after a bulk L2 prefetch issued one
// element ahead.  Below N = 7 a CTA runs EPB small elements side by side.
// Shapes and alternative modes (RINU, G4U, NUB = 1): StageShapes in
// bk5_inst.cu.  N = 15 (one u row = 128 B) is bk5_stage16 below, with
// tensor-map copies and the 128-byte swizzle.  HBM per point: u 8 + G 48 +
// w 8 B (the BK5 roofline).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include "bk5_tma.cuh"

namespace nk {

__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// NUB = 2: two u buffers -- u(next) is issued at the START of the current
// element (one whole element of lead time), and the current element's w is
// assembled in its own u buffer after B1 and written back by one bulk store
// (cp.async.bulk.global.shared, SASS UBLKCP) instead of 13-16 strided 8-byte
// stores per thread.  NUB = 1: one u buffer, refilled after F3.
// RINU (odd NQ, NUB = 2): R lives in the current u buffer -- u is dead once
// F1..F3 have read it, so ur is written there after one extra barrier (the
// dense odd-NQ u image IS the pencil layout).  Saves one element buffer,
// which buys a fifth staged G component at NQ = 15.
// EPB: elements per CTA (low orders: EPB small elements side by side, each
// with its own buffers and NQ^2 threads; one barrier sequence per group).
// Shared layout of R and S in the stage kernels: the pencil layout, except at
// NQ = 12 where the padded row stride 13 puts two-way conflicts on every
// k-pencil access (the G phase and B3: 72 of the thread's 144 element-buffer
// accesses): dense rows (R = 12) and plane stride 156 (= 12 mod 16) make the
// k-pencil and j-column orientations conflict-free, and the i-rows -- read
// and written with 16-byte accesses (ROW16) -- two-way.
template <int NQ> struct StageLayout : PencilLayout<NQ> {
  static constexpr bool ROW16 = false;
};
template <> struct StageLayout<12> {
  static constexpr int R = 12, P = 156, VOL = 12 * 156;
  static constexpr bool ROW16 = true;
  __device__ __forceinline__ static int idx(int k, int j, int i) { return k * P + j * R + i; }
};

// G4U (NUB = 2, EPB = 1, NGS <= 4): G component NGS of the CURRENT element is
// staged in the spare u buffer while F1..F3 run (issued at the element's
// start), and u(next) goes into that buffer after the G phase instead -- one
// more staged component (of the two that do not fit at NQ = 15) for half an
// element less of u lead time.
template <int NQ, int NGS, int NUB, bool RINU = false, int EPB = 1, bool G4U = false>
struct StageCfg {
  static_assert(NGS >= 1 && NGS <= 6, "NGS");
  static_assert(NUB == 1 || NUB == 2, "NUB");
  static_assert(!RINU || (NQ % 2 == 1 && NUB == 2), "R in the u buffer: odd NQ, two u buffers");
  static_assert(!G4U || (NUB == 2 && EPB == 1 && !RINU && NGS <= 4), "G4U");
  static constexpr int NQ2 = NQ * NQ, NQ3 = NQ2 * NQ;
  static constexpr int VOL = StageLayout<NQ>::VOL;
  static constexpr int UB = (NQ3 + 2 + 1) & ~1;         // doubles, even: 16-B aligned next
  static constexpr int GBUF = (NGS * NQ3 + 1 + 1) & ~1;
  static constexpr int THREADS = EPB * NQ2;
  // layout (doubles): U[NUB][EPB] | G[EPB] | R[EPB] | S[EPB] | red[32] ; mbarriers u[NUB], g
  static size_t smem_bytes() {
    return sizeof(double) * ((size_t)EPB * (NUB * UB + GBUF + (RINU ? 1 : 2) * VOL) + 32) +
           (NUB + 2) * sizeof(uint64_t);
  }
};

// PCG (nk_bk5_pcg, the fused BP5 step; EPB = 1, two u buffers, R in its own
// buffer): u is the search direction p.  The element's x / r / invD columns
// are read in the F3 pass (k-pencils: this thread's own column of the staged
// p image, coalesced planes) and the Jacobi-PCG head is applied there --
// deferred x += alpha p, p = invD r + beta p, written to global memory and
// back into the staged image -- before F1 / F2 read it (one extra barrier);
// the stop test and the last-block bookkeeping follow bk5_pencil_tma_pcg.
// Same per-point arithmetic and the same p.Ap partial grouping as the split
// step (nk_cg_xpstep + this kernel's fused dot): bit-identical solves.
// Chunk-gated input (nk_bk5_set_gate; the host-buffer e2e stream): u arrives
// in element order by copy-engine chunks, each followed by a copy of the
// element count it completes into *gate; thread 0 waits until the elements
// a u copy covers are in before issuing it.  Bounded spin (~2 s) so a
// missing gate write cannot hang the device.
__device__ __forceinline__ void gate_wait(const unsigned long long* gate, int64_t need) {
  const long long t0 = clock64();
  unsigned ns = 256;
  for (;;) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(gate) : "memory");
    if ((int64_t)v >= need) break;
    if (clock64() - t0 > 4000000000LL) break;
    __nanosleep(ns);   // hundreds of CTAs poll one line: back off (chunks are ~10s of us apart)
    if (ns < 4096) ns <<= 1;
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ bool gate_ready(const unsigned long long* gate, int64_t need) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(gate) : "memory");
  return (int64_t)v >= need;
}

template <int NQ, int NGS, int NUB, int MINB, bool RINU = false, int EPB = 1,
          bool G4U = false, bool PCG = false>
__global__ void __launch_bounds__(EPB * NQ * NQ, MINB)
bk5_stage(int64_t nlist, const int32_t* __restrict__ elist, const __grid_constant__ DParam<NQ> D,
          const double* __restrict__ G, const double* __restrict__ u, double* __restrict__ w,
          double lam0, const double* __restrict__ B, double lam1,
          const uint8_t* __restrict__ mask, nk_cg_state* st, double* __restrict__ partials,
          int64_t part_base, int64_t reduce_count, int64_t u_len, double* __restrict__ x = nullptr,
          const double* __restrict__ r = nullptr, const double* __restrict__ invD = nullptr,
          double* __restrict__ hist = nullptr, const unsigned long long* gate = nullptr) {
  using L = StageLayout<NQ>;
  using C = StageCfg<NQ, NGS, NUB, RINU, EPB, G4U>;
  static_assert(!PCG || (EPB == 1 && NUB == 2 && !RINU && !G4U), "PCG: EPB 1, two u buffers");
  constexpr int NQ2 = C::NQ2, NQ3 = C::NQ3, VOL = C::VOL;
  extern __shared__ __align__(128) double smem[];
  if (st != nullptr && st->done) return;
  // PCG: the iteration's scalars (bk5_pencil_tma_pcg)
  int cgit = 0;
  bool conv = false, stop = false;
  double alpha_prev = 0.0, beta = 0.0;
  if constexpr (PCG) {
    cgit = st->iter;
    conv = cgit > 0 && st->rr <= st->thresh2;
    stop = cgit > 0 && (conv || cgit >= st->max_iter);
    alpha_prev = st->alpha;
    const double rz = st->rz;
    beta = cgit == 0 ? 0.0 : (st->flexible ? (-alpha_prev * st->zap) / rz : st->rz_new / rz);
  }
  const int t = threadIdx.x;
  const int le = EPB == 1 ? 0 : t / NQ2;       // this thread's element of the group
  const int tt = t - le * NQ2;
  const int a = tt % NQ, b = tt / NQ;
  double* Ub0 = smem;                          // [NUB][EPB][UB]
  double* Gb0 = Ub0 + NUB * EPB * C::UB;       // [EPB][GBUF]
  double* Gb = Gb0 + le * C::GBUF;
  double* Rfix = Gb0 + EPB * C::GBUF + le * VOL;        // (RINU: unused)
  double* Ss = Gb0 + EPB * C::GBUF + (RINU ? 0 : EPB * VOL) + le * VOL;
  double* red = Gb0 + EPB * C::GBUF + (RINU ? 1 : 2) * EPB * VOL;
  uint64_t* ubar = reinterpret_cast<uint64_t*>(red + 32);   // [NUB]
  uint64_t* gbar = ubar + NUB;
  uint64_t* g4bar = gbar + 1;   // (G4U)
  const int64_t stride = gridDim.x;
  const int64_t ngroups = (nlist + EPB - 1) / EPB;
  // w assembled in shared memory and bulk-stored: needs u and w at the same
  // 16-byte phase (then the staged u row and the w row align alike)
  const bool bulkw = NUB == 2 &&
      ((reinterpret_cast<uintptr_t>(u) ^ reinterpret_cast<uintptr_t>(w)) & 15) == 0;
  auto elem_of = [&](int64_t slot) -> int64_t { return elist ? (int64_t)elist[slot] : slot; };
  auto phase_of = [&](int64_t e) -> int {   // 1: the element starts 8 B off 16 B
    return (int)((reinterpret_cast<uintptr_t>(u + e * NQ3) >> 3) & 1);
  };

  // thread 0 only: one mbarrier transaction for the group's EPB copies
  auto u_copy = [&](int64_t s0, int64_t& cnt, int& sh) -> bool {   // -> tail
    sh = phase_of(s0 / NQ3);                              // 8 B off a 16-B boundary
    cnt = (NQ3 + sh + 1) & ~int64_t(1);                   // whole 16-B chunks
    const bool tail = s0 - sh + cnt > u_len;              // would pass the array end
    if (tail) cnt -= 2;
    return tail;
  };
  auto gate_need = [&](int64_t grp) -> int64_t {   // elements group grp's copy covers
    return (grp + 1) * EPB < nlist ? (grp + 1) * EPB : nlist;
  };
  bool upend = false;   // (thread 0, gated input) this group's u is not issued yet
  auto issue_u = [&](int64_t grp, int bi) {
    if (gate != nullptr) gate_wait(gate, gate_need(grp));
    int64_t tot = 0;
    for (int l = 0; l < EPB; ++l) {
      if (grp * EPB + l >= nlist) break;
      int64_t cnt;
      int sh;
      u_copy(elem_of(grp * EPB + l) * NQ3, cnt, sh);
      tot += cnt;
    }
    mbar_expect_tx(&ubar[bi], (uint32_t)(tot * sizeof(double)));
    for (int l = 0; l < EPB; ++l) {
      if (grp * EPB + l >= nlist) break;
      const int64_t s0 = elem_of(grp * EPB + l) * NQ3;
      int64_t cnt;
      int sh;
      const bool tail = u_copy(s0, cnt, sh);
      double* dst = Ub0 + (bi * EPB + l) * C::UB;
      tma_load_1d(dst, u + s0 - sh, (uint32_t)(cnt * sizeof(double)), &ubar[bi]);
      if (PCG && cgit > 0) {   // the PCG head's columns: towards L2 one element ahead
        prefetch_l2(x + s0 - sh, cnt * (int64_t)sizeof(double));
        prefetch_l2(r + s0 - sh, cnt * (int64_t)sizeof(double));
        prefetch_l2(invD + s0 - sh, cnt * (int64_t)sizeof(double));
      }
      if (tail) {                                         // the one uncovered double
        dst[cnt] = u[s0 - sh + cnt];
        fence_proxy_async();                              // before later bulk writes
      }
    }
  };
  auto issue_g = [&](int64_t grp) {
    constexpr uint32_t GBYTES = (uint32_t)(((NGS * NQ3 + 1) & ~1) * sizeof(double));
    int nv = 0;
    for (int l = 0; l < EPB; ++l) nv += grp * EPB + l < nlist ? 1 : 0;
    mbar_expect_tx(gbar, nv * GBYTES);
    for (int l = 0; l < nv; ++l) {
      const double* src = G + elem_of(grp * EPB + l) * 6 * NQ3;   // always 16-B aligned
      tma_load_1d(Gb0 + l * C::GBUF, src, GBYTES, gbar);
      if (NGS < 6) prefetch_l2(src + NGS * NQ3, (int64_t)(6 - NGS) * NQ3 * sizeof(double));
    }
  };

  // (G4U) component NGS of element e into u buffer bi: 16-B rounded like u
  auto g4_shift = [&](int64_t e) -> int {
    return (int)((reinterpret_cast<uintptr_t>(G + (e * 6 + NGS) * NQ3) >> 3) & 1);
  };
  auto issue_g4 = [&](int64_t e, int bi) {
    const int s4 = g4_shift(e);
    const int64_t cnt = (NQ3 + s4 + 1) & ~int64_t(1);   // stays inside component NGS + 1
    mbar_expect_tx(g4bar, (uint32_t)(cnt * sizeof(double)));
    tma_load_1d(Ub0 + bi * C::UB, G + (e * 6 + NGS) * NQ3 - s4, (uint32_t)(cnt * sizeof(double)),
                g4bar);
  };
  double dot = 0.0;
  if (PCG && stop) {   // the final deferred x update only
    for (int64_t slot = blockIdx.x; slot < ngroups; slot += stride) {
      const int64_t e = elem_of(slot);
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        const int64_t q = e * NQ3 + k * NQ2 + tt;
        x[q] = fma(alpha_prev, u[q], x[q]);
      }
    }
  }
  if (t == 0) {
    for (int i = 0; i < NUB; ++i) mbar_init(&ubar[i], 1);
    mbar_init(gbar, 1);
    if (G4U) mbar_init(g4bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t == 0 && (int64_t)blockIdx.x < ngroups && !(PCG && stop)) {
    issue_u(blockIdx.x, 0);
    issue_g(blockIdx.x);
  }
  __syncthreads();   // the tail store (if any) before the first F1

  int it = 0;
  for (int64_t slot = blockIdx.x; slot < ((PCG && stop) ? 0 : ngroups); slot += stride, ++it) {
    const bool act = EPB == 1 || slot * EPB + le < nlist;
    const int64_t e = act ? elem_of(slot * EPB + le) : 0;
    const int sh = phase_of(e);
    const int bi = NUB == 2 ? (it & 1) : 0;
    double* uS = Ub0 + (bi * EPB + le) * C::UB + sh;
    double* Rr = RINU ? uS : Rfix;
    if (G4U && t == 0) {   // this element's component NGS into the spare u buffer
      bulk_wait_read0();
      issue_g4(e, bi ^ 1);
    } else if (NUB == 2 && t == 0) {
      if (upend) {   // gated: this group's u was not in yet one group ago
        issue_u(slot, bi);
        upend = false;
      }
      if (slot + stride < ngroups) {
        bulk_wait_read0();           // the other buffer's w (previous group) has left
        // gated input: never block the current group on the next one's chunk
        if (gate == nullptr || gate_ready(gate, gate_need(slot + stride)))
          issue_u(slot + stride, bi ^ 1);
        else
          upend = true;
      }
    }
    mbar_wait(&ubar[bi], NUB == 2 ? ((it >> 1) & 1) : (it & 1));
    double ut[NQ], o1[NQ];
    if constexpr (PCG) {   // ---- F3 + the PCG head on this thread's k-column
      double v[NQ];
      const int64_t q0 = e * NQ3 + b * NQ + a;
      if (cgit > 0) {
        double xv[NQ], rv[NQ], dv[NQ];
#pragma unroll
        for (int m = 0; m < NQ; ++m) {
          xv[m] = x[q0 + m * NQ2];
          rv[m] = __ldg(r + q0 + m * NQ2);
          dv[m] = __ldg(invD + q0 + m * NQ2);
        }
#pragma unroll
        for (int m = 0; m < NQ; ++m) {
          const double pv = uS[m * NQ2 + b * NQ + a];
          x[q0 + m * NQ2] = fma(alpha_prev, pv, xv[m]);
          v[m] = fma(beta, pv, dv[m] * rv[m]);
          uS[m * NQ2 + b * NQ + a] = v[m];
          const_cast<double*>(u)[q0 + m * NQ2] = v[m];
        }
      } else {
#pragma unroll
        for (int m = 0; m < NQ; ++m) v[m] = uS[m * NQ2 + b * NQ + a];
      }
      matvec<NQ, false>(D, v, ut);
      __syncthreads();   // (P) the updated p image before F1 / F2
    }
    if (act) {  // ---- F1: i-pencils (j = a, k = b) -> R (RINU: o1, written after (A))
      double v[NQ], o[NQ];
      const double* row = uS + b * NQ2 + a * NQ;
      if (NQ % 2 == 0 && sh == 0) {   // 16-byte rows (sh = 1 only for a misaligned u slice)
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
      if (RINU) {
        matvec<NQ, false>(D, v, o1);
      } else {
        matvec<NQ, false>(D, v, o);
        if (L::ROW16) {
#pragma unroll
          for (int i = 0; i < NQ; i += 2)
            *reinterpret_cast<double2*>(Rr + L::idx(b, a, i)) = make_double2(o[i], o[i + 1]);
        } else {
#pragma unroll
          for (int i = 0; i < NQ; ++i) Rr[L::idx(b, a, i)] = o[i];
        }
      }
      // ---- F2: j-pencils (i = a, k = b) -> S
#pragma unroll
      for (int m = 0; m < NQ; ++m) v[m] = uS[b * NQ2 + m * NQ + a];
      matvec<NQ, false>(D, v, o);
#pragma unroll
      for (int j = 0; j < NQ; ++j) Ss[L::idx(b, j, a)] = o[j];
      if constexpr (!PCG) {   // ---- F3: k-pencils (i = a, j = b) -> ut
#pragma unroll
        for (int m = 0; m < NQ; ++m) v[m] = uS[m * NQ2 + b * NQ + a];
        matvec<NQ, false>(D, v, ut);
      }
    }
    __syncthreads();   // (A)
    if (NUB == 1 && t == 0 && slot + stride < ngroups) issue_u(slot + stride, 0);
    if (RINU) {   // every u read is done: the buffer becomes R
      if (act) {
#pragma unroll
        for (int i = 0; i < NQ; ++i) Rr[L::idx(b, a, i)] = o1[i];
      }
      __syncthreads();   // (A2)
    }
    mbar_wait(gbar, it & 1);
    if (G4U) mbar_wait(g4bar, it & 1);
    const double* g4s = G4U ? Ub0 + (bi ^ 1) * C::UB + g4_shift(e) : nullptr;
    double gt[NQ];
    if (act) {  // ---- G: k-pencils, pointwise symmetric 3x3
      const double* gp = G + e * 6 * NQ3 + b * NQ + a;
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        const int p = k * NQ2 + b * NQ + a;
        double g[6];
#pragma unroll
        for (int c = 0; c < 6; ++c)
          g[c] = c < NGS ? Gb[c * NQ3 + p]
                         : ((G4U && c == NGS) ? g4s[p] : __ldg(gp + c * NQ3 + k * NQ2));
        const int q = L::idx(k, b, a);
        const double ur = Rr[q], us = Ss[q];
        Rr[q] = g[0] * ur + g[1] * us + g[2] * ut[k];
        Ss[q] = g[1] * ur + g[3] * us + g[4] * ut[k];
        gt[k] = g[2] * ur + g[4] * us + g[5] * ut[k];
      }
    }
    __syncthreads();   // (B) G buffer read for the last time
    if (t == 0 && slot + stride < ngroups) {
      issue_g(slot + stride);
      if (G4U) issue_u(slot + stride, bi ^ 1);   // component NGS has been read
    }
    if (act) {  // ---- B2: j-pencils, in place on their own S column
      double v[NQ], o[NQ];
#pragma unroll
      for (int m = 0; m < NQ; ++m) v[m] = Ss[L::idx(b, m, a)];
      matvec<NQ, true>(D, v, o);
#pragma unroll
      for (int j = 0; j < NQ; ++j) Ss[L::idx(b, j, a)] = o[j];
    }
    __syncthreads();
    if (act) {  // ---- B3: k-pencils, S column += D^T gt
      double o[NQ];
      matvec<NQ, true>(D, gt, o);
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        const int q = L::idx(k, b, a);
        Ss[q] = o[k] + Ss[q];
      }
    }
    __syncthreads();
    if (act) {  // ---- B1: i-pencils + epilogue
      double v[NQ], o[NQ];
      double sr[NQ];
      if (L::ROW16) {
#pragma unroll
        for (int m = 0; m < NQ; m += 2) {
          const double2 pr = *reinterpret_cast<const double2*>(Rr + L::idx(b, a, m));
          const double2 ps = *reinterpret_cast<const double2*>(Ss + L::idx(b, a, m));
          v[m] = pr.x;
          v[m + 1] = pr.y;
          sr[m] = ps.x;
          sr[m + 1] = ps.y;
        }
      } else {
#pragma unroll
        for (int m = 0; m < NQ; ++m) {
          v[m] = Rr[L::idx(b, a, m)];
          sr[m] = Ss[L::idx(b, a, m)];
        }
      }
      matvec<NQ, true>(D, v, o);
      const int64_t off = e * NQ3 + b * NQ2 + a * NQ;
      double res[NQ];
#pragma unroll
      for (int i = 0; i < NQ; ++i) res[i] = lam0 * (o[i] + sr[i]);
      double* urow = uS + b * NQ2 + a * NQ;   // NUB = 2: still this element's u
      if (B != nullptr || st != nullptr) {
        double urw[NQ];
#pragma unroll
        for (int i = 0; i < NQ; ++i) urw[i] = (NUB == 2 && !RINU) ? urow[i] : __ldg(u + off + i);
        if (B != nullptr) {
#pragma unroll
          for (int i = 0; i < NQ; ++i) res[i] = fma(lam1 * __ldg(B + off + i), urw[i], res[i]);
        }
        if (mask != nullptr) {
#pragma unroll
          for (int i = 0; i < NQ; ++i) res[i] = mask[off + i] ? res[i] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < NQ; ++i) dot = fma(urw[i], res[i], dot);
      } else if (mask != nullptr) {
#pragma unroll
        for (int i = 0; i < NQ; ++i) res[i] = mask[off + i] ? res[i] : 0.0;
      }
      if (bulkw) {
        // w row into the u row (this thread's own row); the element's two
        // edge doubles that fall outside the 16-byte bulk range go direct
        if (NQ % 2 == 0 && sh == 0) {   // 16-byte stores: even row strides conflict at 8 B
#pragma unroll
          for (int i = 0; i < NQ; i += 2)
            *reinterpret_cast<double2*>(urow + i) = make_double2(res[i], res[i + 1]);
        } else {
#pragma unroll
          for (int i = 0; i < NQ; ++i) urow[i] = res[i];
        }
        fence_proxy_async();
        if (tt == 0 && sh) w[e * NQ3] = res[0];
        if (tt == NQ2 - 1 && ((NQ3 - sh) & 1)) w[e * NQ3 + NQ3 - 1] = res[NQ - 1];
      } else {
        double* wr = w + off;
        if (NQ % 2 == 0 && sh == 0 &&
            ((reinterpret_cast<uintptr_t>(wr) & 15) == 0)) {
#pragma unroll
          for (int i = 0; i < NQ; i += 2)
            *reinterpret_cast<double2*>(wr + i) = make_double2(res[i], res[i + 1]);
        } else {
#pragma unroll
          for (int i = 0; i < NQ; ++i) wr[i] = res[i];
        }
      }
    }
    __syncthreads();   // (C) R, S free for the next element; w rows in shared
    if (bulkw && t == 0) {
      for (int l = 0; l < EPB; ++l) {
        if (slot * EPB + l >= nlist) break;
        const int64_t el = elem_of(slot * EPB + l);
        const int shl = phase_of(el);
        const int64_t cnt = (NQ3 - shl) & ~int64_t(1);
        bulk_store(w + el * NQ3 + shl, Ub0 + (bi * EPB + l) * C::UB + 2 * shl,
                   (uint32_t)(cnt * sizeof(double)));
      }
      bulk_commit();
    }
  }
  if (NUB == 2 && t == 0) bulk_wait0();   // shared source read and global writes done

  if (st != nullptr) {
    double vv[1] = {dot};
    block_sum<1>(vv, red);
    if (t == 0) partials[part_base + blockIdx.x] = vv[0];
    if (reduce_count > 0 && last_block(&st->ticket[0], gridDim.x)) {
      double sres[1];
      reduce_partials<1>(partials, reduce_count, 0, sres, red);
      if (t == 0) {
        if constexpr (PCG) {
          if (cgit > 0 && hist) hist[cgit] = sqrt(st->rr);
          if (stop) {
            st->converged = conv ? 1 : 0;
            st->done = 1;
          } else {
            st->pAp = sres[0];
            if (cgit > 0) st->rz = st->rz_new;
          }
        } else {
          st->pAp = sres[0];
        }
      }
    }
  }
}

// Grid: persistent, min(groups, SMs x resident CTAs per SM).
template <int NQ, int NGS, int NUB, int MINB, bool RINU = false, int EPB = 1, bool G4U = false>
static int64_t stage_grid(int64_t nlist) {
  static int64_t resident = -1;
  if (resident < 0) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    using C = StageCfg<NQ, NGS, NUB, RINU, EPB, G4U>;
    cudaFuncSetAttribute(bk5_stage<NQ, NGS, NUB, MINB, RINU, EPB, G4U>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per,
                                                  bk5_stage<NQ, NGS, NUB, MINB, RINU, EPB, G4U>,
                                                  C::THREADS, C::smem_bytes());
    resident = (int64_t)sms * (per > 0 ? per : 1);
  }
  const int64_t groups = (nlist + EPB - 1) / EPB;
  return groups < resident ? groups : resident;
}

// u_len: doubles in the u array (bounds the 16-byte rounded copies)
template <int NQ, int NGS, int NUB, int MINB, bool RINU = false, int EPB = 1, bool G4U = false>
static int launch_stage(int64_t nlist, const int32_t* elist, const double* Dhost, const double* G,
                        const double* u, double* w, double lam0, const double* B, double lam1,
                        const uint8_t* mask, nk_cg_state* st, double* partials,
                        int64_t part_base, int64_t reduce_count, int64_t u_len, cudaStream_t s) {
  using C = StageCfg<NQ, NGS, NUB, RINU, EPB, G4U>;
  const int64_t grid = stage_grid<NQ, NGS, NUB, MINB, RINU, EPB, G4U>(nlist);
  if (grid == 0) return NK_OK;
  if ((reinterpret_cast<uintptr_t>(u) & 7) || (reinterpret_cast<uintptr_t>(G) & 15)) {
    set_error("bk5_stage: u must be 8-byte and G 16-byte aligned");
    return NK_ERR_INVALID;
  }
  DParam<NQ> D;
  D.set(Dhost);
  const unsigned long long* gate = elist == nullptr ? bk5_gate() : nullptr;
  bk5_stage<NQ, NGS, NUB, MINB, RINU, EPB, G4U><<<(unsigned)grid, C::THREADS, C::smem_bytes(), s>>>(
      nlist, elist, D, G, u, w, lam0, B, lam1, mask, st, partials, part_base, reduce_count, u_len,
      nullptr, nullptr, nullptr, nullptr, gate);
  return check_launch("bk5_stage");
}

// The fused BP5 step on the stage kernel (PCG = true; nk_bk5_pcg at
// N + 1 in 9..15 without an element list).
template <int NQ, int NGS, int MINB>
static int64_t stage_pcg_grid(int64_t nlist) {
  static int64_t resident = -1;
  if (resident < 0) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    using C = StageCfg<NQ, NGS, 2>;
    auto kern = bk5_stage<NQ, NGS, 2, MINB, false, 1, false, true>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, C::THREADS, C::smem_bytes());
    resident = (int64_t)sms * (per > 0 ? per : 1);
  }
  return nlist < resident ? nlist : resident;
}

template <int NQ, int NGS, int MINB>
static int launch_stage_pcg(int64_t nlist, const double* Dhost, const double* G, double* p,
                            double* w, double lam0, const double* B, double lam1,
                            const uint8_t* mask, double* x, const double* r, const double* invD,
                            nk_cg_state* st, double* partials, int64_t part_base,
                            int64_t reduce_count, double* hist, cudaStream_t s) {
  using C = StageCfg<NQ, NGS, 2>;
  const int64_t grid = stage_pcg_grid<NQ, NGS, MINB>(nlist);
  if (grid == 0) return NK_OK;
  if ((reinterpret_cast<uintptr_t>(p) & 7) || (reinterpret_cast<uintptr_t>(G) & 15)) {
    set_error("bk5_stage (PCG): p must be 8-byte and G 16-byte aligned");
    return NK_ERR_INVALID;
  }
  DParam<NQ> D;
  D.set(Dhost);
  bk5_stage<NQ, NGS, 2, MINB, false, 1, false, true>
      <<<(unsigned)grid, C::THREADS, C::smem_bytes(), s>>>(
          nlist, nullptr, D, G, p, w, lam0, B, lam1, mask, st, partials, part_base, reduce_count,
          nlist * (int64_t)C::NQ3, x, r, invD, hist);
  return check_launch("bk5_stage_pcg");
}

#if defined(NK_BK5_NQ) && NK_BK5_NQ == 16   // one translation unit owns the N = 15 kernel
// ---------------------------------------------------------------------------
// N = 15 (NQ = 16): one u row is 128 B, so in the dense image every i-row
// starts on bank 0 and F1's row reads would conflict 8-way.  u is therefore
// moved by a 2-D tensor copy (cp.async.bulk.tensor, tensor map of rows of 16
// doubles, box 16 x 256 = one element) with the 128-byte swizzle: 16-byte
// chunk c of row r lands at chunk c ^ (r mod 8), which makes i-rows (16-byte
// accesses), j- and k-columns (8-byte accesses) all conflict-free.  Shared
// memory (227 KB) holds two u buffers (64 KB), S (32 KB) and four of the six
// G components (128 KB): R lives in the current u buffer (u is dead after
// F1-F3, so ur is written there after one extra barrier), and w is assembled
// there too and leaves by a tensor store with the same swizzle.  G
// components 4 and 5 come from global memory after an L2 prefetch one
// element ahead.
struct Stage16 {
  static constexpr int NQ = 16, NQ2 = 256, NQ3 = 4096, NGS = 4;
  static constexpr int THREADS = NQ2;
  // (bytes) align slack | U0 | U1 | G[NGS] | S | red[32] | 3 mbarriers
  static size_t smem_bytes() {
    return 1024 + sizeof(double) * ((size_t)2 * NQ3 + NGS * NQ3 + NQ3 + 32) + 3 * sizeof(uint64_t);
  }
  // swizzled element (row r = k*16 + j, column i) of a u / R / w buffer
  __device__ __forceinline__ static int sw(int r, int i) {
    return r * 16 + ((((i >> 1) ^ (r & 7))) << 1) + (i & 1);
  }
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int x, int y,
                                             const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(smem_u32(src))
               : "memory");
}

__global__ void __launch_bounds__(256, 1)
bk5_stage16(int64_t nlist, const int32_t* __restrict__ elist, const __grid_constant__ DParam<16> D,
            const __grid_constant__ CUtensorMap tmu, const __grid_constant__ CUtensorMap tmw,
            const double* __restrict__ G, const double* __restrict__ u, double* __restrict__ w,
            double lam0, const double* __restrict__ B, double lam1,
            const uint8_t* __restrict__ mask, nk_cg_state* st, double* __restrict__ partials,
            int64_t part_base, int64_t reduce_count) {
  using C = Stage16;
  using L = PencilLayout<16>;
  constexpr int NQ = 16, NQ2 = C::NQ2, NQ3 = C::NQ3, NGS = C::NGS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (st != nullptr && st->done) return;
  // 1024-B aligned (128-byte swizzle atoms), as an offset from smem_raw so
  // that the compiler keeps the shared address space (LDS / STS, not generic
  // LD / ST through the long scoreboard)
  double* Ub0 = reinterpret_cast<double*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  double* Gb = Ub0 + 2 * NQ3;
  double* Ss = Gb + NGS * NQ3;
  double* red = Ss + NQ3;
  uint64_t* ubar = reinterpret_cast<uint64_t*>(red + 32);   // [2]
  uint64_t* gbar = ubar + 2;

  const int t = threadIdx.x;
  const int a = t & 15, b = t >> 4;
  const int64_t stride = gridDim.x;
  auto elem_of = [&](int64_t slot) -> int64_t { return elist ? (int64_t)elist[slot] : slot; };
  auto issue_u = [&](int64_t slot, int bi) {
    mbar_expect_tx(&ubar[bi], NQ3 * sizeof(double));
    tma_load_2d(Ub0 + bi * NQ3, &tmu, 0, (int)(elem_of(slot) * NQ2), &ubar[bi]);
  };
  auto issue_g = [&](int64_t slot) {
    const double* src = G + elem_of(slot) * 6 * NQ3;
    mbar_expect_tx(gbar, NGS * NQ3 * sizeof(double));
    tma_load_1d(Gb, src, NGS * NQ3 * sizeof(double), gbar);
    prefetch_l2(src + NGS * NQ3, (int64_t)(6 - NGS) * NQ3 * sizeof(double));
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

  double dot = 0.0;
  int it = 0;
  for (int64_t slot = blockIdx.x; slot < nlist; slot += stride, ++it) {
    const int64_t e = elem_of(slot);
    const int bi = it & 1;
    double* Uc = Ub0 + bi * NQ3;
    if (t == 0 && slot + stride < nlist) {
      bulk_wait_read0();   // the other buffer's w (previous element) has left
      issue_u(slot + stride, bi ^ 1);
    }
    mbar_wait(&ubar[bi], (it >> 1) & 1);
    double ut[NQ], o1[NQ];
    {
      double v[NQ], o[NQ];
      // ---- F2: j-pencils (i = a, k = b) -> S
#pragma unroll
      for (int m = 0; m < NQ; ++m) v[m] = Uc[C::sw(b * 16 + m, a)];
      matvec<NQ, false>(D, v, o);
#pragma unroll
      for (int j = 0; j < NQ; ++j) Ss[L::idx(b, j, a)] = o[j];
      // ---- F3: k-pencils (i = a, j = b) -> ut
#pragma unroll
      for (int m = 0; m < NQ; ++m) v[m] = Uc[C::sw(m * 16 + b, a)];
      matvec<NQ, false>(D, v, ut);
      // ---- F1: i-pencils (j = a, k = b) -> o1 (to R = this u buffer after the barrier)
      const int r = b * 16 + a;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double2 p = *reinterpret_cast<const double2*>(Uc + r * 16 + ((c ^ (r & 7)) << 1));
        v[2 * c] = p.x;
        v[2 * c + 1] = p.y;
      }
      matvec<NQ, false>(D, v, o1);
    }
    __syncthreads();   // (A) every u read done: the buffer becomes R
    {
      const int r = b * 16 + a;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<double2*>(Uc + r * 16 + ((c ^ (r & 7)) << 1)) =
            make_double2(o1[2 * c], o1[2 * c + 1]);
    }
    __syncthreads();   // (A2)
    mbar_wait(gbar, it & 1);
    double gt[NQ];
    {  // ---- G: k-pencils (i = a, j = b)
      const double* gp = G + e * 6 * NQ3 + b * NQ + a;
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        const int p = k * NQ2 + b * NQ + a;
        double g[6];
#pragma unroll
        for (int c = 0; c < 6; ++c)
          g[c] = c < NGS ? Gb[c * NQ3 + p] : __ldg(gp + c * NQ3 + k * NQ2);
        const int qr = C::sw(k * 16 + b, a), qs = L::idx(k, b, a);
        const double ur = Uc[qr], us = Ss[qs];
        Uc[qr] = g[0] * ur + g[1] * us + g[2] * ut[k];
        Ss[qs] = g[1] * ur + g[3] * us + g[4] * ut[k];
        gt[k] = g[2] * ur + g[4] * us + g[5] * ut[k];
      }
    }
    __syncthreads();   // (B) G buffer read for the last time
    if (t == 0 && slot + stride < nlist) issue_g(slot + stride);
    {  // ---- B2: j-pencils, in place on their own S column
      double v[NQ], o[NQ];
#pragma unroll
      for (int m = 0; m < NQ; ++m) v[m] = Ss[L::idx(b, m, a)];
      matvec<NQ, true>(D, v, o);
#pragma unroll
      for (int j = 0; j < NQ; ++j) Ss[L::idx(b, j, a)] = o[j];
    }
    __syncthreads();
    {  // ---- B3: k-pencils, S column += D^T gt
      double o[NQ];
      matvec<NQ, true>(D, gt, o);
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        const int q = L::idx(k, b, a);
        Ss[q] = o[k] + Ss[q];
      }
    }
    __syncthreads();
    {  // ---- B1: i-pencils (j = a, k = b) + epilogue; w row back into R's row
      const int r = b * 16 + a;
      double v[NQ], o[NQ];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double2 p = *reinterpret_cast<const double2*>(Uc + r * 16 + ((c ^ (r & 7)) << 1));
        v[2 * c] = p.x;
        v[2 * c + 1] = p.y;
      }
      matvec<NQ, true>(D, v, o);
      const int64_t off = e * NQ3 + b * NQ2 + a * NQ;
      double res[NQ];
#pragma unroll
      for (int i = 0; i < NQ; ++i) res[i] = lam0 * (o[i] + Ss[L::idx(b, a, i)]);
      if (B != nullptr || st != nullptr) {
        double urw[NQ];   // u row from L2 (its buffer now holds R)
#pragma unroll
        for (int i = 0; i < NQ; i += 2) {
          const double2 p = __ldg(reinterpret_cast<const double2*>(u + off + i));
          urw[i] = p.x;
          urw[i + 1] = p.y;
        }
        if (B != nullptr) {
#pragma unroll
          for (int i = 0; i < NQ; ++i) res[i] = fma(lam1 * __ldg(B + off + i), urw[i], res[i]);
        }
        if (mask != nullptr) {
#pragma unroll
          for (int i = 0; i < NQ; ++i) res[i] = mask[off + i] ? res[i] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < NQ; ++i) dot = fma(urw[i], res[i], dot);
      } else if (mask != nullptr) {
#pragma unroll
        for (int i = 0; i < NQ; ++i) res[i] = mask[off + i] ? res[i] : 0.0;
      }
#pragma unroll
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<double2*>(Uc + r * 16 + ((c ^ (r & 7)) << 1)) =
            make_double2(res[2 * c], res[2 * c + 1]);
      fence_proxy_async();
    }
    __syncthreads();   // (C) S free for the next element; w rows in shared
    if (t == 0) {
      tma_store_2d(&tmw, 0, (int)(e * NQ2), Uc);
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

// 2-D tensor map over an array of rows of 16 doubles (128 B), box 16 x 256
// (one N = 15 element), 128-byte swizzle.  cuTensorMapEncodeTiled is fetched
// through the runtime's driver entry point (no link against libcuda).
inline int encode_rows16(CUtensorMap* map, const double* base, int64_t ndoubles,
                         unsigned box_rows = 256) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (enc == nullptr) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc),
                                cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || enc == nullptr) {
      enc = nullptr;
      set_error("bk5_stage16: cuTensorMapEncodeTiled unavailable");
      return NK_ERR_CUDA;
    }
  }
  cuuint64_t dims[2] = {16, (cuuint64_t)(ndoubles / 16)};
  cuuint64_t strides[1] = {16 * sizeof(double)};
  cuuint32_t box[2] = {16, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("bk5_stage16: tensor map encode failed (%d)", (int)r);
    return NK_ERR_CUDA;
  }
  return NK_OK;
}

inline int64_t stage16_grid(int64_t nlist) {
  static int64_t resident = -1;
  if (resident < 0) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(bk5_stage16, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Stage16::smem_bytes());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bk5_stage16, Stage16::THREADS,
                                                  Stage16::smem_bytes());
    resident = (int64_t)sms * (per > 0 ? per : 1);
  }
  return nlist < resident ? nlist : resident;
}

// u and w must be 16-byte aligned (tensor maps); u_len doubles in u and w.
inline int launch_stage16(int64_t nlist, const int32_t* elist, const double* Dhost,
                          const double* G, const double* u, double* w, double lam0,
                          const double* B, double lam1, const uint8_t* mask, nk_cg_state* st,
                          double* partials, int64_t part_base, int64_t reduce_count,
                          int64_t u_len, cudaStream_t s) {
  const int64_t grid = stage16_grid(nlist);
  if (grid == 0) return NK_OK;
  if (((reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(w) |
        reinterpret_cast<uintptr_t>(G)) & 15) || (u_len % 16) != 0) {
    set_error("bk5_stage (N = 15): u, w and G must be 16-byte aligned");
    return NK_ERR_INVALID;
  }
  CUtensorMap tmu, tmw;
  int rc = encode_rows16(&tmu, u, u_len);
  if (rc == NK_OK) rc = encode_rows16(&tmw, w, u_len);
  if (rc != NK_OK) return rc;
  DParam<16> D;
  D.set(Dhost);
  bk5_stage16<<<(unsigned)grid, Stage16::THREADS, Stage16::smem_bytes(), s>>>(
      nlist, elist, D, tmu, tmw, G, u, w, lam0, B, lam1, mask, st, partials, part_base,
      reduce_count);
  return check_launch("bk5_stage16");
}

#endif  // NK_BK5_NQ == 16

}  // namespace nk
