// BK5 variant 3, "pencil": every contraction is a register-resident 1-D
// matrix-vector product with D-hat as a compile-time-indexed kernel parameter.
//
//   w_e = lam0 * sum_{m,m'} D_m^T G_mm' D_m' u_e + lam1 * B_e u_e
//
//
// Why: the k-slab kernel reads D and the neighbour values from shared memory
// for every FMA (~3.4 smem wavefronts per point), which caps it below the HBM
// roofline on B200.  Here a thread owns a whole 1-D line ("pencil") of NQ
// points along one axis, so a contraction along that axis is NQ^2 DFMAs with
// both operands in registers -- D enters as a __grid_constant__ parameter, so
// each DFMA reads it straight from the constant bank.  Changing axis is a
// transpose through shared memory (each value written once, read once), in a
// layout that is bank-conflict free for all three pencil orientations
// (NQ = 8: row stride 8, plane stride 72, i XOR-swizzled by (j>>1 | (k&1)<<2)).
//
// Per element (NQ^2 threads, one per pencil; t = a + NQ*b):
//   F1  i-pencils (j=a,k=b): u row from HBM -> ur = D u        ; U <- u, R <- ur
//   F2  j-pencils (i=a,k=b): v = U[k][:][i]  -> us = D v        ; S <- us
//   F3  k-pencils (i=a,j=b): v = U[:][j][i]  -> ut = D v (regs)
//   G   k-pencils: G from HBM, R,S,ut -> gr,gs (R,S in place), gt (regs)
//   B3  k-pencils: wt = D^T gt                                  ; U <- wt
//   B2  j-pencils: ws = D^T S[k][:][i] + U[k][:][i]              ; U <- ws+wt
//   B1  i-pencils: w  = D^T R[k][j][:] + U[k][j][:]  -> epilogue -> HBM
// Shared traffic: 15 accesses of 8 B per point; HBM: u 8 + G 48 + w 8 B.
#pragma once
#include "bk5_kernels.cuh"

namespace nk {

// Shared layout of one element buffer: idx(k,j,i) = k*P + j*R + i', with
// i' = i ^ ((j>>1) | (k&1)<<2) at NQ = 8 (conflict-free for all three pencil
// orientations) and i' = (i + C2*k) mod NQ otherwise.  (R, P, C2) per order
// come from scripts/smem_layout_search.py: minimum modeled shared wavefronts
// (half-warp, 8-byte banks) over the i-, j- and k-pencil accesses without
// growing the buffer.
template <int NQ> struct PencilPad { static constexpr int R = (NQ % 2 == 0) ? NQ + 1 : NQ,
  P = NQ * R + ((NQ * R) % 2 == 0 ? 1 : 0), C2 = 0; };
template <> struct PencilPad<2> { static constexpr int R = 2, P = 6, C2 = 1; };
template <> struct PencilPad<4> { static constexpr int R = 4, P = 20, C2 = 1; };
template <> struct PencilPad<6> { static constexpr int R = 6, P = 38, C2 = 3; };
template <> struct PencilPad<8> { static constexpr int R = 8, P = 72, C2 = 0; };
template <> struct PencilPad<10> { static constexpr int R = 10, P = 101, C2 = 0; };
template <> struct PencilPad<12> { static constexpr int R = 13, P = 156, C2 = 0; };
template <> struct PencilPad<14> { static constexpr int R = 14, P = 197, C2 = 0; };
template <> struct PencilPad<16> { static constexpr int R = 16, P = 256, C2 = 0; };

template <int NQ>
struct PencilLayout {
  static constexpr int R = PencilPad<NQ>::R;
  static constexpr int P = PencilPad<NQ>::P;
  static constexpr int C2 = PencilPad<NQ>::C2;
  static constexpr int VOL = NQ * P;
  __device__ __forceinline__ static int idx(int k, int j, int i) {
    if (NQ == 8) return k * P + j * R + (i ^ ((j >> 1) | ((k & 1) << 2)));
    if (NQ == 16) return k * P + j * R + (i ^ j);   // conflict-free, no padding
    if (C2 != 0) return k * P + j * R + ((i + C2 * k) % NQ);
    return k * P + j * R + i;
  }
};

template <int NQ, int EPB_, int MINB_>
struct PencilCfg {
  static constexpr int NQ2 = NQ * NQ, NQ3 = NQ * NQ * NQ;
  static constexpr int EPB = EPB_;
  static constexpr int THREADS = EPB * NQ2;
  static constexpr int MINB = MINB_;
  static constexpr int VOL = PencilLayout<NQ>::VOL;
  static size_t smem_bytes() { return sizeof(double) * ((size_t)EPB * 3 * VOL + 32); }
};

// out[q] = sum_m D[q][m] v[m]   (TRANS: sum_m D[m][q] v[m]), by the
// even-odd split of D-hat (DParam): ~NQ^2/2 multiply-adds instead of NQ^2.
template <int NQ, bool TRANS>
__device__ __forceinline__ void matvec(const DParam<NQ>& D, const double (&v)[NQ],
                                       double (&out)[NQ]) {
  constexpr int H = NQ / 2, ODD = NQ & 1, HE = H + ODD;
  constexpr int OFF = TRANS ? DParam<NQ>::EOF_ : 0;
  double s[H > 0 ? H : 1], d[H > 0 ? H : 1];
#pragma unroll
  for (int m = 0; m < H; ++m) {
    s[m] = v[m] + v[NQ - 1 - m];
    d[m] = v[m] - v[NQ - 1 - m];
  }
#pragma unroll
  for (int q = 0; q < H; ++q) {
    double e = 0.0, o = 0.0;
#pragma unroll
    for (int m = 0; m < H; ++m) {
      e = fma(D.eo[OFF + DParam<NQ>::ei(q, m)], s[m], e);
      o = fma(D.eo[OFF + DParam<NQ>::oi(q, m)], d[m], o);
    }
    if (ODD) e = fma(D.eo[OFF + DParam<NQ>::ei(q, H)], v[H], e);
    out[q] = o + e;
    out[NQ - 1 - q] = o - e;
  }
  if (ODD) {
    double mm = 0.0;
#pragma unroll
    for (int m = 0; m < H; ++m) mm = fma(D.eo[OFF + DParam<NQ>::mi(m)], d[m], mm);
    out[H] = mm;
  }
}

// NC = 3: the three velocity components of one element run back to back in
// the same CTA (vector Helmholtz): G is fetched from HBM once
// (L2 prefetch at CTA start) and re-read from L2 by components 1 and 2, so HBM
// moves 104 B per point for three components instead of 3 x 72, while the
// register and shared footprint stays that of the scalar kernel.
template <int NQ, int EPB, int MINB, int NC = 1, bool CDOT = false, bool LOOP = false>
__global__ void __launch_bounds__(EPB * NQ * NQ, MINB)
bk5_pencil(int64_t nlist, const int32_t* __restrict__ elist, const __grid_constant__ DParam<NQ> D,
           const double* __restrict__ G, const double* __restrict__ u_, double* __restrict__ w_,
           double lam0, const double* __restrict__ B, double lam1,
           const uint8_t* __restrict__ mask, nk_cg_state* st, double* __restrict__ partials,
           int64_t part_base, int64_t reduce_count, int pfG, int64_t pf_ahead,
           int64_t cstride = 0, int64_t pstride = 0) {
  // NC = 3, CDOT (the batched 3-component PCG, nk_bk5_batch): st points to
  // three CG states; component c's p.Ap partials go to partials + c *
  // pstride and its sum to st[c].pAp; a component whose state is done is
  // skipped (its p no longer changes).
  static_assert(NC == 1 || NC == 3, "NC");
  using L = PencilLayout<NQ>;
  constexpr int NQ2 = NQ * NQ, NQ3 = NQ2 * NQ, VOL = L::VOL;
  extern __shared__ double smem[];
  const int t = threadIdx.x;
  const int le = t / NQ2;
  const int tt = t - le * NQ2;
  const int a = tt % NQ, b = tt / NQ;
  double* red = smem;
  double* U = smem + 32 * NC + (size_t)le * 3 * VOL;
  double* Rr = U + VOL;
  double* Ss = Rr + VOL;

  // LOOP (fused-dot launches at NQ <= 8, launcher): a capped, grid-stride
  // grid -- one partial per resident CTA instead of one per element group,
  // so the last-block ticket and the partial list stay short (thousands of
  // same-address atomics cost ~3 ns each, profiles/r2zf_bk5_dot_cost.jsonl).
  // Without LOOP the loop below runs exactly once (and compiles away: a
  // real loop lets ptxas hoist D-hat's constant-bank operands out of it and
  // spill at NQ >= 12).
  const int64_t nblk = (nlist + EPB - 1) / EPB;
  const int64_t slot0 = (int64_t)blockIdx.x * EPB + le;
  const bool active0 = slot0 < nlist;
  const int64_t e0 = active0 ? (elist ? (int64_t)elist[slot0] : slot0) : 0;
  // PDL prologue (static operands only; L2 prefetches cannot go stale):
  // start this element's G (75% of its bytes) streaming into L2 now, so the
  // G-phase loads after F1-F3 hit L2 instead of waiting on HBM.  The done
  // read is a racy hint that skips it for the no-op iterations after
  // convergence.
  bool live = true;
  if ((NC == 1 || CDOT) && st != nullptr) {
    live = false;
#pragma unroll
    for (int c = 0; c < NC; ++c)
      live = live || *reinterpret_cast<volatile const int*>(&st[c].done) == 0;
  }
  if (live && pfG && active0 && tt == 0)
    prefetch_l2(G + e0 * 6 * NQ3, 6 * NQ3 * (int64_t)sizeof(double));
  // optionally also the element one resident wave ahead
  if (live && pf_ahead > 0 && tt == 0 && slot0 + pf_ahead < nlist) {
    const int64_t ea = elist ? (int64_t)elist[slot0 + pf_ahead] : slot0 + pf_ahead;
    prefetch_l2(G + ea * 6 * NQ3, 6 * NQ3 * (int64_t)sizeof(double));
  }
  pdl_wait();
  pdl_trigger();
  if ((NC == 1 || CDOT) && st != nullptr) {
    bool all_done = true;
#pragma unroll
    for (int c = 0; c < NC; ++c) all_done = all_done && st[c].done;
    if (all_done) return;
  }

  double dot = 0.0;
  int once = 0;   // LOOP = false: exactly one trip, provable at compile time
  for (int64_t blk = blockIdx.x; LOOP ? blk < nblk : once < 1; blk += gridDim.x, ++once) {
  const int64_t slot = blk * EPB + le;
  const bool active = slot < nlist;
  const int64_t e = active ? (elist ? (int64_t)elist[slot] : slot) : 0;
  if (LOOP && blk != blockIdx.x) {
    __syncthreads();   // the previous group's B1 reads of R / U
    if (live && pfG && active && tt == 0)
      prefetch_l2(G + e * 6 * NQ3, 6 * NQ3 * (int64_t)sizeof(double));
  }
  if (pf_ahead > 0 && tt == 0 && slot + pf_ahead < nlist) {
    const int64_t ea = elist ? (int64_t)elist[slot + pf_ahead] : slot + pf_ahead;
    prefetch_l2(u_ + ea * NQ3, NQ3 * (int64_t)sizeof(double));
  }
  if (NC > 1 && active && tt == 0) {
#pragma unroll
    for (int c = 1; c < NC; ++c)
      prefetch_l2(u_ + c * cstride + e * NQ3, NQ3 * (int64_t)sizeof(double));
  }

#pragma unroll
  for (int c = 0; c < NC; ++c) {
  const double* u = u_ + c * cstride;
  double* w = w_ + c * cstride;
  const double* ue = u + e * NQ3;
  if (NC > 1 && c > 0) __syncthreads();  // previous component's B1 reads of R / U
  if (NC > 1 && CDOT && st[c].done) {   // uniform over the grid
    if (t == 0) partials[c * pstride + part_base + blockIdx.x] = 0.0;
    continue;
  }

  // ---- F1: i-pencils (j = a, k = b)
  if (active) {
    double v[NQ], o[NQ];
    const double* row = ue + b * NQ2 + a * NQ;
    if (NQ % 2 == 0) {
#pragma unroll
      for (int m = 0; m < NQ; m += 2) {
        const double2 p = __ldg(reinterpret_cast<const double2*>(row + m));
        v[m] = p.x;
        v[m + 1] = p.y;
      }
    } else {
#pragma unroll
      for (int m = 0; m < NQ; ++m) v[m] = __ldg(row + m);
    }
    matvec<NQ, false>(D, v, o);
#pragma unroll
    for (int i = 0; i < NQ; ++i) {
      U[L::idx(b, a, i)] = v[i];
      Rr[L::idx(b, a, i)] = o[i];
    }
  }
  __syncthreads();
  // ---- F2: j-pencils (i = a, k = b) -> us ; F3: k-pencils (i = a, j = b) -> ut
  double ut[NQ];
  if (active) {
    double v[NQ], o[NQ];
#pragma unroll
    for (int m = 0; m < NQ; ++m) v[m] = U[L::idx(b, m, a)];
    matvec<NQ, false>(D, v, o);
#pragma unroll
    for (int j = 0; j < NQ; ++j) Ss[L::idx(b, j, a)] = o[j];
#pragma unroll
    for (int m = 0; m < NQ; ++m) v[m] = U[L::idx(m, b, a)];
    matvec<NQ, false>(D, v, ut);
  }
  __syncthreads();
  // ---- G: k-pencils (i = a, j = b): pointwise 3x3 symmetric multiply
  double gt[NQ];
  if (active) {
    const double* gp = G + e * 6 * NQ3 + b * NQ + a;
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      const double g0 = __ldg(gp + 0 * NQ3 + k * NQ2);
      const double g1 = __ldg(gp + 1 * NQ3 + k * NQ2);
      const double g2 = __ldg(gp + 2 * NQ3 + k * NQ2);
      const double g3 = __ldg(gp + 3 * NQ3 + k * NQ2);
      const double g4 = __ldg(gp + 4 * NQ3 + k * NQ2);
      const double g5 = __ldg(gp + 5 * NQ3 + k * NQ2);
      const int q = L::idx(k, b, a);
      const double ur = Rr[q], us = Ss[q];
      Rr[q] = g0 * ur + g1 * us + g2 * ut[k];
      Ss[q] = g1 * ur + g3 * us + g4 * ut[k];
      gt[k] = g2 * ur + g4 * us + g5 * ut[k];
    }
    // ---- B3: wt = D^T gt  (k-pencil) -> U
    double o[NQ];
    matvec<NQ, true>(D, gt, o);
#pragma unroll
    for (int k = 0; k < NQ; ++k) U[L::idx(k, b, a)] = o[k];
  }
  __syncthreads();
  // ---- B2: j-pencils (i = a, k = b): U <- D^T gs + wt
  if (active) {
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
  // ---- B1: i-pencils (j = a, k = b): w = D^T gr + (ws + wt), epilogue
  if (active) {
    double v[NQ], o[NQ];
#pragma unroll
    for (int m = 0; m < NQ; ++m) v[m] = Rr[L::idx(b, a, m)];
    matvec<NQ, true>(D, v, o);
    const int64_t off = e * NQ3 + b * NQ2 + a * NQ;
    double res[NQ];
#pragma unroll
    for (int i = 0; i < NQ; ++i) res[i] = lam0 * (o[i] + U[L::idx(b, a, i)]);
    if (B != nullptr || st != nullptr) {
      // u row again (L2-resident since F1) for lam1*B*u and the fused p.Ap
      double ur[NQ];
#pragma unroll
      for (int i = 0; i < NQ; ++i) ur[i] = __ldg(ue + b * NQ2 + a * NQ + i);
      if (B != nullptr) {
#pragma unroll
        for (int i = 0; i < NQ; ++i) res[i] = fma(lam1 * __ldg(B + off + i), ur[i], res[i]);
      }
      if (mask != nullptr) {
#pragma unroll
        for (int i = 0; i < NQ; ++i) res[i] = mask[off + i] ? res[i] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < NQ; ++i) dot = fma(ur[i], res[i], dot);
    } else if (mask != nullptr) {
#pragma unroll
      for (int i = 0; i < NQ; ++i) res[i] = mask[off + i] ? res[i] : 0.0;
    }
    double* wr = w + off;
    if (NQ % 2 == 0) {
#pragma unroll
      for (int i = 0; i < NQ; i += 2)
        *reinterpret_cast<double2*>(wr + i) = make_double2(res[i], res[i + 1]);
    } else {
#pragma unroll
      for (int i = 0; i < NQ; ++i) wr[i] = res[i];
    }
  }

  if (NC > 1 && CDOT) {
    // this component's block partial now (no accumulator lives across the
    // next component's contractions: the seq3 register budget is unchanged)
    double vv[1] = {dot};
    block_sum<1>(vv, red);
    if (t == 0) partials[c * pstride + part_base + blockIdx.x] = vv[0];
    dot = 0.0;
  }
  }  // components
  }  // element groups
  if ((NC == 1 || CDOT) && st != nullptr) {
    if (NC == 1) {
      double vv[1] = {dot};
      block_sum<1>(vv, red);
      if (t == 0) partials[part_base + blockIdx.x] = vv[0];
    }
    if (reduce_count > 0 && last_block(&st->ticket[0], gridDim.x)) {
      double s[NC];
      reduce_partials<NC>(partials, reduce_count, pstride, s, red);
      if (t == 0) {
#pragma unroll
        for (int c = 0; c < NC; ++c) st[c].pAp = s[c];
      }
    }
  }
}

// Fused-dot (NC = 1) launches at NQ <= 8 run the LOOP instantiation on a
// grid capped at the resident CTAs; above, the loop would spill (see the
// kernel) and the element counts are small anyway.
template <int NQ> struct PencilDotLoop { static constexpr bool value = NQ <= 8; };

// Partials of a fused-dot (NC = 1) pencil launch.
template <int NQ, int EPB, int MINB>
static int64_t pencil_dot_blocks(int64_t nlist) {
  using C = PencilCfg<NQ, EPB, MINB>;
  constexpr bool LP = PencilDotLoop<NQ>::value;
  const int64_t nblk = (nlist + EPB - 1) / EPB;
  if constexpr (!LP) {
    return nblk;
  } else {
  static int64_t resident = -1;
  if (resident < 0) {
    const size_t smem = C::smem_bytes();
    cudaFuncSetAttribute(bk5_pencil<NQ, EPB, MINB, 1, false, LP>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bk5_pencil<NQ, EPB, MINB, 1, false, LP>,
                                                  C::THREADS, smem);
    resident = (int64_t)sms * (per > 0 ? per : 1);
  }
  return nblk < resident ? nblk : resident;
  }
}

template <int NQ, int EPB, int MINB, int NC, bool CDOT, bool LOOP = false>
static int launch_pencil_k(int64_t nlist, const int32_t* elist, const double* Dhost,
                           const double* G, const double* u, double* w, double lam0,
                           const double* B, double lam1, const uint8_t* mask, nk_cg_state* st,
                           double* partials, int64_t part_base, int64_t reduce_count,
                           cudaStream_t s, int pfG, int64_t cstride, int64_t pstride);

template <int NQ, int EPB, int MINB, int NC = 1>
static int launch_pencil(int64_t nlist, const int32_t* elist, const double* Dhost,
                         const double* G, const double* u, double* w, double lam0,
                         const double* B, double lam1, const uint8_t* mask, nk_cg_state* st,
                         double* partials, int64_t part_base, int64_t reduce_count,
                         cudaStream_t s, int pfG, int64_t cstride = 0, int64_t pstride = 0) {
  if (NC > 1 && st != nullptr)   // per-component fused dots (nk_bk5_batch)
    return launch_pencil_k<NQ, EPB, MINB, NC, (NC > 1)>(nlist, elist, Dhost, G, u, w, lam0, B,
                                                       lam1, mask, st, partials, part_base,
                                                       reduce_count, s, pfG, cstride, pstride);
  if constexpr (NC == 1 && PencilDotLoop<NQ>::value) {
    if (st != nullptr)
      return launch_pencil_k<NQ, EPB, MINB, 1, false, true>(nlist, elist, Dhost, G, u, w, lam0, B,
                                                           lam1, mask, st, partials, part_base,
                                                           reduce_count, s, pfG, cstride, pstride);
  }
  return launch_pencil_k<NQ, EPB, MINB, NC, false>(nlist, elist, Dhost, G, u, w, lam0, B, lam1,
                                                   mask, st, partials, part_base, reduce_count, s,
                                                   pfG, cstride, pstride);
}

template <int NQ, int EPB, int MINB, int NC, bool CDOT, bool LOOP>
static int launch_pencil_k(int64_t nlist, const int32_t* elist, const double* Dhost,
                           const double* G, const double* u, double* w, double lam0,
                           const double* B, double lam1, const uint8_t* mask, nk_cg_state* st,
                           double* partials, int64_t part_base, int64_t reduce_count,
                           cudaStream_t s, int pfG, int64_t cstride, int64_t pstride) {
  using C = PencilCfg<NQ, EPB, MINB>;
  static int64_t resident = -1;  // CTAs resident on the device (one wave)
  const size_t smem = C::smem_bytes() + sizeof(double) * 32 * (NC - 1);
  static bool configured = false;
  if (!configured) {
    cudaError_t err = cudaFuncSetAttribute(bk5_pencil<NQ, EPB, MINB, NC, CDOT, LOOP>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) {
      set_error("bk5_pencil: smem attribute (%zu B): %s", smem, cudaGetErrorString(err));
      return NK_ERR_CUDA;
    }
    configured = true;
  }
  int64_t nblk = (nlist + EPB - 1) / EPB;
  if (nblk == 0) return NK_OK;
  if (resident < 0) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bk5_pencil<NQ, EPB, MINB, NC, CDOT, LOOP>,
                                                  C::THREADS, smem);
    resident = (int64_t)sms * (per > 0 ? per : 1);
  }
  if (LOOP && nblk > resident) nblk = resident;   // = pencil_dot_blocks
  DParam<NQ> D;
  D.set(Dhost);
  // pfG: 0 off, 1 own G into L2, 2 own G + the element one wave ahead
  const int64_t ahead = pfG >= 2 ? resident * EPB : 0;
  launch_ex(st != nullptr ? kPdlStep : 0, bk5_pencil<NQ, EPB, MINB, NC, CDOT, LOOP>,
            dim3((unsigned)nblk), dim3(C::THREADS), smem, s, nlist, elist, D, G, u, w, lam0, B,
            lam1, mask, st, partials, part_base, reduce_count, pfG, ahead, cstride, pstride);
  return check_launch("bk5_pencil");
}

}  // namespace nk

namespace nk {

// ---------------------------------------------------------------------------
// Variant 5, "pencil2": the pencil scheme with TWO shared element buffers.
//   F1 i-pencils: u row (HBM)           -> ur -> R
//   F2 j-pencils: u column (L1/L2)      -> us -> S
//   F3 k-pencils: u column (L1/L2)      -> ut (registers)
//   G  k-pencils: gr -> R, gs -> S in place, gt (registers)
//   B2 j-pencils: S column -> D^T gs    -> S in place (the pencil owns it)
//   B3 k-pencils: D^T gt + S column     -> S in place
//   B1 i-pencils: D^T R row + S row     -> epilogue -> HBM
// 12 shared accesses per point instead of 15 and 2/3 of the shared memory
// (more resident CTAs), for two extra L2 reads of u.
template <int NQ, int EPB>
struct Pencil2Cfg {
  static constexpr int VOL = PencilLayout<NQ>::VOL;
  static size_t smem_bytes() { return sizeof(double) * ((size_t)EPB * 2 * VOL + 32); }
};

template <int NQ, int EPB, int MINB, bool LOOP = false>
__global__ void __launch_bounds__(EPB * NQ * NQ, MINB)
bk5_pencil2(int64_t nlist, const int32_t* __restrict__ elist, const __grid_constant__ DParam<NQ> D,
            const double* __restrict__ G, const double* __restrict__ u, double* __restrict__ w,
            double lam0, const double* __restrict__ B, double lam1,
            const uint8_t* __restrict__ mask, nk_cg_state* st, double* __restrict__ partials,
            int64_t part_base, int64_t reduce_count, int pfG) {
  using L = PencilLayout<NQ>;
  constexpr int NQ2 = NQ * NQ, NQ3 = NQ2 * NQ, VOL = L::VOL;
  extern __shared__ double smem[];
  if (st != nullptr && st->done) return;
  const int t = threadIdx.x;
  const int le = t / NQ2;
  const int tt = t - le * NQ2;
  const int a = tt % NQ, b = tt / NQ;
  double* red = smem;
  double* Rr = smem + 32 + (size_t)le * 2 * VOL;
  double* Ss = Rr + VOL;
  // LOOP: capped grid-stride grid for fused-dot launches (see bk5_pencil)
  const int64_t nblk = (nlist + EPB - 1) / EPB;
  double dot = 0.0;
  int once = 0;   // LOOP = false: exactly one trip, provable at compile time
  for (int64_t blk = blockIdx.x; LOOP ? blk < nblk : once < 1; blk += gridDim.x, ++once) {
  if (LOOP && blk != blockIdx.x) __syncthreads();   // the previous group's B1 reads of R / S
  const int64_t slot = blk * EPB + le;
  const bool active = slot < nlist;
  const int64_t e = active ? (elist ? (int64_t)elist[slot] : slot) : 0;
  const double* ue = u + e * NQ3;
  if (pfG && active && tt == 0) prefetch_l2(G + e * 6 * NQ3, 6 * NQ3 * (int64_t)sizeof(double));

  if (active) {  // F1: i-pencils (j = a, k = b)
    double v[NQ], o[NQ];
    const double* row = ue + b * NQ2 + a * NQ;
    if (NQ % 2 == 0) {
#pragma unroll
      for (int m = 0; m < NQ; m += 2) {
        const double2 p = __ldg(reinterpret_cast<const double2*>(row + m));
        v[m] = p.x;
        v[m + 1] = p.y;
      }
    } else {
#pragma unroll
      for (int m = 0; m < NQ; ++m) v[m] = __ldg(row + m);
    }
    matvec<NQ, false>(D, v, o);
#pragma unroll
    for (int i = 0; i < NQ; ++i) Rr[L::idx(b, a, i)] = o[i];
  }
  double ut[NQ];
  if (active) {  // F2: j-pencils (i = a, k = b) from L1/L2 ; F3: k-pencils (i = a, j = b)
    double v[NQ], o[NQ];
#pragma unroll
    for (int m = 0; m < NQ; ++m) v[m] = __ldg(ue + b * NQ2 + m * NQ + a);
    matvec<NQ, false>(D, v, o);
#pragma unroll
    for (int j = 0; j < NQ; ++j) Ss[L::idx(b, j, a)] = o[j];
#pragma unroll
    for (int m = 0; m < NQ; ++m) v[m] = __ldg(ue + m * NQ2 + b * NQ + a);
    matvec<NQ, false>(D, v, ut);
  }
  __syncthreads();
  double gt[NQ];
  if (active) {  // G: k-pencils
    const double* gp = G + e * 6 * NQ3 + b * NQ + a;
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      const double g0 = __ldg(gp + 0 * NQ3 + k * NQ2), g1 = __ldg(gp + 1 * NQ3 + k * NQ2);
      const double g2 = __ldg(gp + 2 * NQ3 + k * NQ2), g3 = __ldg(gp + 3 * NQ3 + k * NQ2);
      const double g4 = __ldg(gp + 4 * NQ3 + k * NQ2), g5 = __ldg(gp + 5 * NQ3 + k * NQ2);
      const int q = L::idx(k, b, a);
      const double ur = Rr[q], us = Ss[q];
      Rr[q] = g0 * ur + g1 * us + g2 * ut[k];
      Ss[q] = g1 * ur + g3 * us + g4 * ut[k];
      gt[k] = g2 * ur + g4 * us + g5 * ut[k];
    }
  }
  __syncthreads();
  if (active) {  // B2: j-pencils, in place on their own S column
    double v[NQ], o[NQ];
#pragma unroll
    for (int m = 0; m < NQ; ++m) v[m] = Ss[L::idx(b, m, a)];
    matvec<NQ, true>(D, v, o);
#pragma unroll
    for (int j = 0; j < NQ; ++j) Ss[L::idx(b, j, a)] = o[j];
  }
  __syncthreads();
  if (active) {  // B3: k-pencils, S column += D^T gt
    double o[NQ];
    matvec<NQ, true>(D, gt, o);
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      const int q = L::idx(k, b, a);
      Ss[q] = o[k] + Ss[q];
    }
  }
  __syncthreads();
  if (active) {  // B1: i-pencils + epilogue
    double v[NQ], o[NQ];
#pragma unroll
    for (int m = 0; m < NQ; ++m) v[m] = Rr[L::idx(b, a, m)];
    matvec<NQ, true>(D, v, o);
    const int64_t off = e * NQ3 + b * NQ2 + a * NQ;
    double res[NQ];
#pragma unroll
    for (int i = 0; i < NQ; ++i) res[i] = lam0 * (o[i] + Ss[L::idx(b, a, i)]);
    if (B != nullptr || st != nullptr) {
      double urw[NQ];
#pragma unroll
      for (int i = 0; i < NQ; ++i) urw[i] = __ldg(ue + b * NQ2 + a * NQ + i);
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
    double* wr = w + off;
    if (NQ % 2 == 0) {
#pragma unroll
      for (int i = 0; i < NQ; i += 2)
        *reinterpret_cast<double2*>(wr + i) = make_double2(res[i], res[i + 1]);
    } else {
#pragma unroll
      for (int i = 0; i < NQ; ++i) wr[i] = res[i];
    }
  }
  }  // element groups
  if (st != nullptr) {
    double vv[1] = {dot};
    block_sum<1>(vv, red);
    if (t == 0) partials[part_base + blockIdx.x] = vv[0];
    if (reduce_count > 0 && last_block(&st->ticket[0], gridDim.x)) {
      double s[1];
      reduce_partials<1>(partials, reduce_count, 0, s, red);
      if (t == 0) st->pAp = s[0];
    }
  }
}

// Partials of a fused-dot pencil2 launch (capped, LOOP, at NQ <= 8).
template <int NQ, int EPB, int MINB>
static int64_t pencil2_dot_blocks(int64_t nlist) {
  using C = Pencil2Cfg<NQ, EPB>;
  const int64_t nb = (nlist + EPB - 1) / EPB;
  if constexpr (!PencilDotLoop<NQ>::value) {
    return nb;
  } else {
  static int64_t resident = -1;
  if (resident < 0) {
    const size_t smem = C::smem_bytes();
    cudaFuncSetAttribute(bk5_pencil2<NQ, EPB, MINB, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bk5_pencil2<NQ, EPB, MINB, true>,
                                                  EPB * NQ * NQ, smem);
    resident = (int64_t)sms * (per > 0 ? per : 1);
  }
  return nb < resident ? nb : resident;
  }
}

template <int NQ, int EPB, int MINB>
static int launch_pencil2(int64_t nlist, const int32_t* elist, const double* Dhost,
                          const double* G, const double* u, double* w, double lam0,
                          const double* B, double lam1, const uint8_t* mask, nk_cg_state* st,
                          double* partials, int64_t part_base, int64_t reduce_count,
                          cudaStream_t s, int pfG) {
  using C = Pencil2Cfg<NQ, EPB>;
  const size_t smem = C::smem_bytes();
  static bool configured = false;
  if (!configured) {
    cudaError_t err = cudaFuncSetAttribute(bk5_pencil2<NQ, EPB, MINB>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) {
      set_error("bk5_pencil2: smem attribute (%zu B): %s", smem, cudaGetErrorString(err));
      return NK_ERR_CUDA;
    }
    configured = true;
  }
  const int64_t nblk = (nlist + EPB - 1) / EPB;
  if (nblk == 0) return NK_OK;
  DParam<NQ> D;
  D.set(Dhost);
  if constexpr (PencilDotLoop<NQ>::value) {
    if (st != nullptr) {
      static bool lconf = false;
      if (!lconf) {
        cudaFuncSetAttribute(bk5_pencil2<NQ, EPB, MINB, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        lconf = true;
      }
      const int64_t g = pencil2_dot_blocks<NQ, EPB, MINB>(nlist);
      bk5_pencil2<NQ, EPB, MINB, true><<<(unsigned)g, EPB * NQ * NQ, smem, s>>>(
          nlist, elist, D, G, u, w, lam0, B, lam1, mask, st, partials, part_base, reduce_count,
          pfG);
      return check_launch("bk5_pencil2");
    }
  }
  bk5_pencil2<NQ, EPB, MINB><<<(unsigned)nblk, EPB * NQ * NQ, smem, s>>>(
      nlist, elist, D, G, u, w, lam0, B, lam1, mask, st, partials, part_base, reduce_count, pfG);
  return check_launch("bk5_pencil2");
}

}  // namespace nk
