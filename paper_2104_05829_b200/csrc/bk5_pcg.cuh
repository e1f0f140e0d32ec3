// Fused PCG operator step (BP5): Jacobi direction update + deferred x update
// + BK5 + mask + p^T A p, in one pass over the elements.
//
// Iteration structure (SURVEY.md §3 call stack 4) with the
// vector work that reads element rows moved into the BK5 prologue:
//
//   this kernel (iteration k, st->iter = k):
//     k > 0:  test ||r_k|| (st->rr) -> stop on convergence / max_iter
//             x   += alpha_{k-1} p_{k-1}                 (deferred x update)
//             p_k  = invD r_k + beta_k p_{k-1}           (FR or flexible beta)
//     w = mask * (lam0 A_L p_k + lam1 B p_k);  st->pAp = sum_L p_k w
//   then gs(w) -> Ap, and nk_cg_update(x = NULL): r -= alpha_k Ap, rr, rz.
//
// HBM per point: p, r, invD, x read (32) + G (48) + mask (1) + p, x, w
// written (24) = 105 B, replacing BK5 (65) + the p-update pass (32) + the x
// part of the update pass (24).  Same pencil compute as bk5_pencil.cuh.
#pragma once
#include "bk5_pencil.cuh"

namespace nk {

__device__ __forceinline__ double U_p_reload(const double* p, int64_t off, int i) {
  return p[off + i];
}

template <int NQ, int EPB, int MINB>
__global__ void __launch_bounds__(EPB * NQ * NQ, MINB)
bk5_pencil_pcg(int64_t nlist, const int32_t* __restrict__ elist,
               const __grid_constant__ DParam<NQ> D, const double* __restrict__ G,
               double* __restrict__ p, double* __restrict__ w, double lam0,
               const double* __restrict__ B, double lam1, const uint8_t* __restrict__ mask,
               double* __restrict__ x, const double* __restrict__ r,
               const double* __restrict__ invD, nk_cg_state* st, double* __restrict__ partials,
               int64_t part_base, int64_t reduce_count, double* __restrict__ hist) {
  using L = PencilLayout<NQ>;
  constexpr int NQ2 = NQ * NQ, NQ3 = NQ2 * NQ, VOL = L::VOL;
  extern __shared__ double smem[];
  if (st->done) return;
  const int it = st->iter;
  const bool conv = it > 0 && st->rr <= st->thresh2;
  const bool stop = it > 0 && (conv || it >= st->max_iter);
  const double alpha_prev = st->alpha;
  const double rz = st->rz;
  const double beta = it == 0 ? 0.0 : (st->flexible ? (-alpha_prev * st->zap) / rz
                                                    : st->rz_new / rz);

  const int t = threadIdx.x;
  const int le = t / NQ2;
  const int tt = t - le * NQ2;
  const int a = tt % NQ, b = tt / NQ;
  double* red = smem;
  double* U = smem + 32 + (size_t)le * 3 * VOL;
  double* Rr = U + VOL;
  double* Ss = Rr + VOL;

  const int64_t slot = (int64_t)blockIdx.x * EPB + le;
  const bool active = slot < nlist;
  const int64_t e = active ? (elist ? (int64_t)elist[slot] : slot) : 0;
  const int64_t off = e * NQ3 + b * NQ2 + a * NQ;  // this thread's i-row
  if (active && !stop && tt == 0) prefetch_l2(G + e * 6 * NQ3, 6 * NQ3 * (int64_t)sizeof(double));

  // ---- prologue on the i-row (j = a, k = b): x, p updates
  double prow[NQ];
  if (active) {
    if (NQ % 2 == 0) {  // 16-byte row accesses (rows are 16-B aligned for even NQ)
#pragma unroll
      for (int i = 0; i < NQ; i += 2) {
        const double2 pv = *reinterpret_cast<const double2*>(p + off + i);
        prow[i] = pv.x;
        prow[i + 1] = pv.y;
      }
      if (it > 0) {
#pragma unroll
        for (int i = 0; i < NQ; i += 2) {
          double2 xv = *reinterpret_cast<const double2*>(x + off + i);
          xv.x = fma(alpha_prev, prow[i], xv.x);
          xv.y = fma(alpha_prev, prow[i + 1], xv.y);
          *reinterpret_cast<double2*>(x + off + i) = xv;
        }
        if (!stop) {
#pragma unroll
          for (int i = 0; i < NQ; i += 2) {
            const double2 rv = __ldg(reinterpret_cast<const double2*>(r + off + i));
            const double2 dv = __ldg(reinterpret_cast<const double2*>(invD + off + i));
            prow[i] = fma(beta, prow[i], dv.x * rv.x);
            prow[i + 1] = fma(beta, prow[i + 1], dv.y * rv.y);
            *reinterpret_cast<double2*>(p + off + i) = make_double2(prow[i], prow[i + 1]);
          }
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < NQ; ++i) prow[i] = p[off + i];
      if (it > 0) {
#pragma unroll
        for (int i = 0; i < NQ; ++i) x[off + i] = fma(alpha_prev, prow[i], x[off + i]);
        if (!stop) {
#pragma unroll
          for (int i = 0; i < NQ; ++i)
            prow[i] = fma(beta, prow[i], __ldg(invD + off + i) * __ldg(r + off + i));
#pragma unroll
          for (int i = 0; i < NQ; ++i) p[off + i] = prow[i];
        }
      }
    }
  }
  double dot = 0.0;
  if (!stop) {  // block-uniform
    // ---- F1: i-pencils
    if (active) {
      double o[NQ];
      matvec<NQ, false>(D, prow, o);
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        U[L::idx(b, a, i)] = prow[i];
        Rr[L::idx(b, a, i)] = o[i];
      }
    }
    __syncthreads();
    double ut[NQ];
    if (active) {  // F2 (j-pencils) -> S ; F3 (k-pencils) -> ut
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
    if (active) {  // G (k-pencils), B3 -> U
      double gt[NQ];
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
      double o[NQ];
      matvec<NQ, true>(D, gt, o);
#pragma unroll
      for (int k = 0; k < NQ; ++k) U[L::idx(k, b, a)] = o[k];
    }
    __syncthreads();
    if (active) {  // B2 (j-pencils)
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
    if (active) {  // B1 (i-pencils) + epilogue
      double v[NQ], o[NQ];
#pragma unroll
      for (int m = 0; m < NQ; ++m) v[m] = Rr[L::idx(b, a, m)];
      matvec<NQ, true>(D, v, o);
      double res[NQ];
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        // p row re-read (written by this thread in the prologue; L1/L2 hit)
        // rather than held live across the kernel -- keeps registers down
        const double pi = U_p_reload(p, off, i);
        double vv = lam0 * (o[i] + U[L::idx(b, a, i)]);
        if (B != nullptr) vv = fma(lam1 * __ldg(B + off + i), pi, vv);
        if (mask != nullptr) vv = mask[off + i] ? vv : 0.0;
        res[i] = vv;
        dot = fma(pi, vv, dot);
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
  }

  double vv[1] = {dot};
  block_sum<1>(vv, red);
  if (t == 0) partials[part_base + blockIdx.x] = vv[0];
  if (reduce_count > 0 && last_block(&st->ticket[0], gridDim.x)) {
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
  }
}

template <int NQ, int EPB, int MINB>
static int launch_pencil_pcg(int64_t nlist, const int32_t* elist, const double* Dhost,
                             const double* G, double* p, double* w, double lam0, const double* B,
                             double lam1, const uint8_t* mask, double* x, const double* r,
                             const double* invD, nk_cg_state* st, double* partials,
                             int64_t part_base, int64_t reduce_count, double* hist,
                             cudaStream_t s) {
  using C = PencilCfg<NQ, EPB, MINB>;
  const size_t smem = C::smem_bytes();
  static bool configured = false;
  if (!configured) {
    cudaError_t err = cudaFuncSetAttribute(bk5_pencil_pcg<NQ, EPB, MINB>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) {
      set_error("bk5_pencil_pcg: smem attribute (%zu B): %s", smem, cudaGetErrorString(err));
      return NK_ERR_CUDA;
    }
    configured = true;
  }
  const int64_t nblk = (nlist + EPB - 1) / EPB;
  if (nblk == 0) return NK_OK;
  DParam<NQ> D;
  D.set(Dhost);
  bk5_pencil_pcg<NQ, EPB, MINB><<<(unsigned)nblk, C::THREADS, smem, s>>>(
      nlist, elist, D, G, p, w, lam0, B, lam1, mask, x, r, invD, st, partials, part_base,
      reduce_count, hist);
  return check_launch("bk5_pencil_pcg");
}


// N = 1 (NQ = 2, 8 points per element): the pencil machinery (shared
// transposes, barriers) costs more than the element's arithmetic, so each
// element is owned by 8 consecutive lanes, one point per lane: every load
// (p, r, invD, x, G's six components) is warp-coalesced, and the three
// 2-point derivatives and their transposes swap partner values with xor
// shuffles (lane bit 0 = i, 1 = j, 2 = k).  Both kernels below share it:
// the plain apply (nk_bk5 at N = 1) and the fused PCG step (the
// p-multigrid's iterative order-1 coarse solve).
constexpr int kN1PtThreads = 256;

// (G grad p)ᵀ grad at point q = k*4 + j*2 + i of the lane's element; all
// 32 lanes must call it (shuffles).  g = the point's six G components.
__device__ __forceinline__ double n1_point_stiffness(double pv, const double (&g)[6],
                                                     const DParam<2>& D, int q) {
  const int i = q & 1, j = (q >> 1) & 1, k = q >> 2;
  const double pi = __shfl_xor_sync(0xffffffffu, pv, 1);
  const double pj = __shfl_xor_sync(0xffffffffu, pv, 2);
  const double pk = __shfl_xor_sync(0xffffffffu, pv, 4);
  // d/dr at (i,j,k) = D[i][0] u(0,j,k) + D[i][1] u(1,j,k)
  const double ur = i ? D.d[2] * pi + D.d[3] * pv : D.d[0] * pv + D.d[1] * pi;
  const double us = j ? D.d[2] * pj + D.d[3] * pv : D.d[0] * pv + D.d[1] * pj;
  const double ut = k ? D.d[2] * pk + D.d[3] * pv : D.d[0] * pv + D.d[1] * pk;
  const double gr = g[0] * ur + g[1] * us + g[2] * ut;
  const double gs = g[1] * ur + g[3] * us + g[4] * ut;
  const double gt = g[2] * ur + g[4] * us + g[5] * ut;
  const double ri = __shfl_xor_sync(0xffffffffu, gr, 1);
  const double sj = __shfl_xor_sync(0xffffffffu, gs, 2);
  const double tk = __shfl_xor_sync(0xffffffffu, gt, 4);
  // transpose: sum_a D[a][i] gr(a,j,k) (+ s, t)
  double v = i ? D.d[1] * ri + D.d[3] * gr : D.d[0] * gr + D.d[2] * ri;
  v += j ? D.d[1] * sj + D.d[3] * gs : D.d[0] * gs + D.d[2] * sj;
  v += k ? D.d[1] * tk + D.d[3] * gt : D.d[0] * gt + D.d[2] * tk;
  return v;
}

template <int NQ_ONE>   // = 2; a template so every translation unit may include it
__global__ void __launch_bounds__(kN1PtThreads)
bk5_n1_pcg(int64_t nlist, const int32_t* __restrict__ elist, const __grid_constant__ DParam<2> D,
           const double* __restrict__ G, double* __restrict__ p, double* __restrict__ w,
           double lam0, const double* __restrict__ B, double lam1,
           const uint8_t* __restrict__ mask, double* __restrict__ x,
           const double* __restrict__ r, const double* __restrict__ invD, nk_cg_state* st,
           double* __restrict__ partials, int64_t part_base, int64_t reduce_count,
           double* __restrict__ hist) {
  __shared__ double red[32];
  if (st->done) return;
  const int it = st->iter;
  const bool conv = it > 0 && st->rr <= st->thresh2;
  const bool stop = it > 0 && (conv || it >= st->max_iter);
  const double alpha_prev = st->alpha;
  const double rz = st->rz;
  const double beta = it == 0 ? 0.0 : (st->flexible ? (-alpha_prev * st->zap) / rz
                                                    : st->rz_new / rz);
  const int t = threadIdx.x;
  const int64_t slot = ((int64_t)blockIdx.x * kN1PtThreads + t) >> 3;
  const int q = t & 7;
  const bool active = slot < nlist;
  const int64_t e = active ? (elist ? (int64_t)elist[slot] : slot) : 0;
  const int64_t pt = e * 8 + q;
  double dot = 0.0;
  // every load issued in one batch (one memory round trip per lane)
  double pv = 0.0, xv = 0.0, rv = 0.0, dv = 0.0, g[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  if (active) {
    pv = p[pt];
    if (it > 0) xv = x[pt];
    if (!stop) {
      if (it > 0) {
        rv = __ldg(r + pt);
        dv = __ldg(invD + pt);
      }
#pragma unroll
      for (int c = 0; c < 6; ++c) g[c] = __ldg(G + e * 48 + c * 8 + q);
    }
  }
  if (it > 0 && active) {
    x[pt] = fma(alpha_prev, pv, xv);
    if (!stop) {
      pv = fma(beta, pv, dv * rv);
      p[pt] = pv;
    }
  }
  if (!stop) {   // grid-uniform
    double v = lam0 * n1_point_stiffness(pv, g, D, q);
    if (active) {
      if (B != nullptr) v = fma(lam1 * __ldg(B + pt), pv, v);
      if (mask != nullptr) v = mask[pt] ? v : 0.0;
      w[pt] = v;
      dot = pv * v;
    }
  }
  double vv[1] = {dot};
  block_sum<1>(vv, red);
  if (t == 0) partials[part_base + blockIdx.x] = vv[0];
  if (reduce_count > 0 && last_block(&st->ticket[0], gridDim.x)) {
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
  }
}

constexpr int64_t kN1DotBlocks = 1184;   // 8 x 148: one resident wave of 256-thread CTAs

template <int NQ_ONE, bool LOOP = false>   // NQ_ONE = 2
__global__ void __launch_bounds__(kN1PtThreads)
bk5_n1(int64_t nlist, const int32_t* __restrict__ elist, const __grid_constant__ DParam<2> D,
       const double* __restrict__ G, const double* __restrict__ u, double* __restrict__ w,
       double lam0, const double* __restrict__ B, double lam1, const uint8_t* __restrict__ mask,
       nk_cg_state* st, double* __restrict__ partials, int64_t part_base, int64_t reduce_count) {
  // LOOP (fused-dot launches): grid-stride over a grid capped at kN1DotBlocks,
  // so the partials / last-block ticket stay short (an uncapped launch at
  // E = 96^3 had 27648 partials, ~50 us of same-address atomics).
  __shared__ double red[32];
  if (st != nullptr && st->done) return;
  const int t = threadIdx.x;
  const int q = t & 7;
  const int64_t nblk = (nlist * 8 + kN1PtThreads - 1) / kN1PtThreads;
  double dot = 0.0;
  int once = 0;
  for (int64_t blk = blockIdx.x; LOOP ? blk < nblk : once < 1; blk += gridDim.x, ++once) {
    const int64_t slot = (blk * kN1PtThreads + t) >> 3;
    const bool active = slot < nlist;
    const int64_t e = active ? (elist ? (int64_t)elist[slot] : slot) : 0;
    const int64_t pt = e * 8 + q;
    const double pv = active ? __ldg(u + pt) : 0.0;
    double g[6];
#pragma unroll
    for (int c = 0; c < 6; ++c) g[c] = active ? __ldg(G + e * 48 + c * 8 + q) : 0.0;
    double v = lam0 * n1_point_stiffness(pv, g, D, q);
    if (active) {
      if (B != nullptr) v = fma(lam1 * __ldg(B + pt), pv, v);
      if (mask != nullptr) v = mask[pt] ? v : 0.0;
      w[pt] = v;
      dot = fma(pv, v, dot);
    }
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

}  // namespace nk
