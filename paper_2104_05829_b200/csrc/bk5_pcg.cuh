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
  for (int q = 0; q < NQ * NQ; ++q) D.d[q] = Dhost[q];
  bk5_pencil_pcg<NQ, EPB, MINB><<<(unsigned)nblk, C::THREADS, smem, s>>>(
      nlist, elist, D, G, p, w, lam0, B, lam1, mask, x, r, invD, st, partials, part_base,
      reduce_count, hist);
  return check_launch("bk5_pencil_pcg");
}


// N = 1 (NQ = 2, 8 points per element): the pencil machinery (shared
// transposes, barriers) costs more than the element's arithmetic, so one
// THREAD owns one element -- p, r, invD, x, w as four 16-B loads each and
// G as 24 -- with the same prologue / epilogue semantics as bk5_pencil_pcg.
// Used by the iterative coarse solve of the p-multigrid (order-1 level).
constexpr int kN1Threads = 128;

template <int NQ_ONE>   // = 2; a template so every translation unit may include it
__global__ void __launch_bounds__(kN1Threads)
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
  const int64_t slot = (int64_t)blockIdx.x * kN1Threads + t;
  const bool active = slot < nlist;
  const int64_t e = active ? (elist ? (int64_t)elist[slot] : slot) : 0;
  const int64_t off = e * 8;
  double dot = 0.0;
  if (active) {
    double pv[8];
#pragma unroll
    for (int q = 0; q < 8; q += 2) {
      const double2 v = *reinterpret_cast<const double2*>(p + off + q);
      pv[q] = v.x;
      pv[q + 1] = v.y;
    }
    if (it > 0) {
#pragma unroll
      for (int q = 0; q < 8; q += 2) {
        double2 xv = *reinterpret_cast<const double2*>(x + off + q);
        xv.x = fma(alpha_prev, pv[q], xv.x);
        xv.y = fma(alpha_prev, pv[q + 1], xv.y);
        *reinterpret_cast<double2*>(x + off + q) = xv;
      }
      if (!stop) {
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
          const double2 rv = __ldg(reinterpret_cast<const double2*>(r + off + q));
          const double2 dv = __ldg(reinterpret_cast<const double2*>(invD + off + q));
          pv[q] = fma(beta, pv[q], dv.x * rv.x);
          pv[q + 1] = fma(beta, pv[q + 1], dv.y * rv.y);
          *reinterpret_cast<double2*>(p + off + q) = make_double2(pv[q], pv[q + 1]);
        }
      }
    }
    if (!stop) {
      // point q = k*4 + j*2 + i;  d/dr along i, d/ds along j, d/dt along k
      double ur[8], us[8], ut[8];
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int q = k * 4 + j * 2 + i;
            ur[q] = D.d[i * 2 + 0] * pv[k * 4 + j * 2 + 0] + D.d[i * 2 + 1] * pv[k * 4 + j * 2 + 1];
            us[q] = D.d[j * 2 + 0] * pv[k * 4 + 0 * 2 + i] + D.d[j * 2 + 1] * pv[k * 4 + 1 * 2 + i];
            ut[q] = D.d[k * 2 + 0] * pv[0 * 4 + j * 2 + i] + D.d[k * 2 + 1] * pv[1 * 4 + j * 2 + i];
          }
      const double* ge = G + e * 48;
      double g[48];
#pragma unroll
      for (int q = 0; q < 48; q += 2) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(ge + q));
        g[q] = v.x;
        g[q + 1] = v.y;
      }
      double gr[8], gs[8], gt[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        gr[q] = g[q] * ur[q] + g[8 + q] * us[q] + g[16 + q] * ut[q];
        gs[q] = g[8 + q] * ur[q] + g[24 + q] * us[q] + g[32 + q] * ut[q];
        gt[q] = g[16 + q] * ur[q] + g[32 + q] * us[q] + g[40 + q] * ut[q];
      }
      double res[8];
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int q = k * 4 + j * 2 + i;
            double v = D.d[0 * 2 + i] * gr[k * 4 + j * 2 + 0] + D.d[1 * 2 + i] * gr[k * 4 + j * 2 + 1];
            v += D.d[0 * 2 + j] * gs[k * 4 + 0 * 2 + i] + D.d[1 * 2 + j] * gs[k * 4 + 1 * 2 + i];
            v += D.d[0 * 2 + k] * gt[0 * 4 + j * 2 + i] + D.d[1 * 2 + k] * gt[1 * 4 + j * 2 + i];
            v *= lam0;
            if (B != nullptr) v = fma(lam1 * __ldg(B + off + q), pv[q], v);
            if (mask != nullptr) v = mask[off + q] ? v : 0.0;
            res[q] = v;
            dot = fma(pv[q], v, dot);
          }
#pragma unroll
      for (int q = 0; q < 8; q += 2)
        *reinterpret_cast<double2*>(w + off + q) = make_double2(res[q], res[q + 1]);
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

}  // namespace nk
