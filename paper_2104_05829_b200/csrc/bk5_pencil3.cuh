// BK5 3-component batch (vector Helmholtz, SPEC.md:403, PAPER.md:995-999,
// SURVEY.md §8a a10): w_c = lam0 A u_c + lam1 B u_c for c = 0, 1, 2 with the
// six geometric factors read from HBM ONCE per element (G is shared by the
// three velocity components).
//
// One element per CTA (NQ^2 threads).  The three components' forward passes
// run first (R_c, S_c in shared memory, t-derivatives in registers); a single
// G pass then loads each k-plane's six factors into registers once and
// applies them to all three components; the three backward passes follow.
// Shared: U + 3 x (R, S) = 7 element buffers; no G staging (the element's G
// is bulk-prefetched into L2 at CTA start).  HBM per point for the three
// components: 3 x (u 8 + w 8) + G 48 + B 8 = 104 B.
#pragma once
#include "bk5_pencil.cuh"

namespace nk {

template <int NQ>
struct Pencil3Cfg {
  static constexpr int NQ2 = NQ * NQ, NQ3 = NQ2 * NQ;
  static constexpr int VOL = PencilLayout<NQ>::VOL;
  static size_t smem_bytes() { return sizeof(double) * (32 + 7 * (size_t)VOL); }
};

template <int NQ, int MINB>
__global__ void __launch_bounds__(NQ * NQ, MINB)
bk5_pencil3(int64_t nlist, const int32_t* __restrict__ elist,
            const __grid_constant__ DParam<NQ> D, const double* __restrict__ G,
            const double* __restrict__ u, double* __restrict__ w, double lam0,
            const double* __restrict__ B, double lam1, int64_t cstride,
            const uint8_t* __restrict__ mask) {
  using L = PencilLayout<NQ>;
  constexpr int NQ2 = NQ * NQ, NQ3 = NQ2 * NQ, VOL = L::VOL;
  extern __shared__ __align__(128) double smem[];
  double* U = smem + 32;
  double* Rr = U + VOL;         // Rr + c*VOL
  double* Ss = Rr + 3 * VOL;    // Ss + c*VOL
  const int t = threadIdx.x;
  const int a = t % NQ, b = t / NQ;
  const int64_t slot = blockIdx.x;
  if (slot >= nlist) return;
  const int64_t e = elist ? (int64_t)elist[slot] : slot;
  if (t == 0) prefetch_l2(G + e * 6 * NQ3, 6 * NQ3 * (int64_t)sizeof(double));

  double ut[3][NQ];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double* ue = u + c * cstride + e * NQ3;
    {  // F1: i-pencils -> R_c, U <- u_c
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
        Rr[c * VOL + L::idx(b, a, i)] = o[i];
      }
    }
    __syncthreads();
    {  // F2 -> S_c ; F3 -> ut_c
      double v[NQ], o[NQ];
#pragma unroll
      for (int m = 0; m < NQ; ++m) v[m] = U[L::idx(b, m, a)];
      matvec<NQ, false>(D, v, o);
#pragma unroll
      for (int j = 0; j < NQ; ++j) Ss[c * VOL + L::idx(b, j, a)] = o[j];
#pragma unroll
      for (int m = 0; m < NQ; ++m) v[m] = U[L::idx(m, b, a)];
      matvec<NQ, false>(D, v, ut[c]);
    }
    __syncthreads();
  }

  // ---- G pass (k-pencils): each plane's factors loaded once for 3 components
  double gt[3][NQ];
  {
    const double* gp = G + e * 6 * NQ3 + b * NQ + a;
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      const double g0 = __ldg(gp + 0 * NQ3 + k * NQ2), g1 = __ldg(gp + 1 * NQ3 + k * NQ2);
      const double g2 = __ldg(gp + 2 * NQ3 + k * NQ2), g3 = __ldg(gp + 3 * NQ3 + k * NQ2);
      const double g4 = __ldg(gp + 4 * NQ3 + k * NQ2), g5 = __ldg(gp + 5 * NQ3 + k * NQ2);
      const int q = L::idx(k, b, a);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double ur = Rr[c * VOL + q], us = Ss[c * VOL + q], uu = ut[c][k];
        Rr[c * VOL + q] = g0 * ur + g1 * us + g2 * uu;
        Ss[c * VOL + q] = g1 * ur + g3 * us + g4 * uu;
        gt[c][k] = g2 * ur + g4 * us + g5 * uu;
      }
    }
  }

#pragma unroll
  for (int c = 0; c < 3; ++c) {
    {  // B3: wt_c -> U
      double o[NQ];
      matvec<NQ, true>(D, gt[c], o);
#pragma unroll
      for (int k = 0; k < NQ; ++k) U[L::idx(k, b, a)] = o[k];
    }
    __syncthreads();
    {  // B2
      double v[NQ], o[NQ];
#pragma unroll
      for (int m = 0; m < NQ; ++m) v[m] = Ss[c * VOL + L::idx(b, m, a)];
      matvec<NQ, true>(D, v, o);
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        const int q = L::idx(b, j, a);
        U[q] = o[j] + U[q];
      }
    }
    __syncthreads();
    {  // B1 + epilogue
      double v[NQ], o[NQ];
#pragma unroll
      for (int m = 0; m < NQ; ++m) v[m] = Rr[c * VOL + L::idx(b, a, m)];
      matvec<NQ, true>(D, v, o);
      const int64_t off = e * NQ3 + b * NQ2 + a * NQ;
      const double* urow = u + c * cstride + off;   // L1/L2-resident since F1
      double res[NQ];
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        double vv = lam0 * (o[i] + U[L::idx(b, a, i)]);
        if (B != nullptr) vv = fma(lam1 * __ldg(B + off + i), __ldg(urow + i), vv);
        if (mask != nullptr) vv = mask[off + i] ? vv : 0.0;
        res[i] = vv;
      }
      double* wr = w + c * cstride + off;
      if (NQ % 2 == 0) {
#pragma unroll
        for (int i = 0; i < NQ; i += 2)
          *reinterpret_cast<double2*>(wr + i) = make_double2(res[i], res[i + 1]);
      } else {
#pragma unroll
        for (int i = 0; i < NQ; ++i) wr[i] = res[i];
      }
    }
    __syncthreads();
  }
}

template <int NQ, int MINB>
static int launch_pencil3(int64_t nlist, const int32_t* elist, const double* Dhost,
                          const double* G, const double* u, double* w, double lam0,
                          const double* B, double lam1, int64_t cstride, const uint8_t* mask,
                          cudaStream_t s) {
  using C = Pencil3Cfg<NQ>;
  const size_t smem = C::smem_bytes();
  static bool configured = false;
  if (!configured) {
    cudaError_t err = cudaFuncSetAttribute(bk5_pencil3<NQ, MINB>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) {
      set_error("bk5_pencil3: smem attribute (%zu B): %s", smem, cudaGetErrorString(err));
      return NK_ERR_CUDA;
    }
    configured = true;
  }
  if (nlist == 0) return NK_OK;
  DParam<NQ> D;
  D.set(Dhost);
  bk5_pencil3<NQ, MINB><<<(unsigned)nlist, NQ * NQ, smem, s>>>(nlist, elist, D, G, u, w, lam0, B,
                                                              lam1, cstride, mask);
  return check_launch("bk5_pencil3");
}

}  // namespace nk
