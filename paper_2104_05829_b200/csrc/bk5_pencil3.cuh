// BK5 3-component batch (vector Helmholtz, SPEC.md:403, PAPER.md:995-999,
// SURVEY.md §8a a10): w_c = lam0 A u_c + lam1 B u_c for c = 0, 1, 2 with the
// six geometric factors read from HBM ONCE per element (G is shared by the
// three velocity components).
//
// One element per CTA (NQ^2 threads).  G (and B, swizzled for the i-pencil
// epilogue) are staged in shared memory with 16-byte cp.async copies; the
// three components then run the pencil pipeline of bk5_pencil.cuh against
// the staged factors.  HBM per point: 3 x (u 8 + w 8) + G 48 + B 8 = 104 B.
#pragma once
#include "bk5_pencil.cuh"

namespace nk {

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

template <int NQ>
struct Pencil3Cfg {
  static constexpr int NQ2 = NQ * NQ, NQ3 = NQ2 * NQ;
  static constexpr int VOL = PencilLayout<NQ>::VOL;
  // doubles: red[32] | G[6 NQ3] | B[VOL] | U R S
  static size_t smem_bytes() { return sizeof(double) * (32 + 6 * NQ3 + 4 * VOL); }
};

template <int NQ, int MINB>
__global__ void __launch_bounds__(NQ * NQ, MINB)
bk5_pencil3(int64_t nlist, const int32_t* __restrict__ elist,
            const __grid_constant__ DParam<NQ> D, const double* __restrict__ G,
            const double* __restrict__ u, double* __restrict__ w, double lam0,
            const double* __restrict__ B, double lam1, int64_t cstride,
            const uint8_t* __restrict__ mask) {
  static_assert(NQ % 2 == 0, "16-byte staging of G needs even NQ");
  using L = PencilLayout<NQ>;
  constexpr int NQ2 = NQ * NQ, NQ3 = NQ2 * NQ, VOL = L::VOL;
  extern __shared__ __align__(128) double smem[];
  double* sG = smem + 32;
  double* sB = sG + 6 * NQ3;
  double* U = sB + VOL;
  double* Rr = U + VOL;
  double* Ss = Rr + VOL;
  const int t = threadIdx.x;
  const int a = t % NQ, b = t / NQ;
  const int64_t slot = blockIdx.x;
  if (slot >= nlist) return;
  const int64_t e = elist ? (int64_t)elist[slot] : slot;

  {  // stage G (16-B cp.async, coalesced) and B (swizzled like U)
    const double* gsrc = G + e * 6 * NQ3;
    for (int q = 2 * t; q < 6 * NQ3; q += 2 * NQ2) cp_async16(sG + q, gsrc + q);
    if (B != nullptr) {
#pragma unroll
      for (int k = 0; k < NQ; ++k) sB[L::idx(k, b, a)] = __ldg(B + e * NQ3 + k * NQ2 + t);
    }
    cp_async_wait_all();
  }
  __syncthreads();

  for (int c = 0; c < 3; ++c) {
    const double* ue = u + c * cstride + e * NQ3;
    // ---- F1: i-pencils (j = a, k = b)
    {
      double v[NQ], o[NQ];
      const double* row = ue + b * NQ2 + a * NQ;
#pragma unroll
      for (int m = 0; m < NQ; m += 2) {
        const double2 p = __ldg(reinterpret_cast<const double2*>(row + m));
        v[m] = p.x;
        v[m + 1] = p.y;
      }
      matvec<NQ, false>(D, v, o);
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        U[L::idx(b, a, i)] = v[i];
        Rr[L::idx(b, a, i)] = o[i];
      }
    }
    __syncthreads();
    double ut[NQ];
    {  // F2 -> S ; F3 -> ut
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
    {
      double gt[NQ];
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        const int pp = k * NQ2 + t;
        const double g0 = sG[0 * NQ3 + pp], g1 = sG[1 * NQ3 + pp], g2 = sG[2 * NQ3 + pp];
        const double g3 = sG[3 * NQ3 + pp], g4 = sG[4 * NQ3 + pp], g5 = sG[5 * NQ3 + pp];
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
    {  // B2
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
    {  // B1 + epilogue
      double v[NQ], o[NQ];
#pragma unroll
      for (int m = 0; m < NQ; ++m) v[m] = Rr[L::idx(b, a, m)];
      matvec<NQ, true>(D, v, o);
      const int64_t off = e * NQ3 + b * NQ2 + a * NQ;
      const double* urow = ue + b * NQ2 + a * NQ;  // L1/L2-resident since F1
      double res[NQ];
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        double vv = lam0 * (o[i] + U[L::idx(b, a, i)]);
        if (B != nullptr) vv = fma(lam1 * sB[L::idx(b, a, i)], __ldg(urow + i), vv);
        if (mask != nullptr) vv = mask[off + i] ? vv : 0.0;
        res[i] = vv;
      }
      double* wr = w + c * cstride + off;
#pragma unroll
      for (int i = 0; i < NQ; i += 2)
        *reinterpret_cast<double2*>(wr + i) = make_double2(res[i], res[i + 1]);
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
  for (int q = 0; q < NQ * NQ; ++q) D.d[q] = Dhost[q];
  bk5_pencil3<NQ, MINB><<<(unsigned)nlist, NQ * NQ, smem, s>>>(nlist, elist, D, G, u, w, lam0, B,
                                                              lam1, cstride, mask);
  return check_launch("bk5_pencil3");
}

}  // namespace nk
