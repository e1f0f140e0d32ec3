// Overlapping Schwarz smoothing with fast-diagonalisation local solves
// (SPEC.md:410-418 fdm_local_solve, 499-507
// schwarz_smooth; (N+3)^3 extended
// elements, FDM cost ~12E(N+3)^4, ASM with the counting weight, RAS).
// oracle/schwarz.py states the algorithm on the CPU.
//
//   nk_fdm           one element per CTA, (N+3)^2 threads, each owning one
//                    1-D line of the extended box in shared memory:
//                    gather r (- sub) on the element and the face-neighbour
//                    layers -> S_x^T, S_y^T along lines -> (S_z^T, 1/Lambda,
//                    S_z) fused in one pass -> S_y, S_x -> extended (ASM) or
//                    own-point (RAS) output.  The 1-D S are per element
//                    (deformed meshes) and read broadcast from shared memory.
//                    6 (N+3)^4 DFMA per element, 2 (N+3)^3 shared transposes.
//   nk_schwarz_post  z = mask * W * (own points of the extended / own
//                    output) fused with the Chebyshev vector update
//                    d = a d + b z, e (+)= d.
#include "common.cuh"

namespace nk {

// One thread's 1-D contraction of its line L[0..NQE) (stride ST) in place:
// forward (FWD): L[a] = sum_i S[i][a] L[i]   (S^T), optionally scaled by
//                1 / (lam0 (lab + lz[a]) + lam1), 0 when that sum is +inf;
// backward:      L[i] = sum_a S[i][a] L[a].
// S is read from shared memory with every thread of the warp on the same
// address (broadcast); only the line lives in registers.
template <int NQE, int ST, bool FWD>
__device__ __forceinline__ void fdm_line(double* L, const double* __restrict__ Sm,
                                         const double* lz, double lab, double lam0,
                                         double lam1) {
  double v[NQE];
#pragma unroll
  for (int i = 0; i < NQE; ++i) v[i] = L[i * ST];
#pragma unroll 2
  for (int a = 0; a < NQE; ++a) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < NQE; ++i) s = fma(FWD ? Sm[i * NQE + a] : Sm[a * NQE + i], v[i], s);
    if (lz != nullptr) {
      const double lsum = lab + lz[a];
      s = isinf(lsum) ? 0.0 : s / fma(lam0, lsum, lam1);
    }
    L[a * ST] = s;
  }
}

template <int NQE>
__global__ void __launch_bounds__(NQE * NQE)
fdm_kernel(int64_t nelem, const double* __restrict__ r, const double* __restrict__ sub,
           double* __restrict__ res_out, const int32_t* __restrict__ fmap,
           const double* __restrict__ Sg, const double* __restrict__ lamg, double lam0,
           double lam1, double* __restrict__ out, int out_ext, const nk_cg_state* st) {
  if (st != nullptr && st->done) return;
  constexpr int NQ = NQE - 2;            // N + 1
  constexpr int NQ2 = NQ * NQ, NQ3 = NQ2 * NQ;
  constexpr int LS = NQE + 1;            // padded line stride
  constexpr int PS = NQE * LS;           // plane stride
  constexpr int NT = NQE * NQE;
  extern __shared__ __align__(16) double fdm_smem[];
  double* A = fdm_smem;                  // [k][j][i], padded lines
  double* Ss = A + NQE * PS;             // Ss[d][p][mode]
  double* Ls = Ss + 3 * NQE * NQE;       // lambda[d][mode]
  const int64_t e = blockIdx.x;
  const int t = threadIdx.x;
  const double* Se = Sg + e * 3 * NQE * NQE;
  for (int q = t; q < 3 * NQE * NQE; q += NT) Ss[q] = __ldg(Se + q);
  if (t < 3 * NQE) Ls[t] = __ldg(lamg + e * 3 * NQE + t);
  // own points (coalesced) + zero elsewhere
  const int64_t ob = e * NQ3;
  for (int q = t; q < NQE * NQE * NQE; q += NT) {
    const int i = q % NQE, j = (q / NQE) % NQE, k = q / (NQE * NQE);
    A[k * PS + j * LS + i] = 0.0;
  }
  __syncthreads();
  for (int q = t; q < NQ3; q += NT) {
    const int i = q % NQ, j = (q / NQ) % NQ, k = q / NQ2;
    double v = __ldg(r + ob + q);
    if (sub) v -= __ldg(sub + ob + q);
    if (res_out) res_out[ob + q] = v;
    A[(k + 1) * PS + (j + 1) * LS + (i + 1)] = v;
  }
  // face-neighbour layers: face f, tangential (a, b) slow/fast
  const int32_t* fm = fmap + e * 6 * NQ2;
  for (int q = t; q < 6 * NQ2; q += NT) {
    const int32_t src = __ldg(fm + q);
    if (src < 0) continue;
    const int f = q / NQ2, ab = q % NQ2, a = ab / NQ + 1, b = ab % NQ + 1;
    const int pos = (f & 1) ? NQE - 1 : 0;
    double v = __ldg(r + src);
    if (sub) v -= __ldg(sub + src);
    int idx;
    if (f < 2) idx = a * PS + b * LS + pos;        // x faces: (k, j)
    else if (f < 4) idx = a * PS + pos * LS + b;   // y faces: (k, i)
    else idx = pos * PS + a * LS + b;              // z faces: (j, i)
    A[idx] = v;
  }
  __syncthreads();
  const double* Sx = Ss;
  const double* Sy = Ss + NQE * NQE;
  const double* Sz = Ss + 2 * NQE * NQE;
  const int t1 = t / NQE, t0 = t % NQE;
  // forward x: line (k = t1, j = t0) along i
  fdm_line<NQE, 1, true>(A + t1 * PS + t0 * LS, Sx, nullptr, 0.0, 0.0, 0.0);
  __syncthreads();
  // forward y: line (k = t1, i = t0) along j
  fdm_line<NQE, LS, true>(A + t1 * PS + t0, Sy, nullptr, 0.0, 0.0, 0.0);
  __syncthreads();
  // z: forward + inverse Kronecker-sum spectrum, then backward, on one line
  // (j = t1 -> mode b, i = t0 -> mode a); dropped points have lambda = +inf
  fdm_line<NQE, PS, true>(A + t1 * LS + t0, Sz, Ls + 2 * NQE, Ls[t0] + Ls[NQE + t1], lam0, lam1);
  fdm_line<NQE, PS, false>(A + t1 * LS + t0, Sz, nullptr, 0.0, 0.0, 0.0);
  __syncthreads();
  // backward y, backward x
  fdm_line<NQE, LS, false>(A + t1 * PS + t0, Sy, nullptr, 0.0, 0.0, 0.0);
  __syncthreads();
  fdm_line<NQE, 1, false>(A + t1 * PS + t0 * LS, Sx, nullptr, 0.0, 0.0, 0.0);
  __syncthreads();
  if (out_ext) {
    double* o = out + e * NQE * NQE * NQE;
    for (int q = t; q < NQE * NQE * NQE; q += NT) {
      const int i = q % NQE, j = (q / NQE) % NQE, k = q / (NQE * NQE);
      o[q] = A[k * PS + j * LS + i];
    }
  } else {
    for (int q = t; q < NQ3; q += NT) {
      const int i = q % NQ, j = (q / NQ) % NQ, k = q / NQ2;
      out[ob + q] = A[(k + 1) * PS + (j + 1) * LS + (i + 1)];
    }
  }
}

__global__ void __launch_bounds__(256)
schwarz_post_kernel(int nq, int64_t n, const double* __restrict__ src, int src_ext,
                    const double* __restrict__ W, const uint8_t* __restrict__ mask,
                    double* __restrict__ d, double* __restrict__ e, double a, double b,
                    int e_acc, const nk_cg_state* st) {
  if (st != nullptr && st->done) return;
  const int nq2 = nq * nq, nq3 = nq2 * nq, nqe = nq + 2, nqe2 = nqe * nqe;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride) {
    double z;
    if (src_ext) {
      const int64_t el = q / nq3;
      const int p = (int)(q - el * nq3);
      const int i = p % nq, j = (p / nq) % nq, k = p / nq2;
      z = __ldg(src + el * nqe2 * nqe + (int64_t)(k + 1) * nqe2 + (j + 1) * nqe + (i + 1));
    } else {
      z = __ldg(src + q);
    }
    if (W) z *= __ldg(W + q);
    if (mask && !mask[q]) z = 0.0;
    double dv = b * z;
    if (d) {
      if (a != 0.0) dv = fma(a, d[q], dv);
      d[q] = dv;
    }
    e[q] = e_acc ? e[q] + dv : dv;
  }
}

template <int NQE>
static int launch_fdm(int64_t E, const double* r, const double* sub, double* res_out,
                      const int32_t* fmap, const double* S, const double* lam, double lam0,
                      double lam1, double* out, int out_ext, const nk_cg_state* st,
                      cudaStream_t s) {
  constexpr size_t smem = sizeof(double) * (NQE * NQE * (NQE + 1) + 3 * NQE * NQE + 3 * NQE);
  static bool configured = false;
  if (!configured) {
    cudaError_t err = cudaFuncSetAttribute(fdm_kernel<NQE>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) {
      set_error("fdm: smem attribute: %s", cudaGetErrorString(err));
      return NK_ERR_CUDA;
    }
    configured = true;
  }
  fdm_kernel<NQE><<<(unsigned)E, NQE * NQE, smem, s>>>(E, r, sub, res_out, fmap, S, lam, lam0,
                                                      lam1, out, out_ext, st);
  return check_launch("fdm");
}

}  // namespace nk

using namespace nk;

extern "C" int nk_fdm(int N, int64_t nelem, const double* r, const double* sub, double* res_out,
                      const int32_t* fmap, const double* Smat, const double* lam, double lam0,
                      double lam1, double* out, int out_ext, const nk_cg_state* st,
                      nk_stream_t stream) {
  if (N < NK_MIN_ORDER || N > NK_MAX_ORDER) {
    set_error("fdm: order %d outside [%d, %d]", N, NK_MIN_ORDER, NK_MAX_ORDER);
    return NK_ERR_UNSUPPORTED;
  }
  if (nelem < 0 || nelem > 0x7fffffffLL ||
      (nelem > 0 && (!r || !fmap || !Smat || !lam || !out))) {
    set_error("fdm: invalid arguments (nelem=%lld)", (long long)nelem);
    return NK_ERR_INVALID;
  }
  if (nelem == 0) return NK_OK;
  cudaStream_t s = S(stream);
  switch (N + 3) {
#define NK_FDM_CASE(Q) \
  case Q:              \
    return launch_fdm<Q>(nelem, r, sub, res_out, fmap, Smat, lam, lam0, lam1, out, out_ext, st, s);
    NK_FDM_CASE(4) NK_FDM_CASE(5) NK_FDM_CASE(6) NK_FDM_CASE(7) NK_FDM_CASE(8) NK_FDM_CASE(9)
    NK_FDM_CASE(10) NK_FDM_CASE(11) NK_FDM_CASE(12) NK_FDM_CASE(13) NK_FDM_CASE(14)
    NK_FDM_CASE(15) NK_FDM_CASE(16) NK_FDM_CASE(17) NK_FDM_CASE(18)
#undef NK_FDM_CASE
    default: break;
  }
  set_error("fdm: order %d not instantiated", N);
  return NK_ERR_UNSUPPORTED;
}

extern "C" int nk_schwarz_post(int N, int64_t nelem, const double* src, int src_ext,
                               const double* W, const uint8_t* mask, double* d, double* e,
                               double a, double b, int e_acc, const nk_cg_state* st,
                               nk_stream_t stream) {
  if (N < NK_MIN_ORDER || N > NK_MAX_ORDER || nelem < 0 || (nelem > 0 && (!src || !e))) {
    set_error("schwarz_post: invalid arguments (N=%d nelem=%lld)", N, (long long)nelem);
    return NK_ERR_INVALID;
  }
  const int nq = N + 1;
  const int64_t n = nelem * nq * nq * nq;
  if (n == 0) return NK_OK;
  int64_t g = (n + 255) / 256;
  if (g > 8 * 148) g = 8 * 148;
  schwarz_post_kernel<<<(unsigned)g, 256, 0, S(stream)>>>(nq, n, src, src_ext, W, mask, d, e, a,
                                                          b, e_acc, st);
  return check_launch("schwarz_post");
}
