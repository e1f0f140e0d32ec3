// p-multigrid building blocks (SPEC.md:489-527,
// PAPER.md:274-313): order-to-order tensor-product transfer, the fused
// Chebyshev-Jacobi vector step and the dense coarse matvec.  The V-cycle is
// sequenced on the host (paper_2104_05829_b200/multigrid.py) from these plus
// nk_bk5 + gs at every level; every kernel takes the PCG state so a graph
// replay after convergence does no work.
//
// All three are HBM-streaming kernels:
//   nk_interp3   restriction reads in, sub, wt (24 B per fine point) and writes
//                1/8-ish of that; prolongation reads the coarse field, reads +
//                writes the fine one (17 B per fine point with the mask).
//   nk_cheb_step 32-56 B per point.
//   nk_dense_matvec  8 n^2 B (the explicit inverse of the coarse operator);
//   nk_dense_matvec32 the same with the inverse stored in FP32 (4 n^2 B).
#include "common.cuh"

namespace nk {

static unsigned grid_stride(int64_t n, int threads, int64_t cap) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

struct TransferM {
  double m[16 * 16];  // row-major no x ni
};

// One element per CTA.  v (ni^3) -> t1 (ni^2 no) -> t2 (ni no^2) -> out (no^3):
// contraction order i, j, k (oracle/pmg.py:_interp3).
__global__ void __launch_bounds__(256)
interp3_kernel(int ni, int no, const __grid_constant__ TransferM M, const double* __restrict__ in,
               const double* __restrict__ sub, const double* __restrict__ wt,
               const uint8_t* __restrict__ mask, double* __restrict__ out, int accumulate,
               const nk_cg_state* st) {
  if (st != nullptr && st->done) return;
  extern __shared__ __align__(16) double sm[];
  const int ni2 = ni * ni, ni3 = ni2 * ni, no2 = no * no, no3 = no2 * no;
  double* v = sm;
  double* t1 = v + ni3;
  double* t2 = t1 + ni2 * no;
  const int64_t e = blockIdx.x;
  const int64_t ib = e * ni3, ob = e * no3;
  for (int q = threadIdx.x; q < ni3; q += blockDim.x) {
    double x = __ldg(in + ib + q);
    if (sub) x -= __ldg(sub + ib + q);
    if (wt) x *= __ldg(wt + ib + q);
    v[q] = x;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < ni2 * no; q += blockDim.x) {  // t1[k][j][a]
    const int a = q % no, kj = q / no;
    const double* row = M.m + a * ni;
    const double* src = v + kj * ni;
    double s = 0.0;
    for (int i = 0; i < ni; ++i) s = fma(row[i], src[i], s);
    t1[q] = s;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < ni * no2; q += blockDim.x) {  // t2[k][b][a]
    const int a = q % no, b = (q / no) % no, k = q / no2;
    const double* row = M.m + b * ni;
    const double* src = t1 + k * ni * no + a;
    double s = 0.0;
    for (int j = 0; j < ni; ++j) s = fma(row[j], src[j * no], s);
    t2[q] = s;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < no3; q += blockDim.x) {  // out[c][b][a]
    const int ba = q % no2, c = q / no2;
    const double* row = M.m + c * ni;
    const double* src = t2 + ba;
    double s = 0.0;
    for (int k = 0; k < ni; ++k) s = fma(row[k], src[k * no2], s);
    if (mask && !mask[ob + q]) s = 0.0;
    out[ob + q] = accumulate ? out[ob + q] + s : s;
  }
}

__global__ void __launch_bounds__(256)
cheb_step_kernel(int64_t n, const double* __restrict__ r, const double* __restrict__ Aq,
                 const double* __restrict__ invD, double* __restrict__ res_out,
                 double* __restrict__ d, double* __restrict__ e, double a, double b, int e_acc,
                 const nk_cg_state* st) {
  if (st != nullptr && st->done) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride) {
    double rv = r[q];
    if (Aq) rv -= __ldg(Aq + q);
    if (res_out) res_out[q] = rv;
    const double z = __ldg(invD + q) * rv;
    const double dv = a != 0.0 ? a * d[q] + b * z : b * z;
    d[q] = dv;
    e[q] = e_acc ? e[q] + dv : dv;
  }
}

// y = A x, one warp per row, fixed lane-strided order (deterministic).
__global__ void __launch_bounds__(256)
dense_matvec_kernel(int64_t n, const double* __restrict__ A, const double* __restrict__ x,
                    double* __restrict__ y, const nk_cg_state* st) {
  if (st != nullptr && st->done) return;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < n;
       row += warps) {
    const double* a = A + row * n;
    double s = 0.0;
    if ((n & 1) == 0) {
      // four independent 16-B row loads in flight per lane (the matrix is
      // streamed once per V-cycle: memory-level parallelism is the limiter);
      // fixed association (s0 + s1) + (s2 + s3) keeps the sum deterministic
      const double2* a2 = reinterpret_cast<const double2*>(a);
      const double2* x2 = reinterpret_cast<const double2*>(x);
      const int64_t n2 = n >> 1;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int64_t c = lane;
      for (; c + 96 < n2; c += 128) {
        const double2 a0 = __ldcs(a2 + c), a1 = __ldcs(a2 + c + 32);
        const double2 a2v = __ldcs(a2 + c + 64), a3 = __ldcs(a2 + c + 96);
        const double2 x0 = __ldg(x2 + c), x1 = __ldg(x2 + c + 32);
        const double2 x2v = __ldg(x2 + c + 64), x3 = __ldg(x2 + c + 96);
        s0 = fma(a0.y, x0.y, fma(a0.x, x0.x, s0));
        s1 = fma(a1.y, x1.y, fma(a1.x, x1.x, s1));
        s2 = fma(a2v.y, x2v.y, fma(a2v.x, x2v.x, s2));
        s3 = fma(a3.y, x3.y, fma(a3.x, x3.x, s3));
      }
      for (; c < n2; c += 32) {
        const double2 av = __ldcs(a2 + c);
        const double2 xv = __ldg(x2 + c);
        s0 = fma(av.y, xv.y, fma(av.x, xv.x, s0));
      }
      s = (s0 + s1) + (s2 + s3);
    } else {
      for (int64_t c = lane; c < n; c += 32) s = fma(__ldcs(a + c), __ldg(x + c), s);
    }
    s = warp_sum(s);
    if (lane == 0) y[row] = s;
  }
}

// y = A x with A stored in FP32 (the 32-bit smoothing mode's coarse inverse:
// half the bytes of the streamed n^2 matrix), products and sums in FP64.
// Same warp-per-row structure, four 16-B (4-float) loads in flight per lane.
__global__ void __launch_bounds__(256)
dense_matvec32_kernel(int64_t n, int64_t lda, const float* __restrict__ A,
                      const double* __restrict__ x, double* __restrict__ y,
                      const nk_cg_state* st) {
  if (st != nullptr && st->done) return;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < n;
       row += warps) {
    const float* a = A + row * lda;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int64_t c = 0;
    {   // lda: a multiple of 4, columns n..lda-1 of A zero, x[n..lda) finite
      const float4* a4 = reinterpret_cast<const float4*>(a);
      const double2* x2 = reinterpret_cast<const double2*>(x);
      const int64_t n4 = lda >> 2;
      int64_t q = lane;
      for (; q + 96 < n4; q += 128) {
        float4 av[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) av[u] = __ldcs(a4 + q + 32 * u);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double2 xa = __ldg(x2 + 2 * (q + 32 * u)), xb = __ldg(x2 + 2 * (q + 32 * u) + 1);
          double& acc = u == 0 ? s0 : (u == 1 ? s1 : (u == 2 ? s2 : s3));
          acc = fma((double)av[u].w, xb.y, fma((double)av[u].z, xb.x,
                fma((double)av[u].y, xa.y, fma((double)av[u].x, xa.x, acc))));
        }
      }
      for (; q < n4; q += 32) {
        const float4 av = __ldcs(a4 + q);
        const double2 xa = __ldg(x2 + 2 * q), xb = __ldg(x2 + 2 * q + 1);
        s0 = fma((double)av.w, xb.y, fma((double)av.z, xb.x,
             fma((double)av.y, xa.y, fma((double)av.x, xa.x, s0))));
      }
      c = n;
    }
    for (int64_t cc = c + lane; cc < n; cc += 32) s0 = fma((double)__ldcs(a + cc), __ldg(x + cc), s0);
    double s = warp_sum((s0 + s1) + (s2 + s3));
    if (lane == 0) y[row] = s;
  }
}

// Specialised transfer for the order pairs the p-multigrid uses (pmg_orders:
// N+1 <-> N/2+1 and N/2+1 <-> 2): one element per CTA, max(NI, NO)^2 threads,
// each contraction a per-thread line in registers with the transfer matrix in
// the constant bank (compile-time indices), odd-pitched shared rows.  The
// generic kernel above runs every other pair.
template <int NI, int NO>
struct TransferMT {
  double m[NO * NI];
};

template <int NI, int NO>
__global__ void __launch_bounds__((NI > NO ? NI * NI : NO * NO))
interp3_fast(const __grid_constant__ TransferMT<NI, NO> M, const double* __restrict__ in,
             const double* __restrict__ sub, const double* __restrict__ wt,
             const uint8_t* __restrict__ mask, double* __restrict__ out, int accumulate,
             const nk_cg_state* st) {
  if (st != nullptr && st->done) return;
  constexpr int TH = NI > NO ? NI * NI : NO * NO;
  constexpr int PI = NI | 1, PO = NO | 1;         // odd row pitches
  constexpr int SA = NI * NI * PI > NI * NO * PO ? NI * NI * PI : NI * NO * PO;
  extern __shared__ double ismem[];
  double* v = ismem;                               // [k][j][i]
  double* t2 = ismem;                              // [k][b][a]  (v is dead by then)
  double* t1 = ismem + SA;                         // [k][j][a]
  const int64_t e = blockIdx.x;
  const int t = threadIdx.x;
  const int64_t ib = e * NI * NI * NI, ob = e * NO * NO * NO;
  for (int q = t; q < NI * NI * NI; q += TH) {
    double x = __ldg(in + ib + q);
    if (sub) x -= __ldg(sub + ib + q);
    if (wt) x *= __ldg(wt + ib + q);
    v[(q / NI) * PI + q % NI] = x;
  }
  __syncthreads();
  if (t < NI * NI) {                               // i -> a on line (k, j) = t
    double x[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) x[i] = v[t * PI + i];
#pragma unroll
    for (int a = 0; a < NO; ++a) {
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i < NI; ++i) acc = fma(M.m[a * NI + i], x[i], acc);
      t1[t * PO + a] = acc;
    }
  }
  __syncthreads();
  if (t < NI * NO) {                               // j -> b on line (k, a)
    const int k = t / NO, a = t % NO;
    double x[NI];
#pragma unroll
    for (int j = 0; j < NI; ++j) x[j] = t1[(k * NI + j) * PO + a];
#pragma unroll
    for (int b = 0; b < NO; ++b) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < NI; ++j) acc = fma(M.m[b * NI + j], x[j], acc);
      t2[(k * NO + b) * PO + a] = acc;
    }
  }
  __syncthreads();
  if (t < NO * NO) {                               // k -> c on line (b, a)
    const int b = t / NO, a = t % NO;
    double x[NI];
#pragma unroll
    for (int k = 0; k < NI; ++k) x[k] = t2[(k * NO + b) * PO + a];
#pragma unroll
    for (int c = 0; c < NO; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < NI; ++k) acc = fma(M.m[c * NI + k], x[k], acc);
      const int64_t o = ob + (c * NO + b) * NO + a;
      if (mask && !mask[o]) acc = 0.0;
      out[o] = accumulate ? out[o] + acc : acc;
    }
  }
}

template <int NI, int NO>
static int launch_interp_fast(int64_t nelem, const double* Mh, const double* in,
                              const double* sub, const double* wt, const uint8_t* mask,
                              double* out, int accumulate, const nk_cg_state* st,
                              cudaStream_t s) {
  TransferMT<NI, NO> T;
  for (int q = 0; q < NO * NI; ++q) T.m[q] = Mh[q];
  constexpr int TH = NI > NO ? NI * NI : NO * NO;
  constexpr int PI = NI | 1, PO = NO | 1;
  constexpr int SA = NI * NI * PI > NI * NO * PO ? NI * NI * PI : NI * NO * PO;
  constexpr size_t smem = sizeof(double) * (SA + NI * NI * PO);
  static bool configured = false;
  if (!configured) {
    cudaError_t err = cudaFuncSetAttribute(interp3_fast<NI, NO>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) {
      set_error("interp3: smem attribute: %s", cudaGetErrorString(err));
      return NK_ERR_CUDA;
    }
    configured = true;
  }
  interp3_fast<NI, NO><<<(unsigned)nelem, TH, smem, s>>>(T, in, sub, wt, mask, out, accumulate,
                                                         st);
  return check_launch("interp3_fast");
}

// the pmg_orders pairs (N = 1..15): N+1 <-> N/2+1 and N/2+1 <-> 2
#define NK_INTERP_PAIRS(X) \
  X(2, 3) X(2, 4) X(2, 5) X(2, 6) X(2, 7) X(2, 8) X(3, 2) X(3, 5) X(3, 6) X(4, 2) X(4, 7) \
  X(4, 8) X(5, 2) X(5, 3) X(5, 9) X(5, 10) X(6, 2) X(6, 3) X(6, 11) X(6, 12) X(7, 2) X(7, 4) \
  X(7, 13) X(7, 14) X(8, 2) X(8, 4) X(8, 15) X(8, 16) X(9, 5) X(10, 5) X(11, 6) X(12, 6) \
  X(13, 7) X(14, 7) X(15, 8) X(16, 8)

static int interp_fast_dispatch(int ni, int no, int64_t nelem, const double* M, const double* in,
                                const double* sub, const double* wt, const uint8_t* mask,
                                double* out, int accumulate, const nk_cg_state* st,
                                cudaStream_t s) {
#define NK_IP_CASE(A, B)                                                                   \
  if (ni == A && no == B)                                                                  \
    return launch_interp_fast<A, B>(nelem, M, in, sub, wt, mask, out, accumulate, st, s);
  NK_INTERP_PAIRS(NK_IP_CASE)
#undef NK_IP_CASE
  return -1;
}

}  // namespace nk

using namespace nk;

extern "C" int nk_interp3(int ni, int no, int64_t nelem, const double* M, const double* in,
                          const double* sub, const double* wt, const uint8_t* mask, double* out,
                          int accumulate, const nk_cg_state* st, nk_stream_t stream) {
  if (ni < 2 || ni > 16 || no < 2 || no > 16 || nelem < 0 || !M ||
      (nelem > 0 && (!in || !out))) {
    set_error("interp3: invalid arguments (ni=%d no=%d nelem=%lld)", ni, no, (long long)nelem);
    return NK_ERR_INVALID;
  }
  if (nelem == 0) return NK_OK;
  if (nelem > 0x7fffffffLL) {
    set_error("interp3: too many elements");
    return NK_ERR_INVALID;
  }
  {
    const int rc = interp_fast_dispatch(ni, no, nelem, M, in, sub, wt, mask, out, accumulate, st,
                                        S(stream));
    if (rc >= 0) return rc;
  }
  TransferM T;
  for (int q = 0; q < no * ni; ++q) T.m[q] = M[q];
  const size_t smem = sizeof(double) * (size_t)(ni * ni * ni + ni * ni * no + ni * no * no);
  static bool configured = false;
  if (!configured) {
    cudaError_t err = cudaFuncSetAttribute(interp3_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(sizeof(double) * 3 * 4096));
    if (err != cudaSuccess) {
      set_error("interp3: smem attribute: %s", cudaGetErrorString(err));
      return NK_ERR_CUDA;
    }
    configured = true;
  }
  interp3_kernel<<<(unsigned)nelem, 256, smem, S(stream)>>>(ni, no, T, in, sub, wt, mask, out,
                                                            accumulate, st);
  return check_launch("interp3");
}

extern "C" int nk_cheb_step(int64_t n, const double* r, const double* Aq, const double* invD,
                            double* res_out, double* d, double* e, double a, double b, int e_acc,
                            const nk_cg_state* st, nk_stream_t stream) {
  if (n < 0 || (n > 0 && (!r || !invD || !d || !e))) {
    set_error("cheb_step: invalid arguments");
    return NK_ERR_INVALID;
  }
  if (n == 0) return NK_OK;
  cheb_step_kernel<<<grid_stride(n, 256, 8 * 148), 256, 0, S(stream)>>>(n, r, Aq, invD, res_out, d,
                                                                         e, a, b, e_acc, st);
  return check_launch("cheb_step");
}

extern "C" int nk_dense_matvec(int64_t n, const double* A, const double* x, double* y,
                               const nk_cg_state* st, nk_stream_t stream) {
  if (n < 0 || (n > 0 && (!A || !x || !y))) {
    set_error("dense_matvec: invalid arguments");
    return NK_ERR_INVALID;
  }
  if (n == 0) return NK_OK;
  dense_matvec_kernel<<<grid_stride(n, 8, 16 * 148), 256, 0, S(stream)>>>(n, A, x, y, st);
  return check_launch("dense_matvec");
}

extern "C" int nk_dense_matvec32(int64_t n, int64_t lda, const float* A, const double* x,
                                 double* y, const nk_cg_state* st, nk_stream_t stream) {
  if (n < 0 || lda < n || (lda & 3) || (n > 0 && (!A || !x || !y))) {
    set_error("dense_matvec32: invalid arguments (lda >= n, a multiple of 4)");
    return NK_ERR_INVALID;
  }
  if (n > 0 && ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(x)) & 15)) {
    set_error("dense_matvec32: A and x must be 16-byte aligned");
    return NK_ERR_INVALID;
  }
  if (n == 0) return NK_OK;
  dense_matvec32_kernel<<<grid_stride(n, 8, 16 * 148), 256, 0, S(stream)>>>(n, lda, A, x, y,
                                                                            st);
  return check_launch("dense_matvec32");
}
