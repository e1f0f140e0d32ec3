// Projection-based initial guesses (SPEC.md:529-537
// ProjectionSpace / project_guess / update): the
// A-orthonormal space of prior solutions is k <= NK_PROJ_MAX stored vectors
// X[q] (and A X[q]) of n local points each.  Projection and the
// Gram-Schmidt update are two HBM-streaming primitives over that block:
//
//   nk_multi_wdot   out[q] = sum_i wt_i X[q]_i y_i   for q < k, one pass over
//                   y (and the k rows of X): (k + 2) * 8 B per point.
//                   Fixed-order two-stage reduction (bitwise reproducible).
//   nk_multi_axpy   y_out = y_in + scale * sum_q c[q] V[q] with c in device
//                   memory, so project -> solve -> update never syncs the
//                   host except for the degeneracy test of the update.
//   nk_vscale       y = x * s[0]^(-1/2) (A-normalisation by a device scalar).
#include "common.cuh"

namespace nk {

constexpr int kProjMax = NK_PROJ_MAX;

static int64_t proj_grid(int64_t n) {
  int64_t g = (n + kVecThreads - 1) / kVecThreads;
  if (g < 1) g = 1;
  if (g > kVecMaxBlocks) g = kVecMaxBlocks;
  return g;
}

template <int K>
__global__ void __launch_bounds__(kVecThreads)
multi_wdot_partial(int64_t n, int k, const double* __restrict__ X, int64_t ldx,
                   const double* __restrict__ y, const double* __restrict__ wt,
                   double* __restrict__ partials) {
  __shared__ double red[K * 32];
  double v[K];
#pragma unroll
  for (int q = 0; q < K; ++q) v[q] = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double t = wt ? __ldg(wt + i) * __ldg(y + i) : __ldg(y + i);
#pragma unroll
    for (int q = 0; q < K; ++q)
      if (q < k) v[q] = fma(__ldg(X + q * ldx + i), t, v[q]);
  }
  block_sum<K>(v, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < K; ++q) partials[q * kVecMaxBlocks + blockIdx.x] = v[q];
  }
}

__global__ void __launch_bounds__(kVecThreads)
multi_wdot_final(int k, int64_t nb, const double* __restrict__ partials, double* out) {
  __shared__ double red[32];
  // one row per pass; k <= 16 passes of a fixed-order block sum
  for (int q = 0; q < k; ++q) {
    double s[1];
    reduce_partials<1>(partials + q * kVecMaxBlocks, nb, 0, s, red);
    if (threadIdx.x == 0) out[q] = s[0];
  }
}

__global__ void __launch_bounds__(kVecThreads)
multi_axpy_kernel(int64_t n, int k, const double* __restrict__ c, double scale,
                  const double* __restrict__ V, int64_t ldv, const double* yin,
                  double* yout) {
  __shared__ double cs[kProjMax];
  if (threadIdx.x < k) cs[threadIdx.x] = scale * c[threadIdx.x];
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double s = 0.0;
    for (int q = 0; q < k; ++q) s = fma(cs[q], __ldg(V + q * ldv + i), s);
    yout[i] = yin ? yin[i] + s : s;
  }
}

__global__ void __launch_bounds__(kVecThreads)
vscale_kernel(int64_t n, const double* __restrict__ x, double* __restrict__ y,
              const double* __restrict__ s) {
  const double f = rsqrt(s[0]);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    y[i] = x[i] * f;
}

template <int K>
static void launch_partial(int64_t g, cudaStream_t s, int64_t n, int k, const double* X,
                           int64_t ldx, const double* y, const double* wt, double* partials) {
  multi_wdot_partial<K><<<(unsigned)g, kVecThreads, 0, s>>>(n, k, X, ldx, y, wt, partials);
}

}  // namespace nk

using namespace nk;

extern "C" int64_t nk_multi_wdot_partials_len(void) {
  return (int64_t)kProjMax * kVecMaxBlocks;
}

extern "C" int nk_multi_wdot(int64_t n, int k, const double* X, int64_t ldx, const double* y,
                             const double* wt, double* out, double* partials,
                             nk_stream_t stream) {
  if (n < 0 || k < 1 || k > kProjMax || !X || !y || !out || !partials || (k > 1 && ldx < n)) {
    set_error("multi_wdot: invalid arguments (n=%lld k=%d)", (long long)n, k);
    return NK_ERR_INVALID;
  }
  cudaStream_t s = S(stream);
  const int64_t g = proj_grid(n);
  // k rounded up to a compiled register width; rows >= k are predicated off
  if (k == 1) launch_partial<1>(g, s, n, k, X, ldx, y, wt, partials);
  else if (k == 2) launch_partial<2>(g, s, n, k, X, ldx, y, wt, partials);
  else if (k <= 4) launch_partial<4>(g, s, n, k, X, ldx, y, wt, partials);
  else if (k <= 8) launch_partial<8>(g, s, n, k, X, ldx, y, wt, partials);
  else launch_partial<kProjMax>(g, s, n, k, X, ldx, y, wt, partials);
  int rc = check_launch("multi_wdot_partial");
  if (rc) return rc;
  multi_wdot_final<<<1, kVecThreads, 0, s>>>(k, g, partials, out);
  return check_launch("multi_wdot_final");
}

extern "C" int nk_multi_axpy(int64_t n, int k, const double* c, double scale, const double* V,
                             int64_t ldv, const double* yin, double* yout, nk_stream_t stream) {
  if (n < 0 || k < 0 || k > kProjMax || !yout || (k > 1 && ldv < n) || (k > 0 && (!c || !V))) {
    set_error("multi_axpy: invalid arguments (n=%lld k=%d)", (long long)n, k);
    return NK_ERR_INVALID;
  }
  if (n == 0) return NK_OK;
  multi_axpy_kernel<<<(unsigned)proj_grid(n), kVecThreads, 0, S(stream)>>>(n, k, c, scale, V,
                                                                          ldv, yin, yout);
  return check_launch("multi_axpy");
}

extern "C" int nk_vscale(int64_t n, const double* x, double* y, const double* s,
                         nk_stream_t stream) {
  if (n < 0 || !x || !y || !s) {
    set_error("vscale: invalid arguments");
    return NK_ERR_INVALID;
  }
  if (n == 0) return NK_OK;
  vscale_kernel<<<(unsigned)proj_grid(n), kVecThreads, 0, S(stream)>>>(n, x, y, s);
  return check_launch("vscale");
}
