// Shared helpers for libnekb200 (error state, launch checks, reductions).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <cstdarg>
#include <string>

#include "../../include/nekb200.h"

#define NK_MIN_ORDER 1
#define NK_MAX_ORDER 15
#define NK_GS_MAX_CLASSES 16

namespace nk {

void set_error(const char* fmt, ...);
const char* get_error();

inline cudaStream_t S(nk_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return NK_ERR_CUDA;
  }
  return NK_OK;
}

// Threads per block for the streaming PCG kernels and the fixed number of
// partial sums they produce.  The partial count does not depend on the GPU so
// reductions are bitwise reproducible across devices.
constexpr int kVecThreads = 256;
constexpr int kVecMaxBlocks = 1184;  // 8 x 148 SMs

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-order block sum of NV values per thread; result valid in thread 0.
// `red` must hold NV * 32 doubles.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = warp_sum(v[q]);
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) red[q * 32 + wid] = v[q];
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double t = lane < nw ? red[q * 32 + lane] : 0.0;
      v[q] = warp_sum(t);
    }
  }
  __syncthreads();
}

// Last-block-done: returns true in exactly one block (the last to finish),
// after all other blocks' prior global writes are visible.  Resets the
// ticket so the next launch (or graph replay) starts from zero.
__device__ __forceinline__ bool last_block(uint32_t* ticket, uint32_t nblocks) {
  __shared__ bool is_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    uint32_t t = atomicAdd(ticket, 1u);
    is_last = (t == nblocks - 1);
    if (is_last) *ticket = 0u;
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}

// Fixed-order sum of partials[0..n) by one block; valid in thread 0.
template <int NV>
__device__ __forceinline__ void reduce_partials(const double* partials, int64_t n,
                                                int64_t stride, double (&out)[NV], double* red) {
#pragma unroll
  for (int q = 0; q < NV; ++q) out[q] = 0.0;
  for (int64_t b = threadIdx.x; b < n; b += blockDim.x) {
#pragma unroll
    for (int q = 0; q < NV; ++q) out[q] += __ldcg(partials + q * stride + b);
  }
  block_sum<NV>(out, red);
}

}  // namespace nk
