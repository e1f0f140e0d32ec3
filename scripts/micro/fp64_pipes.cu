// FP64 pipe micro-benchmark on B200: DFMA vs DMMA.8x8x4 peak issue rate.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_pipes.cu -o fp64_pipes
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma_loop(double* out, int iters) {
  double d[8][2];
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0;
  const double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 8 * 256 * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096, blocks = 148 * 8, threads = 256;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(a);
    dfma_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double fl = 2.0 * 8 * iters * (double)blocks * threads;
    if (rep) printf("{\"pipe\": \"DFMA\", \"tflops\": %.2f}\n", fl / ms / 1e9);
    cudaEventRecord(a);
    dmma_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    fl = 2.0 * 8 * 8 * 4 * 8 * iters * (double)blocks * (threads / 32);
    if (rep) printf("{\"pipe\": \"DMMA.8x8x4\", \"tflops\": %.2f}\n", fl / ms / 1e9);
  }
  return 0;
}
