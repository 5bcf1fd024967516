// Microbenchmark (not product code): FP64 throughput on B200 of DFMA (independent chains) and of
// DMMA (mma.sync.aligned.m8n8k4.row.col.f64), per SM and per GPU.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_bench fp64_bench.cu
#include <cuda_runtime.h>
#include <cstdio>

constexpr int ITERS = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void dmma_kernel(double* out, double a) {
  double A = a + threadIdx.x, B = a - threadIdx.x;
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(A), "d"(B));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int threads : {128, 256, 512, 1024}) {
    for (int k = 0; k < 2; ++k) {
      const int blocks = nsm * (threads >= 512 ? 1 : 2);
      dfma_kernel<<<blocks, threads>>>(d, 1.0000001, 1e-9);
      cudaEventRecord(e0);
      dfma_kernel<<<blocks, threads>>>(d, 1.0000001, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fma_n = (double)blocks * threads * ITERS * 8;
      if (k == 1) printf("DFMA threads/CTA %4d: %.2f TFLOP/s\n", threads, 2 * fma_n / ms / 1e9);
    }
    for (int k = 0; k < 2; ++k) {
      const int blocks = nsm * (threads >= 512 ? 1 : 2);
      dmma_kernel<<<blocks, threads>>>(d, 1.0);
      cudaEventRecord(e0);
      dmma_kernel<<<blocks, threads>>>(d, 1.0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fma_n = (double)blocks * (threads / 32) * ITERS * 4 * 256;
      if (k == 1) printf("DMMA threads/CTA %4d: %.2f TFLOP/s\n", threads, 2 * fma_n / ms / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
