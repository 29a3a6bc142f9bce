// Microbenchmark: FP64 DFMA vs DMMA (mma.sync m8n8k4 f64) peak on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c0[4][2];
  for (int j = 0; j < 4; ++j) { c0[j][0] = 0; c0[j][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c0[j][0]), "+d"(c0[j][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0; for (int j = 0; j < 4; ++j) s += c0[j][0] + c0[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dmma16_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 0.5;
  double c[4][4];
  for (int j = 0; j < 4; ++j) for (int q = 0; q < 4; ++q) c[j][q] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a0), "d"(a1), "d"(b));
    }
  }
  double s = 0; for (int j = 0; j < 4; ++j) for (int q = 0; q < 4; ++q) s += c[j][q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096; float ms;
  for (int threads : {256, 512, 1024}) {
    int blocks = sms * (2048 / threads);
    dfma_kernel<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * blocks * threads * (double)iters * 16 * 8;
    printf("DFMA threads=%d  %.2f TFLOP/s\n", threads, fl / ms / 1e9);
    dmma_kernel<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0); dmma_kernel<<<blocks, threads>>>(out, iters / 4); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * (blocks * threads / 32) * (double)(iters / 4) * 16 * 4 * 256;
    printf("DMMA m8n8k4 threads=%d  %.2f TFLOP/s\n", threads, fl / ms / 1e9);
    dmma16_kernel<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0); dmma16_kernel<<<blocks, threads>>>(out, iters / 4); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * (blocks * threads / 32) * (double)(iters / 4) * 16 * 4 * 512;
    printf("DMMA m16n8k4 threads=%d  %.2f TFLOP/s\n", threads, fl / ms / 1e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
