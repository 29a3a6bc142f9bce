// How many warps / independent accumulators does DMMA need to saturate an SM?
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[CH][2];
  for (int j = 0; j < CH; ++j) c[j][0] = c[j][1] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int j = 0; j < CH; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH> void run(int warps_per_sm, int sms, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int threads = 32 * (warps_per_sm < 32 ? warps_per_sm : 32);
  int blocks = sms * (warps_per_sm * 32 / threads);
  int iters = 4096 / CH * 16;
  k<CH><<<blocks, threads>>>(out, 16);
  cudaEventRecord(e0); k<CH><<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
  cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * (blocks * threads / 32) * (double)iters * CH * 256;
  printf("warps/SM=%2d chains=%2d  %.2f TFLOP/s\n", warps_per_sm, CH, fl / ms / 1e9);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 64 * 32);
  for (int w : {4, 8, 12, 16, 32}) { run<4>(w, sms, out); run<8>(w, sms, out); run<16>(w, sms, out); run<32>(w, sms, out); }
  return 0;
}
