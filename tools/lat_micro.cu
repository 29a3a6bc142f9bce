// Latency micro-benchmarks for the latency-bound solver chain (B200):
// dependent DFMA, rsqrt(double), DMMA m8n8k4, __syncthreads (256 thr), shfl.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__global__ void k(double* out, long long* t, int n) {
    double x = out[threadIdx.x] + 1.0, y = 1.0001;
    long long t0, t1;
    __syncthreads();
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, y, 0.5);
    t1 = clock64();
    if (threadIdx.x == 0) t[0] = (t1 - t0) / n;
    out[threadIdx.x] = x;
    x = 2.0 + threadIdx.x;
    __syncthreads();
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = rsqrt(x) + 1.5;
    t1 = clock64();
    if (threadIdx.x == 0) t[1] = (t1 - t0) / n;
    out[threadIdx.x] += x;
    x = 2.0 + threadIdx.x;
    __syncthreads();
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = sqrt(x) + 1.5;
    t1 = clock64();
    if (threadIdx.x == 0) t[2] = (t1 - t0) / n;
    out[threadIdx.x] += x;
    double c0 = 0, c1 = 0;
    __syncthreads();
    t0 = clock64();
    for (int i = 0; i < n; ++i) dmma(c0, c1, x, y);
    t1 = clock64();
    if (threadIdx.x == 0) t[3] = (t1 - t0) / n;
    out[threadIdx.x] += c0 + c1;
    __syncthreads();
    t0 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    t1 = clock64();
    if (threadIdx.x == 0) t[4] = (t1 - t0) / n;
    x = threadIdx.x;
    __syncthreads();
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1.0;
    t1 = clock64();
    if (threadIdx.x == 0) t[5] = (t1 - t0) / n;
    out[threadIdx.x] += x;
    __shared__ double sm[256];
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    int idx = threadIdx.x;
    t0 = clock64();
    for (int i = 0; i < n; ++i) { x = sm[idx]; idx = ((int)x + 1) & 255; }
    t1 = clock64();
    if (threadIdx.x == 0) t[6] = (t1 - t0) / n;
    out[threadIdx.x] += x;
    x = 1.0 + threadIdx.x;
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = 1.0 / x + 0.5;
    t1 = clock64();
    if (threadIdx.x == 0) t[7] = (t1 - t0) / n;
    out[threadIdx.x] += x;
}
int main() {
    double* o; long long* t; cudaMalloc(&o, 8 * 256); cudaMalloc(&t, 8 * 16);
    cudaMemset(o, 0, 8 * 256);
    for (int thr : {32, 256}) {
        k<<<1, thr>>>(o, t, 1000);
        long long h[16];
        cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
        printf("threads=%d cycles: dfma %lld rsqrt %lld sqrt %lld dmma(dep) %lld syncthreads %lld shfl+add %lld lds(dep) %lld div %lld\n",
               thr, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
