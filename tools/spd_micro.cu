// Micro-benchmark + correctness check of the 64x64 diagonal-block
// factorisation used on the solver's critical path (spd.cu potrf_inv64).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        tools/spd_micro.cu -o tools/spd_micro
#include <cstring>
#include "../paper_2408_01654_b200/csrc/spd.cu"

namespace dpv {
std::atomic<int64_t> g_launches{0};
bool g_timing = false;
void set_error(const std::string&) {}
void clear_error() {}
void timer_push(const char*, cudaStream_t, bool) {}
int sm_count() { return 148; }
}  // namespace dpv

using namespace dpv;

__global__ void k_bench(const double* A, double* L, double* Xo, long long* cyc, int reps) {
    extern __shared__ double sm[];
    double* D = sm;
    double* X = sm + kT * kLD;
    double* Y = sm + 2 * kT * kLD;
    double* W = Y + 8 * 64;
    __shared__ int bad;
    long long total = 0;
    for (int r = 0; r < reps; ++r) {
        for (int x = threadIdx.x; x < 64 * 64; x += kThreads) D[(x >> 6) * kLD + (x & 63)] = A[x];
        if (threadIdx.x == 0) bad = -1;
        __syncthreads();
        const long long t0 = clock64();
        potrf_inv64(D, X, Y, W, &bad);
        const long long t1 = clock64();
        total += t1 - t0;
    }
    for (int x = threadIdx.x; x < 64 * 64; x += kThreads) {
        L[x] = D[(x >> 6) * kLD + (x & 63)];
        Xo[x] = X[(x >> 6) * kLD + (x & 63)];
    }
    if (threadIdx.x == 0) { cyc[0] = total / reps; cyc[1] = bad; }
}

__global__ void k_fb8(const double* A, long long* cyc, int reps) {
    extern __shared__ double sm[];
    double* D = sm;
    double* Y = sm + kT * kLD;
    __shared__ int bad;
    long long tot = 0;
    for (int r = 0; r < reps; ++r) {
        for (int x = threadIdx.x; x < 64 * 64; x += 32) D[(x >> 6) * kLD + (x & 63)] = A[x];
        bad = -1;
        __syncwarp();
        long long t0 = clock64();
        factor_block8(D, Y, r & 7, &bad);
        long long t1 = clock64();
        tot += t1 - t0;
    }
    if (threadIdx.x == 0) cyc[0] = tot / reps;
}

__global__ void k_bar(long long* cyc, int reps) {
    __shared__ double x[256];
    x[threadIdx.x] = threadIdx.x;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        __syncthreads();
        x[threadIdx.x] += x[(threadIdx.x + 1) & 255];
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
}

int main() {
    std::vector<double> A(64 * 64), M(64 * 64);
    srand(1);
    for (auto& v : M) v = (rand() / (double)RAND_MAX) - 0.5;
    for (int i = 0; i < 64; ++i)
        for (int j = 0; j < 64; ++j) {
            double s = 0;
            for (int k = 0; k < 64; ++k) s += M[i * 64 + k] * M[j * 64 + k];
            A[i * 64 + j] = s + (i == j ? 64.0 : 0.0);
        }
    double *dA, *dL, *dX;
    long long* dc;
    cudaMalloc(&dA, 8 * 4096); cudaMalloc(&dL, 8 * 4096); cudaMalloc(&dX, 8 * 4096);
    cudaMalloc(&dc, 16);
    cudaMemcpy(dA, A.data(), 8 * 4096, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    k_bench<<<1, kThreads, kSmemBytes>>>(dA, dL, dX, dc, getenv("REPS") ? atoi(getenv("REPS")) : 20);
    std::vector<double> L(4096), X(4096);
    long long c[2];
    cudaMemcpy(L.data(), dL, 8 * 4096, cudaMemcpyDeviceToHost);
    cudaMemcpy(X.data(), dX, 8 * 4096, cudaMemcpyDeviceToHost);
    cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost);
    double e1 = 0, e2 = 0;
    for (int i = 0; i < 64; ++i)
        for (int j = 0; j <= i; ++j) {
            double s = 0, t = 0;
            for (int k = 0; k <= j; ++k) s += L[i * 64 + k] * L[j * 64 + k];
            for (int k = j; k <= i; ++k) t += X[i * 64 + k] * L[k * 64 + j];
            e1 = fmax(e1, fabs(s - A[i * 64 + j]));
            e2 = fmax(e2, fabs(t - (i == j ? 1.0 : 0.0)));
        }
    {
        cudaFuncSetAttribute(k_fb8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
        k_fb8<<<1, 32, kSmemBytes>>>(dA, dc, 64);
        long long f; cudaMemcpy(&f, dc, 8, cudaMemcpyDeviceToHost);
        k_bar<<<1, 256>>>(dc, 1000);
        long long b; cudaMemcpy(&b, dc, 8, cudaMemcpyDeviceToHost);
        printf("factor_block8 (1 warp): %lld cycles; barrier+lds/sts step (256 thr): %lld cycles\n", f, b);
    }
    unsigned long long hl = 0, hx = 0;
    for (int x = 0; x < 4096; ++x) {
        unsigned long long u, v;
        memcpy(&u, &L[x], 8);
        memcpy(&v, &X[x], 8);
        hl = hl * 1000003ull ^ u;
        hx = hx * 1000003ull ^ v;
    }
    printf("bits: L %016llx X %016llx\n", hl, hx);
    printf("potrf_inv64: %lld cycles (%.2f us @1.965GHz), bad=%lld, |LL^T-A|=%.2e |XL-I|=%.2e  %s\n",
           c[0], c[0] / 1965.0, c[1], e1, e2, cudaGetErrorString(cudaDeviceSynchronize()));
}
