// Isolated timing of the TMA correlation kernel at the cfg3 bench shape
// (47232 edges, 52 feature frames of 120x160x128 bf16 + the 30x40 level,
// 2 levels) for pipeline-shape experiments: compile with
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -DDPV_CORR_SMEM_KB=.. -DDPV_CORR_CTAS=.. \
//        tools/corr_micro.cu -o tools/corr_micro -lcuda
#include "../paper_2408_01654_b200/csrc/corr_tma.cu"

#include <cstdio>
#include <random>
#include <vector>

namespace dpv {
std::atomic<int64_t> g_launches{0};
bool g_timing = false;
void set_error(const std::string& m) { fprintf(stderr, "error: %s\n", m.c_str()); }
void clear_error() {}
void timer_push(const char*, cudaStream_t, bool) {}
int sm_count() { return 148; }
}  // namespace dpv

int main(int argc, char** argv) {
    const int64_t E = argc > 1 ? atol(argv[1]) : 47232;
    const int sorted = argc > 2 ? atoi(argv[2]) : 0;
    const int H = argc > 3 ? atoi(argv[3]) : 120, W = argc > 4 ? atoi(argv[4]) : 160;
    const int F = argc > 5 ? atoi(argv[5]) : 52, wide = argc > 6 ? atoi(argv[6]) : 0;
    const int C = 128, h1 = H / 4, w1 = W / 4;
    const int64_t NP = argc > 3 ? 80 : 192000;
    std::mt19937 rng(0);
    std::normal_distribution<float> nd(0.f, 1.f / sqrtf((float)C));
    auto fill = [&](std::vector<__nv_bfloat16>& v) { for (auto& x : v) x = __float2bfloat16(nd(rng)); };
    std::vector<__nv_bfloat16> f0((size_t)F * H * W * C), f1((size_t)F * h1 * w1 * C), g((size_t)NP * 9 * C);
    fill(f0); fill(f1); fill(g);
    std::vector<double> co(E * 18);
    std::vector<int32_t> ii(E), jj(E);
    std::uniform_real_distribution<double> ux(-3, W + 3), uy(-3, H + 3);
    std::uniform_int_distribution<int> up(0, NP - 1), uf(0, F - 1);
    for (int64_t e = 0; e < E; ++e) {
        const double bx = ux(rng), by = uy(rng);
        for (int c = 0; c < 9; ++c) {
            co[e * 18 + 2 * c] = bx + (c % 3);
            co[e * 18 + 2 * c + 1] = (wide && e % 97 == 5) ? 5.0 * c : by + (c / 3);
        }
        ii[e] = up(rng);
        jj[e] = uf(rng);
    }
    if (sorted) std::sort(jj.begin(), jj.end());
    void *d0, *d1, *dg, *dc, *di, *dj, *dout;
    cudaMalloc(&d0, f0.size() * 2); cudaMalloc(&d1, f1.size() * 2); cudaMalloc(&dg, g.size() * 2);
    cudaMalloc(&dc, co.size() * 8); cudaMalloc(&di, E * 4); cudaMalloc(&dj, E * 4);
    cudaMalloc(&dout, E * 2 * 441 * 4);
    cudaMemcpy(d0, f0.data(), f0.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(d1, f1.data(), f1.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dg, g.data(), g.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dc, co.data(), co.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(di, ii.data(), E * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dj, jj.data(), E * 4, cudaMemcpyHostToDevice);
    auto run = [&]() {
        return dpv::corr_tma(dg, NP, d0, d1, F, (const double*)dc, (const int32_t*)di,
                             (const int32_t*)dj, E, C, H, W, h1, w1, 2, (float*)dout, 0);
    };
    for (int r = 0; r < 3; ++r) run();
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    const int reps = 20;
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) run();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    const double bytes = E * (72.0 + 2 * 9 * 49 * 4 + 12) + (double)F * (H * W + h1 * w1) * C * 2 +
                         (double)E * 9 * C * 2;
    printf("corr SMEM_KB=%d CTAS=%d NP=%d NS=%d NG=%d: %.3f ms (%lld edges, sorted=%d) %.0f GB/s "
           "algorithmic  err=%s\n", DPV_CORR_SMEM_KB, DPV_CORR_CTAS,
           dpv::CorrCfg<2>::NP, dpv::CorrCfg<2>::NS, dpv::CorrCfg<2>::NG, ms, (long long)E, sorted, bytes / ms / 1e6,
           cudaGetErrorString(cudaDeviceSynchronize()));
}
