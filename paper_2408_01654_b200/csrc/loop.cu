// Proximity loop-closure detection on the device (
// restates pkg/src/patchslam/loop.py:64-85).  Every candidate pair
// (old, recent) with recent - old >= gap is one thread (enumerated in the
// reference's insertion order: recent ascending, then old ascending); the
// centre distance is evaluated exactly as numpy's norm (no FMA contraction:
// sqrt((dx*dx + dy*dy) + dz*dz)), hits are compacted and stably radix-sorted
// by distance, so the output order is the reference's bit for bit.
#include <cub/cub.cuh>

#include <cmath>

#include "problem.cuh"

namespace dpv {
namespace {

__device__ __forceinline__ void decode(int64_t q, int64_t& r, int64_t& o) {
    // q -> (r, o) with r(r+1)/2 <= q < (r+1)(r+2)/2, o = q - r(r+1)/2
    int64_t x = (int64_t)((sqrt(8.0 * (double)q + 1.0) - 1.0) * 0.5);
    while (x * (x + 1) / 2 > q) --x;
    while ((x + 1) * (x + 2) / 2 <= q) ++x;
    r = x;
    o = q - x * (x + 1) / 2;
}

__global__ void k_detect(int64_t T, int64_t gap, const double* __restrict__ c, double thr,
                         double* dist, int64_t* idx, uint8_t* flag) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < T;
         q += (int64_t)gridDim.x * blockDim.x) {
        int64_t r, o;
        decode(q, r, o);
        const int64_t recent = gap + r, old = o;
        const double dx = __dsub_rn(c[3 * old], c[3 * recent]);
        const double dy = __dsub_rn(c[3 * old + 1], c[3 * recent + 1]);
        const double dz = __dsub_rn(c[3 * old + 2], c[3 * recent + 2]);
        const double d = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                        __dmul_rn(dz, dz)));
        dist[q] = d;
        idx[q] = q;
        flag[q] = d < thr ? 1 : 0;
    }
}

__global__ void k_pairs_out(int64_t m, int64_t gap, const int64_t* q_sorted, int64_t* pairs) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r, o;
        decode(q_sorted[i], r, o);
        pairs[2 * i] = o;
        pairs[2 * i + 1] = gap + r;
    }
}

struct Buf {
    std::vector<void*> p;
    cudaStream_t st;
    ~Buf() {
        for (void* x : p) cudaFreeAsync(x, st);
    }
    template <typename T>
    int32_t get(T** out, int64_t n) {
        void* q = nullptr;
        DPV_CUDA(cudaMallocAsync(&q, sizeof(T) * (size_t)std::max<int64_t>(n, 1), st));
        p.push_back(q);
        *out = reinterpret_cast<T*>(q);
        return DPV_OK;
    }
};

}  // namespace

int32_t proximity_detect(const double* centers, int64_t n, int64_t gap, double thr,
                         int64_t* pairs, int64_t cap, int64_t* count, cudaStream_t st) {
    *count = 0;
    if (n < gap + 1 || !(thr > 0.0)) return DPV_OK;
    const int64_t m = n - gap;
    const int64_t T = m * (m + 1) / 2;
    DPV_ARG(T < ((int64_t)1 << 31), "too many candidate pairs");
    Buf b{{}, st};
    double *dist, *dist_sel, *dist_s;
    int64_t *idx, *idx_sel, *idx_s, *nsel;
    uint8_t* flag;
    DPV_TRY(b.get(&dist, T));
    DPV_TRY(b.get(&idx, T));
    DPV_TRY(b.get(&flag, T));
    DPV_TRY(b.get(&dist_sel, T));
    DPV_TRY(b.get(&idx_sel, T));
    DPV_TRY(b.get(&nsel, 1));
    DPV_TSTART("detect", st);
    k_detect<<<grid_for(T, 256), 256, 0, st>>>(T, gap, centers, thr, dist, idx, flag);
    DPV_CHECK_LAUNCH();
    size_t tb = 0;
    DPV_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, dist, flag, dist_sel, nsel, (int)T, st));
    void* tmp;
    DPV_TRY(b.get(reinterpret_cast<char**>(&tmp), (int64_t)tb + 16));
    DPV_CUDA(cub::DeviceSelect::Flagged(tmp, tb, dist, flag, dist_sel, nsel, (int)T, st));
    size_t tb2 = 0;
    DPV_CUDA(cub::DeviceSelect::Flagged(nullptr, tb2, idx, flag, idx_sel, nsel, (int)T, st));
    void* tmp2;
    DPV_TRY(b.get(reinterpret_cast<char**>(&tmp2), (int64_t)tb2 + 16));
    DPV_CUDA(cub::DeviceSelect::Flagged(tmp2, tb2, idx, flag, idx_sel, nsel, (int)T, st));
    int64_t k = 0;
    DPV_CUDA(cudaMemcpyAsync(&k, nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    DPV_CUDA(cudaStreamSynchronize(st));
    *count = k;
    if (k == 0 || !pairs) return DPV_OK;
    DPV_ARG(cap >= k, "pair buffer too small (call again with the returned count)");
    DPV_TRY(b.get(&dist_s, k));
    DPV_TRY(b.get(&idx_s, k));
    size_t tb3 = 0;
    DPV_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb3, dist_sel, dist_s, idx_sel, idx_s, (int)k,
                                             0, 64, st));
    void* tmp3;
    DPV_TRY(b.get(reinterpret_cast<char**>(&tmp3), (int64_t)tb3 + 16));
    DPV_CUDA(cub::DeviceRadixSort::SortPairs(tmp3, tb3, dist_sel, dist_s, idx_sel, idx_s, (int)k, 0,
                                             64, st));
    k_pairs_out<<<grid_for(k, 256), 256, 0, st>>>(k, gap, idx_s, pairs);
    DPV_CHECK_LAUNCH();
    DPV_CUDA(cudaStreamSynchronize(st));
    return DPV_OK;
}

}  // namespace dpv
