// K1: on-the-fly per-edge correlation lookup (Eq. 4).
// The reference package has no correlation code; conventions are
// pinned by the float64 oracle (oracle/corr_oracle.py) and DESIGN.md:
//   * features channels-last: gmap (patches, p*p, C), fmap_l (frames, H_l, W_l, C)
//   * level-l coordinate = level-0 coordinate / 4^l (4x4 average-pool pyramid)
//   * out[e, l, cell, a, b] = <g(cell), f_l(P'(cell) + (b - r, a - r))>, bilinear
//     f with out-of-bounds taps = 0; evaluated as the bilinear blend of the
//     (2r+2)^2 integer-tap dot products (the dot is linear).
// The dense correlation volume is never stored: each CTA stages the union of
// its edge's tap windows (<= 12x12 taps) in shared memory once and reuses it
// for all p*p cells.
#include <cuda_bf16.h>

#include "problem.cuh"

namespace dpv {
namespace {

constexpr int kMaxWin = 12;      // staged window side (taps)
constexpr int kCells = 9;        // p = 3

template <typename T>
__device__ __forceinline__ float4 load4(const T* p);
template <>
__device__ __forceinline__ float4 load4<float>(const float* p) {
    return __ldg(reinterpret_cast<const float4*>(p));
}
template <>
__device__ __forceinline__ float4 load4<__nv_bfloat16>(const __nv_bfloat16* p) {
    const uint2 raw = __ldg(reinterpret_cast<const uint2*>(p));
    const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&raw.x);
    const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&raw.y);
    const float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
    return make_float4(fa.x, fa.y, fb.x, fb.y);
}

// coordinate -> (floor, frac); non-finite or huge -> far out of bounds
__device__ __forceinline__ void split_coord(double v, int& i0, float& frac) {
    if (!(fabs(v) < 1e7)) {
        i0 = -(1 << 28);
        frac = 0.f;
        return;
    }
    const double f = floor(v);
    i0 = (int)f;
    frac = (float)(v - f);
}

template <typename T>
__global__ void __launch_bounds__(192) k_corr(
    const T* __restrict__ gmap, const T* __restrict__ fmap, const double* __restrict__ coords,
    const int32_t* __restrict__ ii, const int32_t* __restrict__ jj, int64_t E, int C, int H,
    int Wd, int level, int levels, int radius, float* __restrict__ out) {
    extern __shared__ float sm[];
    const int ld = C + 4;
    const int D = 2 * radius + 2;          // integer taps per side
    const int O = 2 * radius + 1;          // outputs per side
    float* g = sm;                          // kCells x ld
    float* S = g + kCells * ld;             // kCells x D*D dot products
    float* win = S + kCells * 64;           // window taps x ld
    __shared__ int cx0[kCells], cy0[kCells];
    __shared__ float cfx[kCells], cfy[kCells];
    __shared__ int bx0, by0, bw, bh;
    const double scale = level == 0 ? 1.0 : 0.25;
    const int tid = threadIdx.x;
    for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
        const int32_t pi = ii[e], fj = jj[e];
        if (tid < kCells) {
            int x0, y0;
            float fx, fy;
            split_coord(coords[(e * kCells + tid) * 2] * scale, x0, fx);
            split_coord(coords[(e * kCells + tid) * 2 + 1] * scale, y0, fy);
            cx0[tid] = x0; cy0[tid] = y0; cfx[tid] = fx; cfy[tid] = fy;
        }
        // stage patch features
        const T* gp = gmap + (int64_t)pi * kCells * C;
        for (int x = tid * 4; x < kCells * C; x += blockDim.x * 4) {
            const int c = x / C, k = x % C;
            *reinterpret_cast<float4*>(g + c * ld + k) = load4<T>(gp + x);
        }
        __syncthreads();
        if (tid == 0) {
            int mnx = cx0[0], mxx = cx0[0], mny = cy0[0], mxy = cy0[0];
            for (int c = 1; c < kCells; ++c) {
                mnx = min(mnx, cx0[c]); mxx = max(mxx, cx0[c]);
                mny = min(mny, cy0[c]); mxy = max(mxy, cy0[c]);
            }
            bx0 = mnx - radius; by0 = mny - radius;
            bw = mxx - mnx + D; bh = mxy - mny + D;
        }
        __syncthreads();
        const bool staged = bw <= kMaxWin && bh <= kMaxWin;
        const T* fp = fmap + (int64_t)fj * H * Wd * C;
        if (staged) {
            const int ntap = bw * bh;
            const int c4 = C / 4;
            for (int x = tid; x < ntap * c4; x += blockDim.x) {
                const int tp = x / c4, k = (x % c4) * 4;
                const int py = by0 + tp / bw, px = bx0 + tp % bw;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (py >= 0 && py < H && px >= 0 && px < Wd)
                    v = load4<T>(fp + ((int64_t)py * Wd + px) * C + k);
                *reinterpret_cast<float4*>(win + tp * ld + k) = v;
            }
        }
        __syncthreads();
        // dot products: thread = (cell group of 3, tap), 3 dots sharing the tap load
        if (tid < 3 * 64) {
            const int cg = tid / 64, tap = tid % 64;
            if (tap < D * D) {
                const int ty = tap / D, tx = tap % D;
                float acc[3] = {0.f, 0.f, 0.f};
                if (staged) {
                    int off[3];
                    for (int q = 0; q < 3; ++q) {
                        const int c = cg * 3 + q;
                        off[q] = ((cy0[c] - radius + ty - by0) * bw + (cx0[c] - radius + tx - bx0)) * ld;
                    }
                    for (int k = 0; k < C; k += 4) {
#pragma unroll
                        for (int q = 0; q < 3; ++q) {
                            const float4 f = *reinterpret_cast<const float4*>(win + off[q] + k);
                            const float4 gg =
                                *reinterpret_cast<const float4*>(g + (cg * 3 + q) * ld + k);
                            acc[q] = fmaf(f.x, gg.x, acc[q]);
                            acc[q] = fmaf(f.y, gg.y, acc[q]);
                            acc[q] = fmaf(f.z, gg.z, acc[q]);
                            acc[q] = fmaf(f.w, gg.w, acc[q]);
                        }
                    }
                } else {
                    for (int q = 0; q < 3; ++q) {
                        const int c = cg * 3 + q;
                        const int py = cy0[c] - radius + ty, px = cx0[c] - radius + tx;
                        if (py >= 0 && py < H && px >= 0 && px < Wd) {
                            const T* f = fp + ((int64_t)py * Wd + px) * C;
                            for (int k = 0; k < C; k += 4) {
                                const float4 fv = load4<T>(f + k);
                                const float4 gg = *reinterpret_cast<const float4*>(g + c * ld + k);
                                acc[q] = fmaf(fv.x, gg.x, acc[q]);
                                acc[q] = fmaf(fv.y, gg.y, acc[q]);
                                acc[q] = fmaf(fv.z, gg.z, acc[q]);
                                acc[q] = fmaf(fv.w, gg.w, acc[q]);
                            }
                        }
                    }
                }
                for (int q = 0; q < 3; ++q) S[(cg * 3 + q) * 64 + tap] = acc[q];
            }
        }
        __syncthreads();
        // bilinear blend of integer-tap dots -> (2r+1)^2 outputs per cell
        float* o = out + ((e * levels + level) * kCells) * (int64_t)(O * O);
        for (int x = tid; x < kCells * O * O; x += blockDim.x) {
            const int c = x / (O * O), ab = x % (O * O), a = ab / O, b = ab % O;
            const float dx = cfx[c], dy = cfy[c];
            const float* s = S + c * 64;
            const float v = (1.f - dy) * ((1.f - dx) * s[a * D + b] + dx * s[a * D + b + 1]) +
                            dy * ((1.f - dx) * s[(a + 1) * D + b] + dx * s[(a + 1) * D + b + 1]);
            o[x] = v;
        }
        __syncthreads();
    }
}

template <typename T>
int32_t launch_corr(const void* gmap, const void* fmap, const double* coords, const int32_t* ii,
                    const int32_t* jj, int64_t E, int C, int H, int Wd, int level, int levels,
                    int radius, float* out, cudaStream_t st) {
    const int ld = C + 4;
    const size_t smem = sizeof(float) * ((size_t)kCells * ld + kCells * 64 +
                                         (size_t)kMaxWin * kMaxWin * ld);
    DPV_ARG(smem <= 220 * 1024, "channel count too large for the staged window");
    static size_t cur = 0;
    DPV_TRY(ensure_smem(k_corr<T>, smem, cur));
    const int grid = (int)std::min<int64_t>(E, (int64_t)sm_count() * 16);
    DPV_TSTART("corr", st);
    k_corr<T><<<grid, 192, smem, st>>>(reinterpret_cast<const T*>(gmap),
                                        reinterpret_cast<const T*>(fmap), coords, ii, jj, E, C,
                                        H, Wd, level, levels, radius, out);
    DPV_CHECK_LAUNCH();
    return DPV_OK;
}

// level-1 pyramid: 4x4 average pool, channels-last (DPVO avg_pool2d(4, 4))
template <typename T>
__global__ void k_avg_pool4(const T* __restrict__ in, int64_t F, int H, int W, int C,
                            T* __restrict__ out) {
    const int H4 = H / 4, W4 = W / 4;
    const int64_t total = F * H4 * W4 * C;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(x % C);
        int64_t r = x / C;
        const int j = (int)(r % W4);
        r /= W4;
        const int i = (int)(r % H4);
        const int64_t f = r / H4;
        float s = 0.f;
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b)
                s += (float)in[((f * H + 4 * i + a) * W + 4 * j + b) * C + c];
        out[x] = (T)(s * 0.0625f);
    }
}

}  // namespace

int32_t avg_pool4(const void* in, int64_t F, int H, int W, int C, int dtype, void* out,
                  cudaStream_t st) {
    const int64_t total = F * (H / 4) * (W / 4) * C;
    if (total == 0) return DPV_OK;
    DPV_TSTART("avg_pool4", st);
    if (dtype == 0)
        k_avg_pool4<float><<<grid_for(total, 256), 256, 0, st>>>(
            reinterpret_cast<const float*>(in), F, H, W, C, reinterpret_cast<float*>(out));
    else
        k_avg_pool4<__nv_bfloat16><<<grid_for(total, 256), 256, 0, st>>>(
            reinterpret_cast<const __nv_bfloat16*>(in), F, H, W, C,
            reinterpret_cast<__nv_bfloat16*>(out));
    DPV_CHECK_LAUNCH();
    return DPV_OK;
}

int32_t corr(const void* gmap, const void* fmap0, const void* fmap1, const double* coords,
             const int32_t* ii, const int32_t* jj, int64_t E, int C, int h0, int w0, int h1,
             int w1, int levels, int radius, int dtype, float* out, cudaStream_t st) {
    DPV_ARG(C % 4 == 0, "channels must be a multiple of 4");
    DPV_ARG(radius <= 3, "radius <= 3 (8x8 integer taps)");
    if (E == 0) return DPV_OK;
    for (int l = 0; l < levels; ++l) {
        const void* f = l == 0 ? fmap0 : fmap1;
        const int H = l == 0 ? h0 : h1, Wd = l == 0 ? w0 : w1;
        if (dtype == 0)
            DPV_TRY(launch_corr<float>(gmap, f, coords, ii, jj, E, C, H, Wd, l, levels, radius,
                                       out, st));
        else
            DPV_TRY(launch_corr<__nv_bfloat16>(gmap, f, coords, ii, jj, E, C, H, Wd, l, levels,
                                               radius, out, st));
    }
    return DPV_OK;
}

}  // namespace dpv
