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

#include <algorithm>
#include <cstdlib>

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

// ---------------------------------------------------------------------------
// bf16 features on the tensor cores.  Per (edge, level) the union window of
// the 9 cells' 8x8 tap grids (<= kMmaTaps taps; ~81 at these scales) and the
// patch's 9 feature vectors are staged in shared memory with cp.async, then
//   S (16 x taps) = G (16 x C, rows >= 9 zero) * Win^T (C x taps)
// runs on mma.sync.m16n8k16 bf16 -> fp32 (K = C); each cell's 7x7 outputs
// are the bilinear blend of its 8x8 block of S.  Items are double-buffered
// (the next window streams in while the current one multiplies).  Windows
// wider than kMmaTaps fall back to per-cell dots from global memory.
constexpr int kMmaTaps = 104;     // 13 n-tiles of 8
constexpr int kMmaThreads = 128;

__device__ __forceinline__ void mma_bf16(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}

struct CorrMeta {
    int x0[kCells], y0[kCells];
    float fx[kCells], fy[kCells];
    int bx0, by0, bw, bh;
    int staged;
    int64_t e;
};

template <int C>
__global__ void __launch_bounds__(kMmaThreads) k_corr_mma(
    const __nv_bfloat16* __restrict__ gmap, const __nv_bfloat16* __restrict__ fmap,
    const double* __restrict__ coords, const int32_t* __restrict__ ii,
    const int32_t* __restrict__ jj, int64_t E, int H, int Wd, int level, int levels,
    float* __restrict__ out) {
    constexpr int LDK = C + 8;                      // bf16 per staged row (272 B at C=128)
    constexpr int BUF = (16 + kMmaTaps) * LDK;      // bf16 per buffer: G rows + window taps
    constexpr int radius = 3, D = 8, O = 7;
    extern __shared__ __align__(16) unsigned char smraw[];
    __nv_bfloat16* const buf0 = reinterpret_cast<__nv_bfloat16*>(smraw);
    auto buf = [&](int b) { return buf0 + b * BUF; };
    float* S = reinterpret_cast<float*>(smraw + 2 * sizeof(__nv_bfloat16) * BUF);  // 9 x kMmaTaps
    __shared__ CorrMeta meta[2];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, t4 = lane & 3;
    const double scale = level == 0 ? 1.0 : 0.25;
    // G rows 9..15 stay zero
    for (int x = tid; x < 7 * LDK; x += kMmaThreads) {
        buf(0)[9 * LDK + x] = __float2bfloat16(0.f);
        buf(1)[9 * LDK + x] = __float2bfloat16(0.f);
    }
    // metadata + async staging of item e into buffer b
    auto stage = [&](int64_t e, int b) {
        CorrMeta& M = meta[b];
        if (tid < kCells) {
            int x0, y0;
            float fx, fy;
            split_coord(coords[(e * kCells + tid) * 2] * scale, x0, fx);
            split_coord(coords[(e * kCells + tid) * 2 + 1] * scale, y0, fy);
            M.x0[tid] = x0; M.y0[tid] = y0; M.fx[tid] = fx; M.fy[tid] = fy;
        }
        __syncthreads();
        if (tid == 0) {
            int mnx = M.x0[0], mxx = M.x0[0], mny = M.y0[0], mxy = M.y0[0];
            for (int c = 1; c < kCells; ++c) {
                mnx = min(mnx, M.x0[c]); mxx = max(mxx, M.x0[c]);
                mny = min(mny, M.y0[c]); mxy = max(mxy, M.y0[c]);
            }
            M.bx0 = mnx - radius; M.by0 = mny - radius;
            M.bw = mxx - mnx + D; M.bh = mxy - mny + D;
            M.staged = (mxx - mnx) < 64 && (mxy - mny) < 64 && M.bw * M.bh <= kMmaTaps;
            M.e = e;
        }
        __syncthreads();
        __nv_bfloat16* G = buf(b);
        __nv_bfloat16* Win = buf(b) + 16 * LDK;
        const __nv_bfloat16* gp = gmap + (int64_t)ii[e] * kCells * C;
        constexpr int CH = C / 8;                   // 16-byte chunks per row
        for (int x = tid; x < kCells * CH; x += kMmaThreads)
            cp16(G + (x / CH) * LDK + (x % CH) * 8, gp + (int64_t)x * 8);
        if (M.staged) {
            const __nv_bfloat16* fp = fmap + (int64_t)jj[e] * H * Wd * C;
            const int ntap = M.bw * M.bh;
            for (int x = tid; x < ntap * CH; x += kMmaThreads) {
                const int tp = x / CH, k = (x % CH) * 8;
                const int py = M.by0 + tp / M.bw, px = M.bx0 + tp % M.bw;
                __nv_bfloat16* dst = Win + tp * LDK + k;
                if (py >= 0 && py < H && px >= 0 && px < Wd)
                    cp16(dst, fp + ((int64_t)py * Wd + px) * C + k);
                else
                    *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
            }
            // zero the pad taps of the last n-tile
            const int ntile_taps = ((ntap + 7) / 8) * 8;
            for (int x = tid; x < (ntile_taps - ntap) * CH; x += kMmaThreads)
                *reinterpret_cast<uint4*>(Win + (ntap + x / CH) * LDK + (x % CH) * 8) =
                    make_uint4(0, 0, 0, 0);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    int64_t e = blockIdx.x;
    if (e >= E) return;
    stage(e, 0);
    int b = 0;
    for (; e < E; e += gridDim.x, b ^= 1) {
        const int64_t en = e + gridDim.x;
        if (en < E) {
            stage(en, b ^ 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        const CorrMeta& M = meta[b];
        const __nv_bfloat16* G = buf(b);
        const __nv_bfloat16* Win = buf(b) + 16 * LDK;
        if (M.staged) {
            const int ntiles = (M.bw * M.bh + 7) / 8;
            float acc[4][4];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0.f;
#pragma unroll 2
            for (int k0 = 0; k0 < C; k0 += 16) {
                uint32_t a[4];
                a[0] = *reinterpret_cast<const uint32_t*>(G + g * LDK + k0 + 2 * t4);
                a[1] = *reinterpret_cast<const uint32_t*>(G + (g + 8) * LDK + k0 + 2 * t4);
                a[2] = *reinterpret_cast<const uint32_t*>(G + g * LDK + k0 + 2 * t4 + 8);
                a[3] = *reinterpret_cast<const uint32_t*>(G + (g + 8) * LDK + k0 + 2 * t4 + 8);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int nt = warp + 4 * q;
                    if (nt < ntiles) {
                        const __nv_bfloat16* bp = Win + (nt * 8 + g) * LDK + k0 + 2 * t4;
                        mma_bf16(acc[q], a, *reinterpret_cast<const uint32_t*>(bp),
                                 *reinterpret_cast<const uint32_t*>(bp + 8));
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int nt = warp + 4 * q;
                if (nt < ntiles) {
                    const int col = nt * 8 + 2 * t4;
                    S[g * kMmaTaps + col] = acc[q][0];
                    S[g * kMmaTaps + col + 1] = acc[q][1];
                    if (g == 0) {
                        S[8 * kMmaTaps + col] = acc[q][2];
                        S[8 * kMmaTaps + col + 1] = acc[q][3];
                    }
                }
            }
        }
        __syncthreads();
        float* o = out + ((M.e * levels + level) * kCells) * (int64_t)(O * O);
        if (M.staged) {
            for (int x = tid; x < kCells * O * O; x += kMmaThreads) {
                const int c = x / (O * O), ab = x % (O * O), a = ab / O, bb = ab % O;
                const float dx = M.fx[c], dy = M.fy[c];
                const int base = (M.y0[c] - radius + a - M.by0) * M.bw + (M.x0[c] - radius + bb - M.bx0);
                const float* sp = S + c * kMmaTaps + base;
                o[x] = (1.f - dy) * ((1.f - dx) * sp[0] + dx * sp[1]) +
                       dy * ((1.f - dx) * sp[M.bw] + dx * sp[M.bw + 1]);
            }
        } else {
            // wide window: per-cell integer-tap dots straight from global memory
            const __nv_bfloat16* fp = fmap + (int64_t)jj[M.e] * H * Wd * C;
            for (int x = tid; x < kCells * D * D; x += kMmaThreads) {
                const int c = x / (D * D), ty = (x % (D * D)) / D, tx = x % D;
                const int py = M.y0[c] - radius + ty, px = M.x0[c] - radius + tx;
                float acc = 0.f;
                if (py >= 0 && py < H && px >= 0 && px < Wd) {
                    const __nv_bfloat16* f = fp + ((int64_t)py * Wd + px) * C;
                    for (int k = 0; k < C; ++k)
                        acc += __bfloat162float(f[k]) * __bfloat162float(G[c * LDK + k]);
                }
                S[c * kMmaTaps + ty * D + tx] = acc;
            }
            __syncthreads();
            for (int x = tid; x < kCells * O * O; x += kMmaThreads) {
                const int c = x / (O * O), ab = x % (O * O), a = ab / O, bb = ab % O;
                const float dx = M.fx[c], dy = M.fy[c];
                const float* sp = S + c * kMmaTaps + a * D + bb;
                o[x] = (1.f - dy) * ((1.f - dx) * sp[0] + dx * sp[1]) +
                       dy * ((1.f - dx) * sp[D] + dx * sp[D + 1]);
            }
        }
        __syncthreads();
    }
}

template <int C>
int32_t launch_corr_mma(const void* gmap, const void* fmap, const double* coords,
                        const int32_t* ii, const int32_t* jj, int64_t E, int H, int Wd,
                        int level, int levels, float* out, cudaStream_t st) {
    const size_t smem = 2 * sizeof(__nv_bfloat16) * (16 + kMmaTaps) * (C + 8) +
                        sizeof(float) * kCells * kMmaTaps;
    static size_t cur = 0;
    DPV_TRY(ensure_smem(k_corr_mma<C>, smem, cur));
    int per_sm = 0;
    DPV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_corr_mma<C>, kMmaThreads,
                                                           smem));
    const int grid = (int)std::min<int64_t>(E, (int64_t)sm_count() * std::max(1, per_sm));
    DPV_TSTART("corr", st);
    k_corr_mma<C><<<grid, kMmaThreads, smem, st>>>(
        reinterpret_cast<const __nv_bfloat16*>(gmap), reinterpret_cast<const __nv_bfloat16*>(fmap),
        coords, ii, jj, E, H, Wd, level, levels, out);
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
        else if (radius == 3 && C == 128)
            DPV_TRY(launch_corr_mma<128>(gmap, f, coords, ii, jj, E, H, Wd, l, levels, out, st));
        else if (radius == 3 && C == 64)
            DPV_TRY(launch_corr_mma<64>(gmap, f, coords, ii, jj, E, H, Wd, l, levels, out, st));
        else if (radius == 3 && C == 256)
            DPV_TRY(launch_corr_mma<256>(gmap, f, coords, ii, jj, E, H, Wd, l, levels, out, st));
        else
            DPV_TRY(launch_corr<__nv_bfloat16>(gmap, f, coords, ii, jj, E, C, H, Wd, l, levels,
                                               radius, out, st));
    }
    return DPV_OK;
}

}  // namespace dpv
