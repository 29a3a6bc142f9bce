// K1 on TMA + tensor cores (bf16 features, radius 3), the B200 path of the
// correlation lookup (Eq. 4; conventions pinned by
// oracle/corr_oracle.py, see corr.cu).
//
// Per (edge, level) item the union of the 9 cells' 8x8 tap grids is a 10x10
// window of the target frame's feature map (cells of a 3x3 patch lie within
// ~1 px of each other at 1/4 resolution; wider spreads take a slow path).
// A PRODUCER warp runs S stages ahead: it reads the item's K2 coordinates,
// computes the window origin and per-cell offsets / bilinear weights, and
// issues TMA tile loads (cp.async.bulk.tensor, 128B swizzle, hardware zero
// fill outside the image) of the window (10x10 taps x 64 channels per box)
// and of the patch features, completing on an mbarrier.  Four CONSUMER warps
// run S (16 x 104) = G (16 x C) * Win^T on mma.sync.m16n8k16 (bf16 -> fp32)
// from the swizzled tiles and blend each cell's 7x7 outputs bilinearly from
// its 8x8 block of S, then release the stage.  No per-thread address math or
// bounds checks on the staging path; the dense volume is never stored.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>

#include "problem.cuh"

namespace dpv {
namespace {

constexpr int kCellsT = 9;
constexpr int kWin = 10;                  // window side (taps)
constexpr int kTapsPad = 104;             // 13 n-tiles of 8
constexpr int kHalfBytes = kTapsPad * 128;   // one 64-channel half of the window (swizzled rows)
constexpr int kGHalfBytes = 16 * 128;     // 16 feature rows x 64 channels
constexpr int kConsumers = 128;

struct CellMeta {
    int ox, oy;        // cell tap-grid origin inside the window (x0 - r - bx0, y0 - r - by0)
    float fx, fy;      // bilinear fractions
};
struct ItemMeta {
    CellMeta cell[kCellsT];
    int bx0, by0, staged, jj;
    int64_t e;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, unsigned tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)),
                 "r"(tx)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        "@!P bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                       int c3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                       uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
// four 8x8 b16 matrices from shared memory; lane l addresses row l % 8 of
// matrix l / 8 (16 contiguous bytes = one swizzle chunk)
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], unsigned addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}

__device__ __forceinline__ void mma_bf16_t(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void split(double v, int& i0, float& fr) {
    if (!(fabs(v) < 1e7)) {
        i0 = -(1 << 28);
        fr = 0.f;
        return;
    }
    const double f = floor(v);
    i0 = (int)f;
    fr = (float)(v - f);
}

// Per-NH (C / 64 channel halves) pipeline shape: stage bytes (window halves,
// patch-feature halves, item metadata; 1024-aligned for the 128B swizzle),
// NS stages in the ring, NP producer warps and NG consumer groups of 4 warps.
// Both NP and NG divide NS, so every stage has ONE producer and ONE consumer
// group, each walking that stage's items in order: an mbarrier parity wait
// can then never alias a phase two completions away (with several producers
// and a group count that does not divide NS, a group could pass its `full`
// wait on a stage whose previous item had not been produced yet).
#ifndef DPV_CORR_SMEM_KB
#define DPV_CORR_SMEM_KB 200      // stage-ring budget per CTA
#endif
#ifndef DPV_CORR_CTAS
#define DPV_CORR_CTAS 1           // CTAs per SM
#endif
template <int NH>
struct CorrCfg {
    static constexpr int SB =
        ((NH * (kHalfBytes + kGHalfBytes) + (int)sizeof(ItemMeta) + 1023) / 1024) * 1024;
    static constexpr int NS0 = (DPV_CORR_SMEM_KB * 1024) / SB;
    // C <= 128: 6 stages, 3 producers (one per pair of stages: a single
    // producer warp, ~400 dependent scalar instructions per item, capped the
    // kernel at ~1 item/us/SM), 3 consumer groups; C = 256: 3 stages, 1
    // producer, 3 groups
    static constexpr int NS = NS0 >= 6 ? 6 : (NS0 >= 3 ? 3 : (NS0 >= 1 ? NS0 : 1));
#ifdef DPV_CORR_NP6                 // pipeline-shape experiments (tools/corr_micro.cu)
    static constexpr int NP = NS == 6 ? DPV_CORR_NP6 : 1;
#else
    static constexpr int NP = NS == 6 ? 3 : 1;
#endif
#ifdef DPV_CORR_NG
    static constexpr int NG = NS >= DPV_CORR_NG ? DPV_CORR_NG : NS;
#else
    static constexpr int NG = NS >= 3 ? 3 : NS;
#endif
    static_assert(NS % NP == 0 && NS % NG == 0, "producers and groups must divide the stages");
    static constexpr int kThreadsT = 32 * NP + NG * kConsumers;
    static constexpr size_t kSmem =
        (size_t)NS * SB + sizeof(float) * NG * kCellsT * kTapsPad + 1024;
};

__device__ __forceinline__ void bar_group(int g) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + g), "n"(kConsumers) : "memory");
}

// One persistent CTA per SM; items are (edge, level) pairs, level fastest, so
// both pyramid levels run in ONE launch.  Warps 0..NP-1 are TMA producers,
// the rest form NG consumer groups of 4 warps; local item k goes to stage
// k % NS, producer k % NP and consumer group k % NG (= stage % NP / % NG).
template <int NH>
__global__ void __launch_bounds__(CorrCfg<NH>::kThreadsT, DPV_CORR_CTAS) k_corr_tma(
    const __grid_constant__ CUtensorMap fmap0_map, const __grid_constant__ CUtensorMap fmap1_map,
    const __grid_constant__ CUtensorMap gmap_map, const __nv_bfloat16* __restrict__ fmap0,
    const __nv_bfloat16* __restrict__ fmap1, const __nv_bfloat16* __restrict__ gmap,
    const double* __restrict__ coords, const int32_t* __restrict__ ii,
    const int32_t* __restrict__ jj, int64_t E, int h0, int w0, int h1, int w1, int levels,
    int vgrid, int64_t chunk, float* __restrict__ out) {
    using Cfg = CorrCfg<NH>;
    constexpr int C = 64 * NH, SB = Cfg::SB, NS = Cfg::NS, NG = Cfg::NG;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // 1024-byte aligned stage ring (pointer arithmetic keeps the shared space)
    unsigned char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint64_t full[NS], empty[NS];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 32);     // every producer lane arrives (below)
            mbar_init(&empty[s], kConsumers);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    // grid-stride items over vgrid virtual CTAs: the CTAs work on neighbouring
    // edges at any time, so the target frames' feature maps stay L2-resident
    // (edges grouped by frame).  Virtual CTA vb's local items are split into
    // chunks of `chunk`; CTA blockIdx.x runs chunk blockIdx.x / vgrid of
    // virtual CTA blockIdx.x % vgrid (one persistent CTA per SM: vgrid =
    // gridDim.x, one chunk).  Short-lived CTAs let a higher-priority stream
    // take SMs back at CTA granularity (the correlation beside the solve).
    const int64_t NV = E * levels;
    const int vb = (int)(blockIdx.x % (unsigned)vgrid);
    const int64_t U0 = (int64_t)(blockIdx.x / (unsigned)vgrid) * chunk;
    const int64_t n_v = NV > vb ? (NV - vb + vgrid - 1) / vgrid : 0;
    const int64_t n_my = n_v > U0 ? min(chunk, n_v - U0) : 0;
    constexpr int radius = 3, D = 8, O = 7;

    constexpr int NP = Cfg::NP;
    if (warp < NP) {
        // ---------------- producers ----------------
        // Producer warp p issues local items u = p, p + NP, ... into stages
        // u % NS (NP divides NS: stage s belongs to producer s % NP).  Per item
        // the producer does ~400 dependent scalar instructions (coordinate
        // split, window origin, metadata, TMA issue) at ~5 cycles each, so a
        // single producer warp per SM capped the kernel at ~1 item/us/SM.
        // K2 coordinates and indices run kLook items ahead: lane group
        // lg = lane / 9 (cells lc = lane % 9) holds the producer's i-th item
        // with i % kLook == lg, loaded kLook iterations before it is used.
        constexpr int kLook = 3;
        const int lg = lane / kCellsT, lc = lane % kCellsT;
        const int64_t n_mine = n_my > warp ? (n_my - warp + NP - 1) / NP : 0;
        double cxr = 0.0, cyr = 0.0;
        int32_t iir = 0, jjr = 0;
        auto edge_of = [&](int64_t v) { return levels == 2 ? (v >> 1) : v; };
        auto fetch = [&](int64_t i) {
            if (i >= n_mine || lg != (int)(i % kLook)) return;
            const int64_t e = edge_of(vb + (U0 + warp + i * NP) * (int64_t)vgrid);
            cxr = __ldg(coords + (e * kCellsT + lc) * 2);
            cyr = __ldg(coords + (e * kCellsT + lc) * 2 + 1);
            if (lc == 0) {
                iir = __ldg(ii + e);
                jjr = __ldg(jj + e);
            }
        };
#pragma unroll
        for (int q = 0; q < kLook; ++q) fetch(q);
        for (int64_t i = 0; i < n_mine; ++i) {
            const int64_t u = warp + i * NP;
            const int64_t v = vb + (U0 + u) * (int64_t)vgrid;
            const int64_t e = edge_of(v);
            const int level = levels == 2 ? (int)(v & 1) : 0;
            const int s = (int)(u % NS);
            const int src = (int)(i % kLook) * kCellsT;
            const double cx = __shfl_sync(0xffffffffu, cxr, src + (lane < kCellsT ? lane : 0));
            const double cy = __shfl_sync(0xffffffffu, cyr, src + (lane < kCellsT ? lane : 0));
            const int32_t iic = __shfl_sync(0xffffffffu, iir, src);
            const int32_t jjc = __shfl_sync(0xffffffffu, jjr, src);
            fetch(i + kLook);
            mbar_wait(&empty[s], (unsigned)(((u / NS) & 1) ^ 1));
            ItemMeta* M = reinterpret_cast<ItemMeta*>(sm + s * SB + NH * (kHalfBytes + kGHalfBytes));
            const double scale = level == 0 ? 1.0 : 0.25;
            int x0 = 0, y0 = 0;
            float fx = 0.f, fy = 0.f;
            if (lane < kCellsT) {
                split(cx * scale, x0, fx);
                split(cy * scale, y0, fy);
            }
            int mnx = lane < kCellsT ? x0 : INT32_MAX, mxx = lane < kCellsT ? x0 : INT32_MIN;
            int mny = lane < kCellsT ? y0 : INT32_MAX, mxy = lane < kCellsT ? y0 : INT32_MIN;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                mnx = min(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
                mxx = max(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
                mny = min(mny, __shfl_xor_sync(0xffffffffu, mny, o));
                mxy = max(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
            }
            const int bx0 = mnx - radius, by0 = mny - radius;
            const bool staged = (mxx - mnx) <= kWin - D && (mxy - mny) <= kWin - D &&
                                mnx > -(1 << 27);
            if (lane < kCellsT) {
                M->cell[lane].ox = staged ? x0 - radius - bx0 : x0 - radius;
                M->cell[lane].oy = staged ? y0 - radius - by0 : y0 - radius;
                M->cell[lane].fx = fx;
                M->cell[lane].fy = fy;
            }
            if (lane == 0) {
                M->bx0 = bx0;
                M->by0 = by0;
                M->staged = (staged ? 1 : 0) | (level << 1);
                M->jj = jjc;
                M->e = e;
            }
            // each lane publishes its own metadata writes with its own
            // (release) arrival; lane 0's also carries the TMA byte count
            if (lane != 0) mbar_arrive(&full[s]);
            if (lane == 0) {
                unsigned char* st = sm + s * SB;
                const unsigned tx = NH * kGHalfBytes + (staged ? NH * kWin * kWin * 128 : 0);
                mbar_arrive_tx(&full[s], tx);
                const int grow = iic * kCellsT;
                const CUtensorMap* fm = level == 0 ? &fmap0_map : &fmap1_map;
#pragma unroll
                for (int h = 0; h < NH; ++h) {
                    tma_2d(st + NH * kHalfBytes + h * kGHalfBytes, &gmap_map, 64 * h, grow,
                           &full[s]);
                    if (staged) tma_4d(st + h * kHalfBytes, fm, 64 * h, bx0, by0, jjc, &full[s]);
                }
            }
        }
        return;
    }
    // ---------------- consumer groups (4 warps each) ----------------
    const int grp = (warp - NP) >> 2, gw = (warp - NP) & 3,
              gtid = tid - 32 * NP - grp * kConsumers;
    float* S = reinterpret_cast<float*>(sm + NS * SB) + grp * (kCellsT * kTapsPad);
    const int g = lane >> 2, t4 = lane & 3;
    // ldmatrix lane roles (128B swizzle: chunk' = chunk ^ (row % 8), rows of
    // a tile start 1024-aligned so row % 8 = lane % 8 for every matrix):
    // A (16 patch rows x 2 chunks): row l%8 + 8*((l/8)&1), chunk +(l/16)
    // B (8 tap rows x 4 chunks = two k-steps): row nt*8 + l%8, chunk +(l/8)
    const int l7 = lane & 7;
    const unsigned offA = (unsigned)((l7 + 8 * ((lane >> 3) & 1)) * 128);
    const unsigned mA = (unsigned)(((lane >> 4) ^ l7) << 4);
    const unsigned offB = (unsigned)((gw * 8 + l7) * 128);
    const unsigned mB = (unsigned)(((lane >> 3) ^ l7) << 4);
    // blend slots of this thread (x = gtid + 128 i < 441), fixed for all items
    int slot_c[4], slot_off[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int x = gtid + kConsumers * i;
        const int c = x / (O * O), ab = x % (O * O);
        slot_c[i] = x < kCellsT * O * O ? c : -1;
        slot_off[i] = c * kTapsPad + (ab / O) * kWin + ab % O;
    }
    for (int64_t u = grp; u < n_my; u += NG) {
        const int s = (int)(u % NS);
        mbar_wait(&full[s], (unsigned)((u / NS) & 1));
        const unsigned char* st = sm + s * SB;
        const ItemMeta* M = reinterpret_cast<const ItemMeta*>(st + NH * (kHalfBytes + kGHalfBytes));
        const unsigned char* Gs = st + NH * kHalfBytes;
        const int level = M->staged >> 1;
        float* o = out + ((M->e * levels + level) * kCellsT) * (int64_t)(O * O);
        if (M->staged & 1) {
            float acc[4][4];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0.f;
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                const unsigned wb = smem_u32(st + h * kHalfBytes) + offB;
                const unsigned gb = smem_u32(Gs + h * kGHalfBytes) + offA;
#pragma unroll
                for (int kc = 0; kc < 8; kc += 4) {     // 16-byte chunk = 8 channels
                    uint32_t a0[4], a1[4];
                    ldsm_x4(a0, gb + ((unsigned)(kc << 4) ^ mA));
                    ldsm_x4(a1, gb + ((unsigned)((kc + 2) << 4) ^ mA));
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        if (gw + 4 * q < 13) {
                            uint32_t b[4];
                            ldsm_x4(b, wb + q * 4096 + ((unsigned)(kc << 4) ^ mB));
                            mma_bf16_t(acc[q], a0, b[0], b[1]);
                            mma_bf16_t(acc[q], a1, b[2], b[3]);
                        }
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int nt = gw + 4 * q;
                if (nt < 13) {
                    const int col = nt * 8 + 2 * t4;
                    *reinterpret_cast<float2*>(S + g * kTapsPad + col) =
                        make_float2(acc[q][0], acc[q][1]);
                    if (g == 0)
                        *reinterpret_cast<float2*>(S + 8 * kTapsPad + col) =
                            make_float2(acc[q][2], acc[q][3]);
                }
            }
            bar_group(grp);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if (slot_c[i] < 0) continue;
                const CellMeta cm = M->cell[slot_c[i]];
                const float* sp = S + slot_off[i] + cm.oy * kWin + cm.ox;
                o[gtid + kConsumers * i] =
                    (1.f - cm.fy) * ((1.f - cm.fx) * sp[0] + cm.fx * sp[1]) +
                    cm.fy * ((1.f - cm.fx) * sp[kWin] + cm.fx * sp[kWin + 1]);
            }
        } else {
            // wide or non-finite window: per-cell integer-tap dots from global memory
            const int H = level == 0 ? h0 : h1, Wd = level == 0 ? w0 : w1;
            const __nv_bfloat16* fp = (level == 0 ? fmap0 : fmap1) + (int64_t)M->jj * H * Wd * C;
            const __nv_bfloat16* gp = gmap + (int64_t)ii[M->e] * kCellsT * C;
            for (int x = gtid; x < kCellsT * D * D; x += kConsumers) {
                const int c = x / (D * D), ty = (x % (D * D)) / D, tx = x % D;
                const int py = M->cell[c].oy + ty, px = M->cell[c].ox + tx;
                float acc = 0.f;
                if (py >= 0 && py < H && px >= 0 && px < Wd) {
                    const __nv_bfloat16* f = fp + ((int64_t)py * Wd + px) * C;
                    for (int k = 0; k < C; ++k)
                        acc += __bfloat162float(f[k]) * __bfloat162float(gp[c * C + k]);
                }
                S[c * kTapsPad + ty * D + tx] = acc;
            }
            bar_group(grp);
            for (int x = gtid; x < kCellsT * O * O; x += kConsumers) {
                const int c = x / (O * O), ab = x % (O * O), a = ab / O, bb = ab % O;
                const float dx = M->cell[c].fx, dy = M->cell[c].fy;
                const float* sp = S + c * kTapsPad + a * D + bb;
                o[x] = (1.f - dy) * ((1.f - dx) * sp[0] + dx * sp[1]) +
                       dy * ((1.f - dx) * sp[D] + dx * sp[D + 1]);
            }
        }
        bar_group(grp);          // S and the stage are free
        mbar_arrive(&empty[s]);
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

}  // namespace

// bf16 features, radius 3, C in {64, 128, 256}, both levels in one launch;
// returns DPV_BAD_ARGS when the TMA path does not apply (the caller falls
// back to corr.cu)
int32_t corr_tma(const void* gmap, int64_t n_patches, const void* fmap0, const void* fmap1,
                 int64_t n_frames, const double* coords, const int32_t* ii, const int32_t* jj,
                 int64_t E, int C, int h0, int w0, int h1, int w1, int levels, float* out,
                 int64_t items_per_cta, cudaStream_t st) {
    auto enc = encode_fn();
    if (!enc || (C != 64 && C != 128 && C != 256) || n_patches < 1 || n_frames < 1 ||
        (levels == 2 && (!fmap1 || h1 < 1 || w1 < 1)) ||
        (reinterpret_cast<uintptr_t>(fmap0) & 15) || (reinterpret_cast<uintptr_t>(gmap) & 15) ||
        (levels == 2 && (reinterpret_cast<uintptr_t>(fmap1) & 15)))
        return DPV_BAD_ARGS;
    CUtensorMap fm[2], gm;
    for (int l = 0; l < 2; ++l) {
        // level 1 absent: encode level 0 twice (never read)
        const bool has = l < levels;
        const int H = has && l == 1 ? h1 : h0, Wd = has && l == 1 ? w1 : w0;
        const void* f = has && l == 1 ? fmap1 : fmap0;
        const cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)Wd, (cuuint64_t)H,
                                    (cuuint64_t)n_frames};
        const cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)Wd * C * 2,
                                       (cuuint64_t)H * Wd * C * 2};
        const cuuint32_t box[4] = {64, kWin, kWin, 1};
        const cuuint32_t es[4] = {1, 1, 1, 1};
        if (enc(&fm[l], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(f), dims, strides,
                box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS)
            return DPV_BAD_ARGS;
    }
    {
        const cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)n_patches * kCellsT};
        const cuuint64_t strides[1] = {(cuuint64_t)C * 2};
        const cuuint32_t box[2] = {64, 16};
        const cuuint32_t es[2] = {1, 1};
        if (enc(&gm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(gmap), dims, strides,
                box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS)
            return DPV_BAD_ARGS;
    }
    auto launch = [&](auto kern, size_t smem, int threads, int slot) -> int32_t {
        static size_t cur[3] = {0, 0, 0};
        DPV_TRY(ensure_smem(kern, smem, cur[slot]));
        const int64_t items = E * levels;
        const int vgrid =
            (int)std::max<int64_t>(1, std::min<int64_t>(items, (int64_t)sm_count() * DPV_CORR_CTAS));
        const int64_t per = (items + vgrid - 1) / vgrid;          // local items per virtual CTA
        const int64_t chunk = items_per_cta > 0 ? std::min(items_per_cta, per) : per;
        const int64_t grid = (int64_t)vgrid * ((per + chunk - 1) / chunk);
        if (grid > INT32_MAX) return DPV_BAD_ARGS;
        DPV_TSTART("corr", st);
        kern<<<(unsigned)grid, threads, smem, st>>>(fm[0], fm[1], gm,
                                          reinterpret_cast<const __nv_bfloat16*>(fmap0),
                                          reinterpret_cast<const __nv_bfloat16*>(fmap1),
                                          reinterpret_cast<const __nv_bfloat16*>(gmap), coords,
                                          ii, jj, E, h0, w0, h1, w1, levels, vgrid, chunk, out);
        DPV_CHECK_LAUNCH();
        return DPV_OK;
    };
    if (C == 64) return launch(k_corr_tma<1>, CorrCfg<1>::kSmem, CorrCfg<1>::kThreadsT, 0);
    if (C == 128) return launch(k_corr_tma<2>, CorrCfg<2>::kSmem, CorrCfg<2>::kThreadsT, 1);
    return launch(k_corr_tma<4>, CorrCfg<4>::kSmem, CorrCfg<4>::kThreadsT, 2);
}

}  // namespace dpv
