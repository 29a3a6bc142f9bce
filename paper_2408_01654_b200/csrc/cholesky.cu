// K4c: FP64 Cholesky factor + solve of the damped reduced camera system
// S(lambda) (ba.py:451-487: scipy cho_factor/cho_solve = LAPACK potrf/potrs;
// block_cholesky.py:48-111 for the block-sparse backend), B200 design:
//
//  * augmented (N+1) x ld row-major lower storage, rhs in row N, so the
//    right-looking factorisation also produces y = L^-1 b;
//  * a FactorPlan decides which 64x64 tiles are touched: dense (every lower
//    tile) or sparse = the symbolic tile-level fill of the pose-block pattern
//    after a symmetric permutation that moves "border" poses (long-range
//    loop-closure couplings) last, so the rest is banded.  The
//    same kernels serve both; the sparse plan skips structurally-zero tiles;
//  * per 64-column panel, on a high-priority stream (the critical path):
//      potrf_inv: one CTA factors the 64x64 diagonal block in shared memory
//                 (one barrier per column) and inverts it;
//      trsm:      L21 = A21 L11^-T as a DMMA product with the inverse;
//      syrk:      intra-group update of the second panel, then the next
//                 group's columns;
//  * the rest of the trailing update on a low-priority stream (look-ahead),
//    K = 128 (two panels per group) on the FP64 tensor cores
//    (mma.sync.m8n8k4.f64 -> DMMA; tcgen05 has no f64 kind);
//  * backward substitution L^T x = y using the diagonal-block inverses: one
//    CTA walking the plan's nonzero tiles (sparse plans), or one cooperative
//    persistent kernel with a grid barrier per panel (dense plans).
#include <mutex>
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "problem.cuh"

namespace cg = cooperative_groups;

namespace dpv {


namespace {

constexpr int kNB = 64;
constexpr int kT = 64;            // tile (rows and cols)
constexpr int kLdS = kNB + 4;     // smem row stride, = 4 (mod 16) doubles
constexpr int kLdP = kNB + 1;     // potrf smem stride

__device__ __forceinline__ void tile_rows(int t, int t_rhs, int64_t N, int64_t& r0, int& nr) {
    if (t == t_rhs) {
        r0 = N;
        nr = 1;
    } else {
        r0 = (int64_t)t * kT;
        nr = (N - r0) < kT ? (int)(N - r0) : kT;
    }
}

// ---------------------------------------------------------------------------
// diagonal block: factor + invert in one CTA (1024 threads)

__global__ void __launch_bounds__(1024) k_potrf_inv(double* __restrict__ A, int64_t ld,
                                                    int64_t N, int64_t c0, int nb,
                                                    double* __restrict__ Linv,
                                                    int32_t* status) {
    extern __shared__ double sm[];
    double* D = sm;                  // 64 x kLdP
    double* X = sm + kNB * kLdP;     // 64 x kLdP inverse
    __shared__ double dinv[kNB];
    const int tid = threadIdx.x;
    const int tx = tid & 63, ty = tid >> 6;   // ty in [0, 16)
    for (int i = ty; i < kNB; i += 16)
        D[i * kLdP + tx] = (tx <= i && i < nb) ? A[(c0 + i) * ld + c0 + tx] : 0.0;
    __syncthreads();
    // T starts as the identity; it becomes the row-unscaled inverse (below)
    for (int i = ty; i < kNB; i += 16) X[i * kLdP + tx] = (i == tx) ? 1.0 : 0.0;
    __syncthreads();
    // Unscaled elimination, one barrier per column.  At step j column j of D
    // and row j of T are final; threads with tx > j update the trailing D,
    // threads with tx <= j update T (forward substitution of L X = I):
    //   D[i][k] -= D[i][j] D[k][j] / d_j,   T[i][c] -= D[i][j] T[j][c] / d_j.
    int bad = -1;
    for (int j = 0; j < nb; ++j) {
        double piv = D[j * kLdP + j];
        if (!(piv > 0.0)) {
            if (bad < 0) bad = j;
            piv = 1.0;
        }
        const double inv = __drcp_rn(piv);
        const double f = (tx > j ? D[tx * kLdP + j] : X[j * kLdP + tx]) * inv;
        double* tgt = tx > j ? D : X;
        if (tx < nb)
            for (int i = j + 1 + ty; i < nb; i += 16)
                if (tx > j ? tx <= i : true) tgt[i * kLdP + tx] -= D[i * kLdP + j] * f;
        __syncthreads();
    }
    // scale: L[i][k] = D[i][k] / sqrt(d_k), diag sqrt(d_k); X[i][c] = T[i][c] / sqrt(d_i)
    if (tid < kNB) {
        const double d = D[tid * kLdP + tid];
        dinv[tid] = (tid < nb && d > 0.0) ? sqrt(d) : 1.0;
    }
    __syncthreads();
    for (int i = ty; i < nb; i += 16) {
        if (tx < i) D[i * kLdP + tx] /= dinv[tx];
        X[i * kLdP + tx] = tx <= i ? X[i * kLdP + tx] / dinv[i] : 0.0;
    }
    __syncthreads();
    if (tid < nb) D[tid * kLdP + tid] = dinv[tid];
    __syncthreads();
    for (int i = ty; i < nb; i += 16)
        if (tx <= i) A[(c0 + i) * ld + c0 + tx] = D[i * kLdP + tx];
    double* out = Linv + (c0 / kNB) * kNB * kNB;
    for (int i = ty; i < kNB; i += 16)
        out[i * kNB + tx] = (i < nb && tx < nb) ? X[i * kLdP + tx] : 0.0;
    if (tid == 0 && bad >= 0 && atomicCAS(status, 0, 1) == 0) status[1] = (int)c0 + bad;
}

// ---------------------------------------------------------------------------
// tensor-core helpers

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

// ---------------------------------------------------------------------------
// Trailing update C -= L_I L_J^T, K = 64 or 128 (one or two panels), over an
// explicit list of 64x64 output tiles (row tile, col tile).  4 warps x 32x32
// on DMMA m8n8k4.  Accumulators start as C (loaded while the first operand
// chunk streams in) and the A fragments are negated, so D = (-L_I) L_J^T + C;
// K streams through a 2-stage cp.async ring of 32-wide chunks.
constexpr int kKC = 32;
constexpr int kLdC = kKC + 4;           // = 4 (mod 16) doubles
constexpr int kStages = 2;

__device__ __forceinline__ void stage_chunk(double* As, double* Bs, const double* __restrict__ A,
                                            int64_t ld, int64_t r0, int nr, int64_t c0t, int nc,
                                            int64_t kc, int64_t kend, int tid) {
    for (int x = tid; x < kT * (kKC / 2); x += 128) {
        const int r = x >> 4, k = (x & 15) * 2;
        const bool kin = kc + k < kend;
        double* da = As + r * kLdC + k;
        double* db = Bs + r * kLdC + k;
        if (r < nr && kin) cp_async16(da, A + (r0 + r) * ld + kc + k);
        else { da[0] = 0.0; da[1] = 0.0; }
        if (r < nc && kin) cp_async16(db, A + (c0t + r) * ld + kc + k);
        else { db[0] = 0.0; db[1] = 0.0; }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}

template <int K>
__global__ void __launch_bounds__(128, 3) k_syrk(double* __restrict__ A, int64_t ld, int64_t N,
                                                 int64_t c0, int kvalid,
                                                 const int2* __restrict__ pairs, int t_rhs) {
    const int2 tp = pairs[blockIdx.x];
    int64_t row0, col0;
    int nr, nc;
    tile_rows(tp.x, t_rhs, N, row0, nr);
    tile_rows(tp.y, t_rhs, N, col0, nc);
    const bool diag = tp.x == tp.y;
    const int64_t kend = c0 + kvalid;
    extern __shared__ double sm[];
    const int tid = threadIdx.x;
    constexpr int NK = K / kKC;
    double* As[kStages] = {sm, sm + 2 * kT * kLdC};
    double* Bs[kStages] = {sm + kT * kLdC, sm + 3 * kT * kLdC};
    stage_chunk(As[0], Bs[0], A, ld, row0, nr, col0, nc, c0, kend, tid);
    const int warp = tid >> 5, lane = tid & 31;
    const int wr = (warp >> 1) * 32, wc = (warp & 1) * 32;
    const int fr = lane >> 2, fk = lane & 3;
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int r = wr + a * 8 + fr;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int cb = wc + b * 8 + 2 * fk;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = cb + h;
                const bool ok = r < nr && c < nc && (!diag || c <= r);
                acc[a][b][h] = ok ? __ldcg(A + (row0 + r) * ld + col0 + c) : 0.0;
            }
        }
    }
#pragma unroll 1
    for (int c = 0; c < NK; ++c) {
        if (c + 1 < NK) {
            stage_chunk(As[(c + 1) & 1], Bs[(c + 1) & 1], A, ld, row0, nr, col0, nc,
                        c0 + (c + 1) * kKC, kend, tid);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        const double* a_s = As[c & 1];
        const double* b_s = Bs[c & 1];
#pragma unroll
        for (int k = 0; k < kKC; k += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) af[a] = -a_s[(wr + a * 8 + fr) * kLdC + k + fk];
#pragma unroll
            for (int b = 0; b < 4; ++b) bf[b] = b_s[(wc + b * 8 + fr) * kLdC + k + fk];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int r = wr + a * 8 + fr;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int cb = wc + b * 8 + 2 * fk;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = cb + h;
                if (r < nr && c < nc && (!diag || c <= r))
                    A[(row0 + r) * ld + col0 + c] = acc[a][b][h];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// L21 = A21 L11^-T on DMMA over the panel's listed row tiles, in place

__global__ void __launch_bounds__(128) k_trsm(double* __restrict__ A, int64_t ld, int64_t N,
                                              int64_t c0, int nb, const double* __restrict__ Linv,
                                              const int* __restrict__ rows, int t_rhs) {
    extern __shared__ double sm[];
    double* As = sm;
    double* Bs = sm + kT * kLdS;
    int64_t row0;
    int nr;
    tile_rows(rows[blockIdx.x], t_rhs, N, row0, nr);
    const double* Li = Linv + (c0 / kNB) * kNB * kNB;
    const int tid = threadIdx.x;
    for (int x = tid; x < kT * (kNB / 2); x += 128) {
        const int r = x >> 5, k = (x & 31) * 2;
        double* da = As + r * kLdS + k;
        if (r < nr && k < nb) cp_async16(da, A + (row0 + r) * ld + c0 + k);
        else { da[0] = 0.0; da[1] = 0.0; }
        cp_async16(Bs + r * kLdS + k, Li + r * kNB + k);   // Bs[n][k] = Linv[n][k]
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    const int warp = tid >> 5, lane = tid & 31;
    const int wr = (warp >> 1) * 32, wc = (warp & 1) * 32;
    const int fr = lane >> 2, fk = lane & 3;
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll 4
    for (int k = 0; k < kNB; k += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) af[a] = As[(wr + a * 8 + fr) * kLdS + k + fk];
#pragma unroll
        for (int b = 0; b < 4; ++b) bf[b] = Bs[(wc + b * 8 + fr) * kLdS + k + fk];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int r = wr + a * 8 + fr;
        if (r >= nr) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int c = wc + b * 8 + 2 * fk;
#pragma unroll
            for (int h = 0; h < 2; ++h)
                if (c + h < nb) A[(row0 + r) * ld + c0 + c + h] = acc[a][b][h];
        }
    }
}

// ---------------------------------------------------------------------------
// backward substitution L^T x = y (y = row N), persistent cooperative kernel

__global__ void __launch_bounds__(256) k_bsub_coop(const double* __restrict__ A, int64_t ld,
                                                   int64_t N, const double* __restrict__ Linv,
                                                   double* __restrict__ part,
                                                   double* __restrict__ x) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double red[4][kNB];
    __shared__ double v[kNB];
    __shared__ double xprev[kNB];
    const int tid = threadIdx.x;
    const int k = tid & 63, rg = tid >> 6;
    const int G = gridDim.x;
    const int np = (int)((N + kNB - 1) / kNB);
    const double* y = A + N * ld;
    for (int p = np - 1; p >= 0; --p) {
        const int64_t c0 = (int64_t)p * kNB;
        const int nb = (N - c0) < kNB ? (int)(N - c0) : kNB;
        const int64_t rs = c0 + nb;              // first row below the block
        const int64_t next_end = (rs + kNB) < N ? rs + kNB : N;
        double acc = 0.0;
        if (k < nb) {
            for (int64_t r = rs + (int64_t)blockIdx.x * 4 + rg; r < N; r += (int64_t)G * 4) {
                const double xr = r < next_end ? xprev[r - rs] : x[r];
                acc += A[r * ld + c0 + k] * xr;
            }
        }
        red[rg][k] = acc;
        __syncthreads();
        double* buf = part + (int64_t)(p & 1) * G * kNB;
        if (tid < kNB) buf[(int64_t)blockIdx.x * kNB + tid] = red[0][tid] + red[1][tid] +
                                                               red[2][tid] + red[3][tid];
        grid.sync();
        if (tid < kNB) {
            double s = 0.0;
            for (int b = 0; b < G; ++b) s += buf[(int64_t)b * kNB + tid];
            v[tid] = tid < nb ? y[c0 + tid] - s : 0.0;
        }
        __syncthreads();
        if (tid < kNB) {
            // x_J = Linv^T v
            const double* Li = Linv + (int64_t)p * kNB * kNB;
            double s = 0.0;
            for (int m = 0; m < nb; ++m) s += Li[m * kNB + tid] * v[m];
            xprev[tid] = s;
            if (blockIdx.x == 0 && tid < nb) x[c0 + tid] = s;
        }
        __syncthreads();
    }
}

// Sparse plans: backward substitution by ONE CTA walking the panels from the
// last, touching only the plan's nonzero row tiles below each diagonal block
// (no grid barriers; ~7 tiles per panel at cfg3).
__global__ void __launch_bounds__(1024) k_bsub_seq(const double* __restrict__ A, int64_t ld,
                                                   int64_t N, const double* __restrict__ Linv,
                                                   const int* __restrict__ rows,
                                                   const int* __restrict__ rows_off, int T,
                                                   double* __restrict__ x) {
    __shared__ double red[16][kNB];
    __shared__ double v[kNB];
    const int tid = threadIdx.x;
    const int k = tid & 63, rg = tid >> 6;
    const double* y = A + N * ld;
    for (int p = T - 1; p >= 0; --p) {
        const int64_t c0 = (int64_t)p * kNB;
        const int nb = (N - c0) < kNB ? (int)(N - c0) : kNB;
        double acc = 0.0;
        if (k < nb) {
            for (int e = rows_off[p]; e < rows_off[p + 1]; ++e) {
                const int t = rows[e];
                if (t >= T) continue;                 // the rhs pseudo-tile
                const int64_t r0 = (int64_t)t * kT;
                const int64_t r1 = (r0 + kT) < N ? r0 + kT : N;
                for (int64_t r = r0 + rg; r < r1; r += 16) acc += A[r * ld + c0 + k] * x[r];
            }
        }
        red[rg][k] = acc;
        __syncthreads();
        if (tid < kNB) {
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < 16; ++q) s += red[q][tid];
            v[tid] = tid < nb ? y[c0 + tid] - s : 0.0;
        }
        __syncthreads();
        if (tid < nb) {
            const double* Li = Linv + (int64_t)p * kNB * kNB;
            double s = 0.0;
            for (int m = 0; m < nb; ++m) s += Li[m * kNB + tid] * v[m];
            x[c0 + tid] = s;
        }
        __syncthreads();
    }
}

struct Ctx {
    cudaStream_t hi = nullptr, lo = nullptr;
    std::vector<cudaEvent_t> ev;
    int coop_blocks = 0;
};

Ctx& ctx() {
    static Ctx c;
    return c;
}

constexpr size_t kPotrfSmem = sizeof(double) * (2 * kNB * kLdP);
constexpr size_t kTileSmem = sizeof(double) * 2 * kT * kLdS;
constexpr size_t kSyrkSmem = sizeof(double) * kStages * 2 * kT * kLdC;

int32_t setup(int64_t ngroups) {
    Ctx& c = ctx();
    if (!c.hi) {
        int lo_prio = 0, hi_prio = 0;
        DPV_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
        DPV_CUDA(cudaStreamCreateWithPriority(&c.hi, cudaStreamNonBlocking, hi_prio));
        DPV_CUDA(cudaStreamCreateWithPriority(&c.lo, cudaStreamNonBlocking, lo_prio));
        static size_t s1 = 0, s2 = 0, s3 = 0, s4 = 0;
        DPV_TRY(ensure_smem(k_potrf_inv, kPotrfSmem, s1));
        DPV_TRY(ensure_smem(k_syrk<64>, kSyrkSmem, s2));
        DPV_TRY(ensure_smem(k_syrk<128>, kSyrkSmem, s3));
        DPV_TRY(ensure_smem(k_trsm, kTileSmem, s4));
        int per_sm = 0;
        DPV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bsub_coop, 256, 0));
        c.coop_blocks = std::max(1, std::min(per_sm, 1) * sm_count());
    }
    while ((int64_t)c.ev.size() < 2 * ngroups + 4) {
        cudaEvent_t e;
        DPV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c.ev.push_back(e);
    }
    return DPV_OK;
}

int32_t launch_syrk(double* A, int64_t ld, int64_t N, int64_t c0, int k, const int2* pairs,
                    int count, int t_rhs, cudaStream_t st) {
    if (count <= 0 || k <= 0) return DPV_OK;
    DPV_TSTART("syrk", st);
    if (k <= 64)
        k_syrk<64><<<count, 128, kSyrkSmem, st>>>(A, ld, N, c0, k, pairs, t_rhs);
    else
        k_syrk<128><<<count, 128, kSyrkSmem, st>>>(A, ld, N, c0, k, pairs, t_rhs);
    DPV_CHECK_LAUNCH();
    return DPV_OK;
}

int32_t factor_panel(double* A, int64_t ld, int64_t N, int p, const FactorPlan& pl,
                     double* linv, int32_t* status, cudaStream_t st) {
    const int64_t c0 = (int64_t)p * kNB;
    const int nb = (int)std::min<int64_t>(kNB, N - c0);
    DPV_TSTART("potrf_inv", st);
    k_potrf_inv<<<1, 1024, kPotrfSmem, st>>>(A, ld, N, c0, nb, linv, status);
    DPV_CHECK_LAUNCH();
    const int cnt = pl.rows_off[p + 1] - pl.rows_off[p];
    if (cnt > 0) {
        DPV_TSTART("trsm", st);
        k_trsm<<<cnt, 128, kTileSmem, st>>>(A, ld, N, c0, nb, linv, pl.d_rows + pl.rows_off[p],
                                            pl.T);
        DPV_CHECK_LAUNCH();
    }
    return DPV_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// plan construction (host): symbolic tile-level fill of the lower pattern

int32_t build_factor_plan(int64_t N, const std::vector<char>* tile_pattern, FactorPlan& pl) {
    const int T = (int)((N + kT - 1) / kT);
    pl.N = N;
    pl.T = T;
    pl.dense = tile_pattern == nullptr;
    std::vector<std::vector<char>> pat(T, std::vector<char>(T, 0));
    for (int i = 0; i < T; ++i)
        for (int j = 0; j <= i; ++j)
            pat[i][j] = pl.dense ? 1 : (*tile_pattern)[(size_t)i * T + j];
    for (int i = 0; i < T; ++i) pat[i][i] = 1;
    // symbolic right-looking fill (block_cholesky.py:93-105 at tile granularity)
    std::vector<std::vector<int>> rows(T);
    for (int j = 0; j < T; ++j) {
        for (int i = j + 1; i < T; ++i)
            if (pat[i][j]) rows[j].push_back(i);
        const auto& r = rows[j];
        for (size_t a = 0; a < r.size(); ++a)
            for (size_t b = 0; b <= a; ++b) pat[r[a]][r[b]] = 1;
    }
    const int t_rhs = T;      // the rhs row N is a dense extra row tile
    std::vector<int> flat_rows;
    pl.rows_off.assign(T + 1, 0);
    for (int p = 0; p < T; ++p) {
        pl.rows_off[p] = (int)flat_rows.size();
        for (int i : rows[p]) flat_rows.push_back(i);
        flat_rows.push_back(t_rhs);
    }
    pl.rows_off[T] = (int)flat_rows.size();
    const int ng = (T + 1) / 2;
    pl.ng = ng;
    std::vector<int2> pairs;
    pl.intra_off.assign(ng + 1, 0);
    pl.next_off.assign(ng + 1, 0);
    pl.rest_off.assign(ng + 1, 0);
    pl.rest_end.assign(ng + 1, 0);
    double flops = 0.0;
    for (int g = 0; g < ng; ++g) {
        const int p0 = 2 * g, p1 = 2 * g + 1;
        pl.intra_off[g] = (int)pairs.size();
        if (p1 < T) {
            for (int i : rows[p0])
                if (i >= p1) pairs.push_back(make_int2(i, p1));
            pairs.push_back(make_int2(t_rhs, p1));
            flops += 2.0 * 64 * 64 * 64 * (rows[p0].size() + 1);
        }
        // row tiles of the group below it
        std::vector<int> rg;
        for (int p : {p0, p1}) {
            if (p >= T) continue;
            for (int i : rows[p])
                if (i > p1) rg.push_back(i);
        }
        std::sort(rg.begin(), rg.end());
        rg.erase(std::unique(rg.begin(), rg.end()), rg.end());
        const int kk = (p1 < T) ? 128 : 64;
        pl.next_off[g] = (int)pairs.size();
        for (int ci : rg) {
            if (ci > p1 + 2) break;
            for (int ri : rg)
                if (ri >= ci) pairs.push_back(make_int2(ri, ci));
            pairs.push_back(make_int2(t_rhs, ci));
        }
        pl.rest_off[g] = (int)pairs.size();
        for (int ci : rg) {
            if (ci <= p1 + 2) continue;
            for (int ri : rg)
                if (ri >= ci) pairs.push_back(make_int2(ri, ci));
            pairs.push_back(make_int2(t_rhs, ci));
        }
        pl.rest_end[g] = (int)pairs.size();
        const double ntile = (double)(pl.rest_end[g] - pl.next_off[g]);
        flops += 2.0 * 64 * 64 * kk * ntile;
    }
    pl.pair_count = (int64_t)pairs.size();
    pl.syrk_flops = flops;
    if (pl.d_rows) cudaFree(pl.d_rows);
    if (pl.d_pairs) cudaFree(pl.d_pairs);
    DPV_CUDA(cudaMalloc(&pl.d_rows, sizeof(int) * std::max<size_t>(1, flat_rows.size())));
    DPV_CUDA(cudaMalloc(&pl.d_pairs, sizeof(int2) * std::max<size_t>(1, pairs.size())));
    DPV_CUDA(cudaMemcpy(pl.d_rows, flat_rows.data(), sizeof(int) * flat_rows.size(),
                        cudaMemcpyHostToDevice));
    if (pl.d_rows_off) cudaFree(pl.d_rows_off);
    DPV_CUDA(cudaMalloc(&pl.d_rows_off, sizeof(int) * pl.rows_off.size()));
    DPV_CUDA(cudaMemcpy(pl.d_rows_off, pl.rows_off.data(), sizeof(int) * pl.rows_off.size(),
                        cudaMemcpyHostToDevice));
    DPV_CUDA(cudaMemcpy(pl.d_pairs, pairs.data(), sizeof(int2) * pairs.size(),
                        cudaMemcpyHostToDevice));
    return DPV_OK;
}

int64_t dense_workspace_doubles(int64_t N) {
    const int64_t np = (N + kNB - 1) / kNB;
    return np * kNB * kNB + 2 * 160 * kNB + 64;
}

// Factor + solve on the augmented matrix following `pl`; x (N) receives
// S^-1 b (in the plan's permuted order).  Panels of 64 columns are grouped
// in pairs so the trailing update runs with K = 128.
int32_t dense_factor_solve(double* A, int64_t ld, int64_t N, int32_t* status, double* x,
                           double* ws, const FactorPlan& pl, cudaStream_t st) {
    DPV_ARG(ld % 8 == 0 && ld >= N + 1, "dense ld must be a multiple of 8 and > N");
    DPV_ARG(pl.N == N, "factor plan built for another size");
    const int T = pl.T, ng = pl.ng;
    // the side streams and events are shared: one enqueuer at a time
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    DPV_TRY(setup(ng));
    Ctx& c = ctx();
    double* linv = ws;
    double* part = ws + (int64_t)T * kNB * kNB;
    cudaEvent_t* evT = c.ev.data();
    cudaEvent_t* evR = c.ev.data() + ng;
    cudaEvent_t fork = c.ev[2 * ng], join_hi = c.ev[2 * ng + 1];
    cudaStream_t hi = c.hi, lo = c.lo;
    DPV_CUDA(cudaEventRecord(fork, st));
    DPV_CUDA(cudaStreamWaitEvent(hi, fork, 0));
    DPV_CUDA(cudaStreamWaitEvent(lo, fork, 0));
    for (int g = 0; g < ng; ++g) {
        const int p0 = 2 * g, p1 = 2 * g + 1;
        const int64_t g0 = (int64_t)p0 * kNB;
        const int64_t g1 = std::min<int64_t>(g0 + 2 * kNB, N);
        DPV_TRY(factor_panel(A, ld, N, p0, pl, linv, status, hi));
        if (p1 < T) {
            DPV_TRY(launch_syrk(A, ld, N, g0, kNB, pl.d_pairs + pl.intra_off[g],
                                pl.next_off[g] - pl.intra_off[g], T, hi));
            DPV_TRY(factor_panel(A, ld, N, p1, pl, linv, status, hi));
        }
        DPV_CUDA(cudaEventRecord(evT[g], hi));
        const int k = (int)(g1 - g0);
        if (g > 0) DPV_CUDA(cudaStreamWaitEvent(hi, evR[g - 1], 0));
        DPV_TRY(launch_syrk(A, ld, N, g0, k, pl.d_pairs + pl.next_off[g],
                            pl.rest_off[g] - pl.next_off[g], T, hi));
        DPV_CUDA(cudaStreamWaitEvent(lo, evT[g], 0));
        DPV_TRY(launch_syrk(A, ld, N, g0, k, pl.d_pairs + pl.rest_off[g],
                            pl.rest_end[g] - pl.rest_off[g], T, lo));
        DPV_CUDA(cudaEventRecord(evR[g], lo));
    }
    DPV_CUDA(cudaEventRecord(join_hi, hi));
    DPV_CUDA(cudaStreamWaitEvent(st, join_hi, 0));
    DPV_CUDA(cudaStreamWaitEvent(st, evR[ng - 1], 0));
    if (!pl.dense && pl.d_rows_off) {
        DPV_TSTART("bsub", st);
        k_bsub_seq<<<1, 1024, 0, st>>>(A, ld, N, linv, pl.d_rows, pl.d_rows_off, T, x);
        DPV_CHECK_LAUNCH();
        return DPV_OK;
    }
    const int G = std::min<int>(c.coop_blocks, 160);
    void* args[] = {&A, &ld, &N, &linv, &part, &x};
    DPV_TSTART("bsub", st);
    DPV_CUDA(cudaLaunchCooperativeKernel((void*)k_bsub_coop, dim3(G), dim3(256), args, 0, st));
    DPV_CHECK_LAUNCH();
    return DPV_OK;
}

}  // namespace dpv
