// K4c: dense FP64 Cholesky factor + solve of the damped reduced camera
// system S(lambda) (ba.py:451-472: scipy cho_factor/cho_solve = LAPACK
// potrf/potrs), B200 design:
//
//  * augmented (N+1) x ld row-major lower storage, rhs in row N, so the
//    right-looking factorisation also produces y = L^-1 b;
//  * per 64-column panel, on a high-priority stream (the critical path):
//      potrf_inv: one CTA factors the 64x64 diagonal block in shared memory
//                 (one barrier per column) and inverts it;
//      trsm:      L21 = A21 L11^-T as a DMMA product with the inverse;
//      syrk_next: the next panel's columns of the trailing update;
//  * the rest of the trailing update A22 -= L21 L21^T on a low-priority
//    stream (depth-1 look-ahead), on the FP64 tensor cores
//    (mma.sync.m8n8k4.f64 -> DMMA; tcgen05 has no f64 kind) with cp.async
//    operand staging and C fragments prefetched into registers;
//  * backward substitution L^T x = y: one cooperative persistent kernel, one
//    grid barrier per panel, using the diagonal-block inverses.
#include <cooperative_groups.h>

#include <cstdlib>
#include <vector>

#include "problem.cuh"

namespace cg = cooperative_groups;

namespace dpv {
namespace {

constexpr int kNB = 64;
constexpr int kT = 64;            // SYRK / TRSM output tile (rows and cols)
constexpr int kLdS = kNB + 4;     // smem row stride, = 4 (mod 16) doubles
constexpr int kLdP = kNB + 1;     // potrf smem stride

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
        const double inv = 1.0 / piv;
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
// trailing update on DMMA

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm(
        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// Trailing update C -= L_I L_J^T with K = 64 or 128 (one or two panels):
// columns [col_lo, col_hi), rows [col_lo, N] (row N = rhs), lower tiles
// only.  64x64 tile per CTA, 4 warps x 32x32 on DMMA m8n8k4.  The
// accumulators start as C itself (loaded while the first operand chunk
// streams in) and the A fragments are negated, so D = (-L_I) L_J^T + C needs
// no extra registers; K streams through a 2-stage cp.async ring of 32-wide
// chunks.  ~110 registers and 74 KB of shared memory -> 3 CTAs / SM.
constexpr int kKC = 32;                 // K chunk
constexpr int kLdC = kKC + 4;           // = 4 (mod 16) doubles
constexpr int kStages = 2;

__device__ __forceinline__ void stage_chunk(double* As, double* Bs, const double* __restrict__ A,
                                            int64_t ld, int64_t N, int64_t row0, int64_t col0,
                                            int64_t col_hi, int64_t kc, int64_t kend, int tid) {
    // 64 rows x 32 doubles per operand = 1024 16-byte chunks -> 8 per thread
    for (int x = tid; x < kT * (kKC / 2); x += 128) {
        const int r = x >> 4, k = (x & 15) * 2;
        const int64_t gr = row0 + r, gc = col0 + r;
        const bool kin = kc + k < kend;
        double* da = As + r * kLdC + k;
        double* db = Bs + r * kLdC + k;
        if (gr <= N && kin) cp_async16(da, A + gr * ld + kc + k);
        else { da[0] = 0.0; da[1] = 0.0; }
        if (gc < col_hi && kin) cp_async16(db, A + gc * ld + kc + k);
        else { db[0] = 0.0; db[1] = 0.0; }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}

template <int K>
__global__ void __launch_bounds__(128, 3) k_syrk(double* __restrict__ A, int64_t ld, int64_t N,
                                                 int64_t c0, int kvalid, int64_t col_lo,
                                                 int64_t col_hi) {
    const int ti = blockIdx.y, tj = blockIdx.x;
    if (tj > ti) return;
    const int64_t row0 = col_lo + (int64_t)ti * kT;
    const int64_t col0 = col_lo + (int64_t)tj * kT;
    const int64_t kend = c0 + kvalid;
    extern __shared__ double sm[];
    const int tid = threadIdx.x;
    constexpr int NK = K / kKC;
    double* As[kStages] = {sm, sm + 2 * kT * kLdC};
    double* Bs[kStages] = {sm + kT * kLdC, sm + 3 * kT * kLdC};
    stage_chunk(As[0], Bs[0], A, ld, N, row0, col0, col_hi, c0, kend, tid);
    const int warp = tid >> 5, lane = tid & 31;
    const int wr = (warp >> 1) * 32, wc = (warp & 1) * 32;
    const int fr = lane >> 2, fk = lane & 3;
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int64_t gr = row0 + wr + a * 8 + fr;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int64_t gc = col0 + wc + b * 8 + 2 * fk;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t cc = gc + h;
                const bool ok = gr <= N && cc < col_hi && (cc <= gr || gr == N);
                acc[a][b][h] = ok ? __ldcg(A + gr * ld + cc) : 0.0;
            }
        }
    }
#pragma unroll 1
    for (int c = 0; c < NK; ++c) {
        if (c + 1 < NK) {
            stage_chunk(As[(c + 1) & 1], Bs[(c + 1) & 1], A, ld, N, row0, col0, col_hi,
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
        const int64_t gr = row0 + wr + a * 8 + fr;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int64_t gc = col0 + wc + b * 8 + 2 * fk;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t cc = gc + h;
                if (gr <= N && cc < col_hi && (cc <= gr || gr == N))
                    A[gr * ld + cc] = acc[a][b][h];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// L21 = A21 L11^-T on DMMA: 64 rows per CTA, K = 64, in place

__global__ void __launch_bounds__(128) k_trsm(double* __restrict__ A, int64_t ld, int64_t N,
                                              int64_t c0, int nb, const double* __restrict__ Linv) {
    extern __shared__ double sm[];
    double* As = sm;
    double* Bs = sm + kT * kLdS;
    const int64_t row0 = c0 + nb + (int64_t)blockIdx.x * kT;
    const double* Li = Linv + (c0 / kNB) * kNB * kNB;
    const int tid = threadIdx.x;
    for (int x = tid; x < kT * (kNB / 2); x += 128) {
        const int r = x >> 5, k = (x & 31) * 2;
        const int64_t gr = row0 + r;
        double* da = As + r * kLdS + k;
        if (gr <= N && k < nb) cp_async16(da, A + gr * ld + c0 + k);
        else { da[0] = 0.0; da[1] = 0.0; }
        cp_async16(Bs + r * kLdS + k, Li + r * kNB + k);   // Bs[n][k] = Linv[n][k]
    }
    cp_async_wait_all();
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
        const int64_t gr = row0 + wr + a * 8 + fr;
        if (gr > N) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int c = wc + b * 8 + 2 * fk;
#pragma unroll
            for (int h = 0; h < 2; ++h)
                if (c + h < nb) A[gr * ld + c0 + c + h] = acc[a][b][h];
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

// C[lo:hi cols, rows >= lo] -= L[:, c0:c0+k] L[...]^T, k <= 128 valid columns
int32_t launch_syrk(double* A, int64_t ld, int64_t N, int64_t c0, int k, int64_t lo,
                    int64_t hi, cudaStream_t st) {
    if (hi <= lo || k <= 0) return DPV_OK;
    const int trows = (int)(((N + 1 - lo) + kT - 1) / kT);
    const int tcols = (int)(((hi - lo) + kT - 1) / kT);
    DPV_TSTART("syrk", st);
    if (k <= 64)
        k_syrk<64><<<dim3(tcols, trows), 128, kSyrkSmem, st>>>(A, ld, N, c0, k, lo, hi);
    else
        k_syrk<128><<<dim3(tcols, trows), 128, kSyrkSmem, st>>>(A, ld, N, c0, k, lo, hi);
    DPV_CHECK_LAUNCH();
    return DPV_OK;
}

int32_t factor_panel(double* A, int64_t ld, int64_t N, int64_t p, double* linv,
                     int32_t* status, cudaStream_t st) {
    const int64_t c0 = p * kNB;
    const int nb = (int)std::min<int64_t>(kNB, N - c0);
    const int64_t below = (N + 1) - (c0 + nb);
    DPV_TSTART("potrf_inv", st);
    k_potrf_inv<<<1, 1024, kPotrfSmem, st>>>(A, ld, N, c0, nb, linv, status);
    DPV_CHECK_LAUNCH();
    if (below > 0) {
        DPV_TSTART("trsm", st);
        k_trsm<<<(int)((below + kT - 1) / kT), 128, kTileSmem, st>>>(A, ld, N, c0, nb, linv);
        DPV_CHECK_LAUNCH();
    }
    return DPV_OK;
}

}  // namespace

int64_t dense_workspace_doubles(int64_t N) {
    const int64_t np = (N + kNB - 1) / kNB;
    return np * kNB * kNB + 2 * 160 * kNB + 64;
}

// Factor + solve on the augmented matrix; x (N) receives S^-1 b.  Panels of
// 64 columns are grouped in pairs so the trailing update runs with K = 128.
int32_t dense_factor_solve(double* A, int64_t ld, int64_t N, int32_t* status, double* x,
                           double* ws, cudaStream_t st) {
    DPV_ARG(ld % 8 == 0 && ld >= N + 1, "dense ld must be a multiple of 8 and > N");
    constexpr int kGroup = 2 * kNB;
    const int64_t np = (N + kNB - 1) / kNB;
    const int64_t ng = (N + kGroup - 1) / kGroup;
    DPV_TRY(setup(ng));
    Ctx& c = ctx();
    double* linv = ws;
    double* part = ws + np * kNB * kNB;
    cudaEvent_t* evT = c.ev.data();
    cudaEvent_t* evR = c.ev.data() + ng;
    cudaEvent_t fork = c.ev[2 * ng], join_hi = c.ev[2 * ng + 1];
    static const bool lookahead = !getenv("DPV_CHOL_LOOKAHEAD") ||
                                  atoi(getenv("DPV_CHOL_LOOKAHEAD")) != 0;
    cudaStream_t hi = lookahead ? c.hi : st, lo = lookahead ? c.lo : st;
    DPV_CUDA(cudaEventRecord(fork, st));
    DPV_CUDA(cudaStreamWaitEvent(hi, fork, 0));
    DPV_CUDA(cudaStreamWaitEvent(lo, fork, 0));
    for (int64_t g = 0; g < ng; ++g) {
        const int64_t g0 = g * kGroup;                       // group columns [g0, g1)
        const int64_t g1 = std::min<int64_t>(g0 + kGroup, N);
        const int64_t p0 = g0 / kNB;
        // first panel, intra-group update of the second panel, second panel
        DPV_TRY(factor_panel(A, ld, N, p0, linv, status, hi));
        if (g0 + kNB < g1) {
            DPV_TRY(launch_syrk(A, ld, N, g0, kNB, g0 + kNB, g1, hi));
            DPV_TRY(factor_panel(A, ld, N, p0 + 1, linv, status, hi));
        }
        DPV_CUDA(cudaEventRecord(evT[g], hi));
        const int k = (int)(g1 - g0);
        const int64_t n1 = std::min<int64_t>(g1 + kGroup, N);   // next group's columns
        // look-ahead: the next group's columns, after the previous rest-update
        if (g > 0) DPV_CUDA(cudaStreamWaitEvent(hi, evR[g - 1], 0));
        DPV_TRY(launch_syrk(A, ld, N, g0, k, g1, n1, hi));
        // the rest of the trailing matrix, low priority
        DPV_CUDA(cudaStreamWaitEvent(lo, evT[g], 0));
        DPV_TRY(launch_syrk(A, ld, N, g0, k, n1, N, lo));
        DPV_CUDA(cudaEventRecord(evR[g], lo));
    }
    DPV_CUDA(cudaEventRecord(join_hi, hi));
    DPV_CUDA(cudaStreamWaitEvent(st, join_hi, 0));
    DPV_CUDA(cudaStreamWaitEvent(st, evR[ng - 1], 0));
    const int G = std::min<int>(c.coop_blocks, 160);
    void* args[] = {&A, &ld, &N, &linv, &part, &x};
    DPV_TSTART("bsub", st);
    DPV_CUDA(cudaLaunchCooperativeKernel((void*)k_bsub_coop, dim3(G), dim3(256), args, 0, st));
    DPV_CHECK_LAUNCH();
    return DPV_OK;
}

}  // namespace dpv
