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
    int bad = -1;
    for (int j = 0; j < nb; ++j) {
        double piv = D[j * kLdP + j];
        if (!(piv > 0.0)) {
            if (bad < 0) bad = j;
            piv = 1.0;
        }
        if (tx > j && tx < nb) {
            const double dk = D[tx * kLdP + j] / piv;
            for (int i = j + 1 + ty; i < nb; i += 16)
                if (tx <= i) D[i * kLdP + tx] -= D[i * kLdP + j] * dk;
        }
        __syncthreads();
    }
    // scale columns: L[i][k] = D[i][k] / sqrt(d_k); diagonal = sqrt(d_k)
    if (tid < kNB) {
        const double d = D[tid * kLdP + tid];
        dinv[tid] = (tid < nb && d > 0.0) ? sqrt(d) : 1.0;
    }
    __syncthreads();
    for (int i = ty; i < nb; i += 16)
        if (tx < i) D[i * kLdP + tx] /= dinv[tx];
    __syncthreads();
    if (tid < nb) D[tid * kLdP + tid] = dinv[tid];
    __syncthreads();
    if (tid < kNB) dinv[tid] = tid < nb ? 1.0 / D[tid * kLdP + tid] : 0.0;
    __syncthreads();
    // X = L^-1 by rows: X[i][c] = -dinv[i] * sum_{c<=m<i} L[i][m] X[m][c], X[i][i] = dinv[i]
    for (int i = 0; i < nb; ++i) {
        // thread (tx = c, ty = part) partial sums over m, reduced across the 16 parts
        double s = 0.0;
        if (tx < i)
            for (int m = tx + ty; m < i; m += 16) s += D[i * kLdP + m] * X[m * kLdP + tx];
        // reduce over ty through shared memory (reuse dinv-free scratch in X's unused row)
        __shared__ double red[16][kNB];
        red[ty][tx] = s;
        __syncthreads();
        if (ty == 0) {
            double t = 0.0;
            for (int q = 0; q < 16; ++q) t += red[q][tx];
            X[i * kLdP + tx] = tx < i ? -dinv[i] * t : (tx == i ? dinv[i] : 0.0);
        }
        __syncthreads();
    }
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
    asm volatile(
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

// columns [col_lo, col_hi), rows [col_lo, N] (row N = rhs); lower tiles only.
// Requires ld % 2 == 0 and 16-byte aligned rows (ld multiple of 8).
__global__ void __launch_bounds__(128) k_syrk(double* __restrict__ A, int64_t ld, int64_t N,
                                              int64_t c0, int nb, int64_t col_lo,
                                              int64_t col_hi) {
    const int ti = blockIdx.y, tj = blockIdx.x;
    if (tj > ti) return;
    const int64_t row0 = col_lo + (int64_t)ti * kT;
    const int64_t col0 = col_lo + (int64_t)tj * kT;
    extern __shared__ double sm[];
    double* As = sm;
    double* Bs = sm + kT * kLdS;
    const int tid = threadIdx.x;
    // async staging of the two 64 x nb panel slices (16-byte chunks)
    for (int x = tid; x < kT * (kNB / 2); x += 128) {
        const int r = x >> 5, k = (x & 31) * 2;
        const int64_t gr = row0 + r, gc = col0 + r;
        double* da = As + r * kLdS + k;
        double* db = Bs + r * kLdS + k;
        if (gr <= N && k < nb) cp_async16(da, A + gr * ld + c0 + k);
        else { da[0] = 0.0; da[1] = 0.0; }
        if (gc < col_hi && k < nb) cp_async16(db, A + gc * ld + c0 + k);
        else { db[0] = 0.0; db[1] = 0.0; }
    }
    const int warp = tid >> 5, lane = tid & 31;
    const int wr = (warp >> 1) * 32, wc = (warp & 1) * 32;
    const int fr = lane >> 2, fk = lane & 3;
    // prefetch this thread's C fragments while the operands stream in
    double cfrag[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int64_t gr = row0 + wr + a * 8 + fr;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int64_t gc = col0 + wc + b * 8 + 2 * fk;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t c = gc + h;
                const bool ok = gr <= N && c < col_hi && (c <= gr || gr == N);
                cfrag[a][b][h] = ok ? A[gr * ld + c] : 0.0;
            }
        }
    }
    cp_async_wait_all();
    __syncthreads();
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
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int64_t gc = col0 + wc + b * 8 + 2 * fk;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t c = gc + h;
                if (gr <= N && c < col_hi && (c <= gr || gr == N))
                    A[gr * ld + c] = cfrag[a][b][h] - acc[a][b][h];
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

int32_t setup(int64_t np) {
    Ctx& c = ctx();
    if (!c.hi) {
        int lo_prio = 0, hi_prio = 0;
        DPV_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
        DPV_CUDA(cudaStreamCreateWithPriority(&c.hi, cudaStreamNonBlocking, hi_prio));
        DPV_CUDA(cudaStreamCreateWithPriority(&c.lo, cudaStreamNonBlocking, lo_prio));
        static size_t s1 = 0, s2 = 0, s3 = 0;
        DPV_TRY(ensure_smem(k_potrf_inv, kPotrfSmem, s1));
        DPV_TRY(ensure_smem(k_syrk, kTileSmem, s2));
        DPV_TRY(ensure_smem(k_trsm, kTileSmem, s3));
        int per_sm = 0;
        DPV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bsub_coop, 256, 0));
        c.coop_blocks = std::max(1, std::min(per_sm, 1) * sm_count());
    }
    while ((int64_t)c.ev.size() < 2 * np + 4) {
        cudaEvent_t e;
        DPV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c.ev.push_back(e);
    }
    return DPV_OK;
}

int32_t launch_syrk(double* A, int64_t ld, int64_t N, int64_t c0, int nb, int64_t lo,
                    int64_t hi, cudaStream_t st) {
    if (hi <= lo) return DPV_OK;
    const int trows = (int)(((N + 1 - lo) + kT - 1) / kT);
    const int tcols = (int)(((hi - lo) + kT - 1) / kT);
    DPV_TSTART("syrk", st);
    k_syrk<<<dim3(tcols, trows), 128, kTileSmem, st>>>(A, ld, N, c0, nb, lo, hi);
    DPV_CHECK_LAUNCH();
    return DPV_OK;
}

}  // namespace

int64_t dense_workspace_doubles(int64_t N) {
    const int64_t np = (N + kNB - 1) / kNB;
    return np * kNB * kNB + 2 * 160 * kNB + 64;
}

// Factor + solve on the augmented matrix; x (N) receives S^-1 b.
int32_t dense_factor_solve(double* A, int64_t ld, int64_t N, int32_t* status, double* x,
                           double* ws, cudaStream_t st) {
    DPV_ARG(ld % 8 == 0 && ld >= N + 1, "dense ld must be a multiple of 8 and > N");
    const int64_t np = (N + kNB - 1) / kNB;
    DPV_TRY(setup(np));
    Ctx& c = ctx();
    double* linv = ws;
    double* part = ws + np * kNB * kNB;
    cudaEvent_t* evT = c.ev.data();
    cudaEvent_t* evR = c.ev.data() + np;
    cudaEvent_t fork = c.ev[2 * np], join_hi = c.ev[2 * np + 1];
    // fork both streams after everything already queued on the caller's stream
    DPV_CUDA(cudaEventRecord(fork, st));
    DPV_CUDA(cudaStreamWaitEvent(c.hi, fork, 0));
    DPV_CUDA(cudaStreamWaitEvent(c.lo, fork, 0));
    for (int64_t p = 0; p < np; ++p) {
        const int64_t c0 = p * kNB;
        const int nb = (int)std::min<int64_t>(kNB, N - c0);
        const int64_t below = (N + 1) - (c0 + nb);
        DPV_TSTART("potrf_inv", c.hi);
        k_potrf_inv<<<1, 1024, kPotrfSmem, c.hi>>>(A, ld, N, c0, nb, linv, status);
        DPV_CHECK_LAUNCH();
        if (below > 0) {
            DPV_TSTART("trsm", c.hi);
            k_trsm<<<(int)((below + kT - 1) / kT), 128, kTileSmem, c.hi>>>(A, ld, N, c0, nb,
                                                                          linv);
            DPV_CHECK_LAUNCH();
        }
        DPV_CUDA(cudaEventRecord(evT[p], c.hi));
        const int64_t s1 = c0 + nb;                       // next panel's first column
        const int64_t s2 = std::min<int64_t>(s1 + kNB, N);
        // look-ahead: the next panel's columns, after the previous rest-update
        if (p > 0) DPV_CUDA(cudaStreamWaitEvent(c.hi, evR[p - 1], 0));
        DPV_TRY(launch_syrk(A, ld, N, c0, nb, s1, s2, c.hi));
        // the rest of the trailing matrix, low priority
        DPV_CUDA(cudaStreamWaitEvent(c.lo, evT[p], 0));
        DPV_TRY(launch_syrk(A, ld, N, c0, nb, s2, N, c.lo));
        DPV_CUDA(cudaEventRecord(evR[p], c.lo));
    }
    // join
    DPV_CUDA(cudaEventRecord(join_hi, c.hi));
    DPV_CUDA(cudaStreamWaitEvent(st, join_hi, 0));
    DPV_CUDA(cudaStreamWaitEvent(st, evR[np - 1], 0));
    const int G = std::min<int>(c.coop_blocks, 160);
    void* args[] = {&A, &ld, &N, &linv, &part, &x};
    DPV_TSTART("bsub", st);
    DPV_CUDA(cudaLaunchCooperativeKernel((void*)k_bsub_coop, dim3(G), dim3(256), args, 0, st));
    DPV_CHECK_LAUNCH();
    return DPV_OK;
}

}  // namespace dpv
