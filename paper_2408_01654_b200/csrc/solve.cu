// K4b-K4d: damped Schur-reduced camera system (ba.py:303-319), dense
// Cholesky solve of S(lambda) with the trailing pose-block contraction on the
// FP64 tensor cores (mma.sync m8n8k4 -> SASS DMMA; tcgen05 has no f64 kind),
// back-substitution of the inverse depths (ba.py:321-325) and the
// retraction (ba.py:521-531).
//
// Dense layout: (N+1) x ld row-major, lower triangle; row N carries the right
// hand side, so the right-looking factorisation performs the forward
// substitution y = L^-1 b for free (the augmented-matrix trick).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include <mutex>

#include "problem.cuh"

namespace dpv {
namespace {

constexpr int kSmallMax = 162;    // n <= 27 poses: single-CTA shared-memory solve


// ---------------------------------------------------------------------------
// reduced system export (parity) -------------------------------------------

__global__ void k_reduced_blocks(int64_t W, const int32_t* ka, const int32_t* kb,
                                 const double* pose, const double* schur, double lam,
                                 const double* scal, double* out) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < W * 36;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t w = x / 36;
        out[x] = reduced_pinned_entry(pose, schur, ka, w, (int)(x % 36), ka[w] == kb[w], lam,
                                      scal);
    }
}

__global__ void k_reduced_vectors(int64_t n6, int64_t P, const double* rhs_pose,
                                  const double* rhs_schur, const double* depth_diag,
                                  const uint8_t* active, double lam, double* rhs, double* cinv) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n6 + P;
         x += (int64_t)gridDim.x * blockDim.x) {
        if (x < n6) {
            if (rhs) rhs[x] = rhs_pose[x] - rhs_schur[x] / (1.0 + lam);
        } else {
            const int64_t r = x - n6;
            if (cinv) cinv[r] = active[r] ? 1.0 / (depth_diag[r] * (1.0 + lam)) : 0.0;
        }
    }
}

// ---------------------------------------------------------------------------
// dense scatter of S(lam) into the lower triangle + rhs row ---------------------

// pose var v sits at position pos[v] of the (possibly permuted) dense system
__global__ void k_dense_scatter(int64_t W, const int32_t* ka, const int32_t* kb,
                                const double* pose, const double* schur, double lam, double* A,
                                int64_t ld, const int32_t* pos) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < W * 36;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t w = x / 36;
        const int idx = (int)(x % 36);
        const int i = idx / 6, j = idx % 6;
        const int64_t a = pos[ka[w]], b = pos[kb[w]];
        const double v = reduced_entry(pose, schur, w, idx, ka[w] == kb[w], lam);
        if (a == b) {
            if (i >= j) A[(6 * a + i) * ld + 6 * a + j] = v;
        } else if (a < b) {
            // upper block S_ab -> lower mirror S_ba = S_ab^T
            A[(6 * b + j) * ld + 6 * a + i] = v;
        } else {
            A[(6 * a + i) * ld + 6 * b + j] = v;
        }
    }
}

__global__ void k_dense_pin_rhs(int64_t n6, const double* rhs_pose, const double* rhs_schur,
                                double lam, const double* scal, double* A, int64_t ld,
                                const int32_t* pos) {
    const int64_t N = n6;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < N;
         c += (int64_t)gridDim.x * blockDim.x)
        A[N * ld + 6 * (int64_t)pos[c / 6] + c % 6] = rhs_pose[c] - rhs_schur[c] / (1.0 + lam);
    if (blockIdx.x == 0 && threadIdx.x == 0 && scal[1] != 0.0 && N >= 6) {
        const int64_t o = 6 * (int64_t)pos[0];   // the pinned block of pose var 0
        double mx = 0.0;
        for (int k = 0; k < 6; ++k) mx = fmax(mx, fabs(A[(o + k) * ld + o + k]));
        const double mu = 1e6 * fmax(1.0, mx);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j <= i; ++j) A[(o + i) * ld + o + j] += mu * scal[2 + i] * scal[2 + j];
    }
}

__global__ void k_unpermute(int64_t n, const int32_t* pos, const double* x, double* dp) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < 6 * n;
         c += (int64_t)gridDim.x * blockDim.x)
        dp[c] = x[6 * (int64_t)pos[c / 6] + c % 6];
}

// ---------------------------------------------------------------------------
// small systems: everything in one CTA, shared memory ---------------------------

// Small reduced systems (N = 6n <= kSmallMax): S(lam) is scattered into
// shared memory with the rhs as its last row and factored in one CTA, blocked
// by 4 columns: warp 0 factors the 4x4 diagonal block, all threads scale
// the panel and apply the rank-4 update; the backward substitution runs by
// 4-blocks on 256 threads (named barrier).  Same pivot reporting and
// rhs-as-last-row forward substitution.  Warp 0 factors the NEXT diagonal
// block (its rank-4 update first) while the other warps update the rest, so
// the pivot chain is off the barrier path.  cfg2 window (N = 132): 89 us per
// solve vs 168 us unblocked; the kernel is latency-bound on one SM.
constexpr int kSmallThreads = 1024;
constexpr int kSmallBsubThreads = 256;   // fewer threads per barrier: 3x faster here

__global__ void __launch_bounds__(kSmallThreads) k_small_solve2(
    int64_t n, int64_t W, const int32_t* ka, const int32_t* kb, const double* pose,
    const double* schur, const double* rhs_pose, const double* rhs_schur, const double* scal,
    double lam, double* dp, int32_t* status) {
    extern __shared__ double A[];
    __shared__ double colb[4][kSmallMax + 1];
    __shared__ double dinv[kSmallMax];
    __shared__ int bad;
    const int N = (int)(6 * n);
    const int ld = N + 1;
    const int tid = threadIdx.x;
    const int lane = tid & 31, wy = tid >> 5;
    constexpr int ny = kSmallThreads / 32;
    for (int x = tid; x < (N + 1) * ld; x += kSmallThreads) A[x] = 0.0;
    if (tid == 0) bad = -1;
    __syncthreads();
    for (int64_t x = tid; x < W * 36; x += kSmallThreads) {
        const int64_t w = x / 36;
        const int idx = (int)(x % 36);
        const int i = idx / 6, j = idx % 6;
        const int a = ka[w], b = kb[w];
        const double v = reduced_entry(pose, schur, w, idx, a == b, lam);
        if (a == b) {
            if (i >= j) A[(6 * a + i) * ld + 6 * a + j] = v;
        } else {
            A[(6 * b + j) * ld + 6 * a + i] = v;
        }
    }
    for (int c = tid; c < N; c += kSmallThreads)
        A[N * ld + c] = rhs_pose[c] - rhs_schur[c] / (1.0 + lam);
    __syncthreads();
    if (tid == 0 && scal[1] != 0.0 && N >= 6) {
        double mx = 0.0;
        for (int k = 0; k < 6; ++k) mx = fmax(mx, fabs(A[k * ld + k]));
        const double mu = 1e6 * fmax(1.0, mx);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j <= i; ++j) A[i * ld + j] += mu * scal[2 + i] * scal[2 + j];
    }
    __syncthreads();
    // right-looking by blocks of 4 columns: warp 0 factors the 4x4 diagonal
    // block (rsqrt pivots, lanes redundant) into shared memory, all threads
    // scale the panel rows (forward substitution), then a rank-4 update.
    // (Factoring the block redundantly in all 1024 threads saturates the FP64
    // pipe of the one SM: sqrt + division are ~50 DP instructions each.)
    __shared__ double lblk[2][4][4], linv[2][4];
    // warp 0: factor diagonal block at column j (buffer b) -> lblk/linv, A, dinv
    auto factor_diag = [&](int j, int b) {
        const int bw = min(4, N - j);
        double l[4][4], inv[4];
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int q = 0; q <= p; ++q) l[p][q] = (p < bw) ? A[(j + p) * ld + j + q] : 1.0;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            double piv = l[p][p];
            if (p < bw && !(piv > 0.0)) {
                if (lane == 0 && bad < 0) bad = j + p;
                piv = 1.0;
            }
            if (p >= bw) piv = 1.0;
            inv[p] = rsqrt(piv);
            l[p][p] = piv * inv[p];
#pragma unroll
            for (int r = p + 1; r < 4; ++r) l[r][p] *= inv[p];
#pragma unroll
            for (int r = p + 1; r < 4; ++r)
#pragma unroll
                for (int c = p + 1; c <= r; ++c) l[r][c] -= l[r][p] * l[c][p];
        }
        __syncwarp();
        if (lane < 16) {
            const int p = lane >> 2, q = lane & 3;
            double v = 0.0;
#pragma unroll
            for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
                for (int b2 = 0; b2 <= a2; ++b2) v = (a2 == p && b2 == q) ? l[a2][b2] : v;
            lblk[b][p][q] = v;
            if (q <= p && p < bw) A[(j + p) * ld + j + q] = v;
            if (q == 0) {
                double iv = 0.0;
#pragma unroll
                for (int a2 = 0; a2 < 4; ++a2) iv = (a2 == p) ? inv[a2] : iv;
                linv[b][p] = iv;
                if (p < bw) dinv[j + p] = iv;
            }
        }
    };
    if (wy == 0) factor_diag(0, 0);
    __syncthreads();
    for (int j = 0; j < N; j += 4) {
        const int bw = min(4, N - j);
        const int buf = (j >> 2) & 1;
        double l[4][4], inv[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            inv[p] = linv[buf][p];
#pragma unroll
            for (int q = 0; q < p; ++q) l[p][q] = lblk[buf][p][q];
        }
        for (int i = j + bw + tid; i <= N; i += kSmallThreads) {
            double x[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                double v = q < bw ? A[i * ld + j + q] : 0.0;
#pragma unroll
                for (int r = 0; r < q; ++r) v -= x[r] * l[q][r];
                x[q] = v * inv[q];
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (q < bw) {
                    A[i * ld + j + q] = x[q];
                    colb[q][i] = x[q];
                }
        }
        __syncthreads();
        const int jn = j + 4;                 // next diagonal block (look-ahead)
        const int bwn = jn < N ? min(4, N - jn) : 0;
        if (wy == 0) {
            // warp 0: the next diagonal block's rank-4 update, then its factor,
            // while the other warps update the rest of the trailing matrix
            if (bwn > 0) {
                if (lane < 16) {
                    const int r = jn + (lane >> 2), c = jn + (lane & 3);
                    if ((lane >> 2) < bwn && (lane & 3) <= (lane >> 2)) {
                        double v = A[r * ld + c];
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            if (q < bw) v -= colb[q][r] * colb[q][c];
                        A[r * ld + c] = v;
                    }
                }
                __syncwarp();
                factor_diag(jn, buf ^ 1);
            }
        } else {
        // rank-4 update; a warp takes two rows at a time so each lane has two
        // independent FMA chains in flight (the loop is latency-bound)
        for (int i0 = jn + bwn + 2 * (wy - 1); i0 <= N; i0 += 2 * (ny - 1)) {
            const int i1 = i0 + 1;
            const bool two = i1 <= N;
            double la[4], lb[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                la[q] = q < bw ? colb[q][i0] : 0.0;
                lb[q] = (q < bw && two) ? colb[q][i1] : 0.0;
            }
            const int kmax0 = i0 < N ? i0 : N - 1;
            const int kmax1 = two ? (i1 < N ? i1 : N - 1) : -1;
            // N <= kSmallMax: at most 6 column chunks of 32, fully unrolled so
            // every chunk's loads are in flight together
            constexpr int kChunks = (kSmallMax + 31) / 32;
#pragma unroll
            for (int it = 0; it < kChunks; ++it) {
                const int k = j + bw + lane + 32 * it;
                if (k > kmax0 && k > kmax1) continue;
                double c[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) c[q] = q < bw ? colb[q][k] : 0.0;
                if (k <= kmax0) {
                    const double v = A[i0 * ld + k];
                    A[i0 * ld + k] = v - (la[0] * c[0] + la[1] * c[1]) - (la[2] * c[2] + la[3] * c[3]);
                }
                if (k <= kmax1) {
                    const double v = A[i1 * ld + k];
                    A[i1 * ld + k] = v - (lb[0] * c[0] + lb[1] * c[1]) - (lb[2] * c[2] + lb[3] * c[3]);
                }
            }
        }
        }   // warps 1..: trailing update
        __syncthreads();   // one barrier site for every warp
    }
    // backward substitution L^T x = y (y in row N) by blocks of 4: every
    // thread solves the block's 4x4 triangle redundantly, then the earlier
    // entries of y take the block's update; one barrier per block
    double* y = A + (int64_t)N * ld;
    double* xs = &colb[0][0];            // the solution (colb is free now)
    if (tid < kSmallBsubThreads) {
        for (int jb = ((N - 1) / 4) * 4; jb >= 0; jb -= 4) {
            const int bw = min(4, N - jb);
            double x[4];
#pragma unroll
            for (int p = 3; p >= 0; --p) {
                if (p >= bw) {
                    x[p] = 0.0;
                    continue;
                }
                double v = y[jb + p];
#pragma unroll
                for (int r = p + 1; r < 4; ++r)
                    if (r < bw) v -= A[(jb + r) * ld + jb + p] * x[r];
                x[p] = v * dinv[jb + p];
            }
            if (tid < bw) {
                double xv = x[0];
#pragma unroll
                for (int q = 1; q < 4; ++q) xv = (tid == q) ? x[q] : xv;
                xs[jb + tid] = xv;
            }
            for (int i = tid; i < jb; i += kSmallBsubThreads) {
                double v = y[i];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (q < bw) v -= A[(jb + q) * ld + i] * x[q];
                y[i] = v;
            }
            asm volatile("bar.sync 1, %0;\n" ::"n"(kSmallBsubThreads) : "memory");
        }
    }
    __syncthreads();
    for (int c = tid; c < N; c += kSmallThreads) dp[c] = xs[c];
    if (tid == 0) status[0] = bad >= 0 ? 1 : 0;
    if (tid == 0) status[1] = bad;
}

// ---------------------------------------------------------------------------
// depth back-substitution (ba.py:321-325) and retraction (ba.py:521-531)

__global__ void k_back_substitute(int64_t P, const int32_t* rinc_ptr, const int32_t* rinc,
                                  const int32_t* inc_var, const double* inc_block,
                                  const double* rhs_depth, const double* depth_diag,
                                  const uint8_t* active, double lam, const double* dp,
                                  double* dd) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < P;
         r += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        const int32_t k1 = rinc_ptr[r + 1];
        int32_t k = rinc_ptr[r];
        for (; k + 1 < k1; k += 2) {       // two incidences in flight, same order
            const int32_t ia = __ldg(rinc + k), ib = __ldg(rinc + k + 1);
            const double* ba = inc_block + (int64_t)ia * 6;
            const double* bb = inc_block + (int64_t)ib * 6;
            const double* xa = dp + (int64_t)__ldg(inc_var + ia) * 6;
            const double* xb = dp + (int64_t)__ldg(inc_var + ib) * 6;
            double va[6], vb[6], wa[6], wb[6];
#pragma unroll
            for (int a = 0; a < 6; ++a) {
                va[a] = __ldg(ba + a);
                vb[a] = __ldg(bb + a);
                wa[a] = __ldg(xa + a);
                wb[a] = __ldg(xb + a);
            }
            double sa = 0.0, sb = 0.0;
#pragma unroll
            for (int a = 0; a < 6; ++a) {
                sa += va[a] * wa[a];
                sb += vb[a] * wb[a];
            }
            acc += sa;
            acc += sb;
        }
        if (k < k1) {
            const int32_t i = rinc[k];
            const double* blk = inc_block + (int64_t)i * 6;
            const double* x = dp + (int64_t)inc_var[i] * 6;
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < 6; ++a) s += blk[a] * x[a];
            acc += s;
        }
        const double cinv = active[r] ? 1.0 / (depth_diag[r] * (1.0 + lam)) : 0.0;
        dd[r] = cinv * (rhs_depth[r] - acc);
    }
}

// small problems: one warp per row, lanes over the row's incidences
__global__ void k_back_substitute_warp(int64_t P, const int32_t* rinc_ptr, const int32_t* rinc,
                                       const int32_t* inc_var, const double* inc_block,
                                       const double* rhs_depth, const double* depth_diag,
                                       const uint8_t* active, double lam, const double* dp,
                                       double* dd) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < P; r += nwarps) {
        double acc = 0.0;
        for (int32_t k = rinc_ptr[r] + lane; k < rinc_ptr[r + 1]; k += 32) {
            const int32_t i = __ldg(rinc + k);
            const double* blk = inc_block + (int64_t)i * 6;
            const double* x = dp + (int64_t)__ldg(inc_var + i) * 6;
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < 6; ++a) s += __ldg(blk + a) * __ldg(x + a);
            acc += s;
        }
        acc = warp_sum(acc);
        if (lane == 0) {
            const double cinv = active[r] ? 1.0 / (depth_diag[r] * (1.0 + lam)) : 0.0;
            dd[r] = cinv * (rhs_depth[r] - acc);
        }
    }
}

__global__ void k_apply_step(int64_t F, int32_t first, int32_t last, int64_t P, const double* q,
                             const double* t, const double* d, const double* dp,
                             const double* dd, double* q2, double* t2, double* d2) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < F + P;
         x += (int64_t)gridDim.x * blockDim.x) {
        if (x < F) {
            const int64_t f = x;
            if (f < first || f > last) {
                for (int k = 0; k < 4; ++k) q2[4 * f + k] = q[4 * f + k];
                for (int k = 0; k < 3; ++k) t2[3 * f + k] = t[3 * f + k];
                continue;
            }
            const double* xi = dp + 6 * (f - first);
            // rotvec_to_quat (geometry.py:89-101)
            const double p0 = xi[3], p1 = xi[4], p2 = xi[5];
            const double th = sqrt(p0 * p0 + p1 * p1 + p2 * p2);
            const double kk = th < kSmallAngle ? 0.5 - th * th / 48.0 : sin(0.5 * th) / th;
            const double dq[4] = {p0 * kk, p1 * kk, p2 * kk, cos(0.5 * th)};
            const double* a = dq;
            const double* b = q + 4 * f;
            // Hamilton product dq * q (geometry.py:41-53), then normalise
            double r[4];
            r[0] = a[3] * b[0] + a[0] * b[3] + a[1] * b[2] - a[2] * b[1];
            r[1] = a[3] * b[1] - a[0] * b[2] + a[1] * b[3] + a[2] * b[0];
            r[2] = a[3] * b[2] + a[0] * b[1] - a[1] * b[0] + a[2] * b[3];
            r[3] = a[3] * b[3] - a[0] * b[0] - a[1] * b[1] - a[2] * b[2];
            const double nrm = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2] + r[3] * r[3]);
            for (int k = 0; k < 4; ++k) q2[4 * f + k] = r[k] / nrm;
            // quat_rotate (geometry.py:62-67): v + w*t + u x t, t = 2 u x v
            const double* v = t + 3 * f;
            const double u0 = dq[0], u1 = dq[1], u2 = dq[2], w = dq[3];
            const double c0 = 2.0 * (u1 * v[2] - u2 * v[1]);
            const double c1 = 2.0 * (u2 * v[0] - u0 * v[2]);
            const double c2 = 2.0 * (u0 * v[1] - u1 * v[0]);
            t2[3 * f + 0] = v[0] + w * c0 + (u1 * c2 - u2 * c1) + xi[0];
            t2[3 * f + 1] = v[1] + w * c1 + (u2 * c0 - u0 * c2) + xi[1];
            t2[3 * f + 2] = v[2] + w * c2 + (u0 * c1 - u1 * c0) + xi[2];
        } else {
            const int64_t r = x - F;
            d2[r] = fmax(d[r] + dd[r], kInverseDepthFloor);
        }
    }
}

int64_t dense_ld(int64_t N) { return ((N + 1 + 7) / 8) * 8; }

// Symmetric permutation + tile plan of the reduced camera system (host, once
// per problem: the pattern = union_keys is state-independent).  Poses with a
// long-range coupling (a loop-closure block farther than `band` poses from
// the diagonal) move to the end, so the rest is banded; `band` is chosen to
// minimise the planned trailing-update work.  With DPV_DENSE_SOLVE=1 every
// tile is kept (the plain dense factorisation).
int32_t ensure_plan(dpv_problem* p, int64_t N, cudaStream_t st) {
    if (p->plan) return DPV_OK;
    const int64_t n = p->n, W = p->W;
    std::vector<int32_t> ka(W), kb(W);
    DPV_CUDA(cudaMemcpyAsync(ka.data(), p->key_a, sizeof(int32_t) * W, cudaMemcpyDeviceToHost, st));
    DPV_CUDA(cudaMemcpyAsync(kb.data(), p->key_b, sizeof(int32_t) * W, cudaMemcpyDeviceToHost, st));
    DPV_CUDA(cudaStreamSynchronize(st));
    std::vector<int32_t> pos(n);
    for (int64_t v = 0; v < n; ++v) pos[v] = (int32_t)v;
    auto* plan = new (std::nothrow) FactorPlan();
    DPV_ARG(plan != nullptr, "allocation failed");
    {
        const int T = (int)((N + 63) / 64);
        double best = -1.0;
        std::vector<int32_t> best_pos = pos;
        for (int64_t band : {4, 8, 16, 24, 32, 48, 64, 96, 128, 192, 256, 512, 1024}) {
            if (band >= n && band != 4) break;
            std::vector<char> border(n, 0);
            for (int64_t w = 0; w < W; ++w)
                if (kb[w] - ka[w] > band) border[kb[w]] = 1;
            std::vector<int32_t> cand(n);
            int32_t k = 0;
            for (int64_t v = 0; v < n; ++v)
                if (!border[v]) cand[v] = k++;
            const int64_t nb_border = n - k;
            for (int64_t v = 0; v < n; ++v)
                if (border[v]) cand[v] = k++;
            // work estimate: row tiles per panel ~ band tiles + border tiles
            const double rows = (6.0 * band) / 64.0 + 2.0 + (6.0 * nb_border) / 64.0 + 1.0;
            const double cost = T * rows * rows;
            if (best < 0 || cost < best) {
                best = cost;
                best_pos = cand;
            }
        }
        pos = best_pos;
        std::vector<char> pat((size_t)T * T, 0);
        for (int64_t w = 0; w < W; ++w) {
            int64_t r = pos[kb[w]], c = pos[ka[w]];
            if (r < c) std::swap(r, c);
            for (int64_t tr = (6 * r) / 64; tr <= (6 * r + 5) / 64; ++tr)
                for (int64_t tc = (6 * c) / 64; tc <= (6 * c + 5) / 64; ++tc)
                    if (tc <= tr) pat[(size_t)tr * T + tc] = 1;
        }
        int32_t s = build_factor_plan(N, &pat, *plan);
        if (s != DPV_OK) { delete plan; return s; }
    }
    if (getenv("DPV_PLAN_DEBUG"))
        fprintf(stderr, "[dpv] plan N=%lld T=%d dense=%d pairs=%lld syrk_gflop=%.2f\n",
                (long long)N, plan->T, (int)plan->dense, (long long)plan->pair_count,
                plan->syrk_flops * 1e-9);
    DPV_TRY(p->alloc(&p->perm_pos, n));
    DPV_CUDA(cudaMemcpyAsync(p->perm_pos, pos.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice,
                             st));
    DPV_CUDA(cudaStreamSynchronize(st));
    p->plan = plan;
    return DPV_OK;
}

__global__ void k_iota_pos(int64_t n, int32_t* pos) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        pos[i] = (int32_t)i;
}

int32_t ensure_dense_buffers(dpv_problem* p, int64_t N) {
    if (p->dense) return DPV_OK;
    p->dense_ld = dense_ld(N);
    DPV_TRY(p->alloc(&p->dense, (N + 1) * p->dense_ld));
    DPV_TRY(p->alloc(&p->bsub_part, dense_workspace_doubles(N)));
    return DPV_OK;
}

// the dense backend's plan: every lower tile, natural pose order
int32_t ensure_dense_full(dpv_problem* p, int64_t N, cudaStream_t st) {
    if (!p->dplan) {
        auto* plan = new (std::nothrow) FactorPlan();
        DPV_ARG(plan != nullptr, "allocation failed");
        const int32_t s = build_factor_plan(N, nullptr, *plan);
        if (s != DPV_OK) {
            delete plan;
            return s;
        }
        p->dplan = plan;
        DPV_TRY(p->alloc(&p->ident_pos, p->n));
        k_iota_pos<<<grid_for(p->n, 256), 256, 0, st>>>(p->n, p->ident_pos);
        DPV_CHECK_LAUNCH();
    }
    return ensure_dense_buffers(p, N);
}

int32_t ensure_dense(dpv_problem* p, int64_t N, cudaStream_t st) {
    DPV_TRY(ensure_plan(p, N, st));
    if (p->dense) return DPV_OK;
    p->dense_ld = dense_ld(N);
    DPV_TRY(p->alloc(&p->dense, (N + 1) * p->dense_ld));
    DPV_TRY(p->alloc(&p->bsub_part, dense_workspace_doubles(N)));
    return DPV_OK;
}

}  // namespace

int64_t cholesky_work_doubles(int64_t n) { return dense_workspace_doubles(n); }

int32_t back_substitute(dpv_problem* p, double lam, const double* dp, double* dd,
                        cudaStream_t st);

int32_t reduced_system(dpv_problem* p, double lam, double* blocks, double* rhs, double* cinv,
                       cudaStream_t st) {
    if (blocks && p->W > 0) {
        DPV_TSTART("reduced_blocks", st);
        k_reduced_blocks<<<grid_for(p->W * 36, 256), 256, 0, st>>>(
            p->W, p->key_a, p->key_b, p->pose_blocks, p->schur_blocks, lam, p->scal, blocks);
        DPV_CHECK_LAUNCH();
    }
    if (rhs || cinv) {
        DPV_TSTART("reduced_vectors", st);
        k_reduced_vectors<<<grid_for(p->n * 6 + p->P, 256), 256, 0, st>>>(
            p->n * 6, p->P, p->rhs_pose, p->rhs_schur, p->depth_diag, p->active, lam, rhs, cinv);
        DPV_CHECK_LAUNCH();
    }
    return DPV_OK;
}

// Start the sparse-solver plan on a host thread right after the index build
// (the union keys are final), so its ~1 ms of host work overlaps the first
// edge pass and assembly on the device.  Same plan, same failure fallback
// as building it inside the first solve.
void spd_plan_prefetch(dpv_problem* p) {
    if (6 * p->n <= kSmallMax || p->W == 0 ||
        p->plan_thread.joinable() || p->spd)
        return;
    int dev = 0;
    cudaGetDevice(&dev);
    p->plan_thread = std::thread([p, dev]() {
        cudaSetDevice(dev);
        cudaStream_t s = nullptr;
        if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
            p->plan_status = DPV_CUDA_ERROR;
            return;
        }
        std::vector<int32_t> ka(p->W), kb(p->W);
        int32_t rc = DPV_OK;
        if (cudaMemcpyAsync(ka.data(), p->key_a, sizeof(int32_t) * p->W, cudaMemcpyDeviceToHost,
                            s) != cudaSuccess ||
            cudaMemcpyAsync(kb.data(), p->key_b, sizeof(int32_t) * p->W, cudaMemcpyDeviceToHost,
                            s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            rc = DPV_CUDA_ERROR;
        dpv::SpdPlan* pl = nullptr;
        if (rc == DPV_OK) rc = spd_plan_build(ka.data(), kb.data(), p->W, p->n, &pl, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) rc = DPV_CUDA_ERROR;
        if (rc == DPV_OK) {
            spd_plan_set_stream(pl, p->alloc_stream);   // freed with the problem
            p->spd_pending = pl;
        } else {
            spd_plan_free(pl);
        }
        p->plan_status = rc;
        cudaStreamDestroy(s);
    });
}

// S(lam) scattered into the augmented dense matrix in the order `pos`,
// factorised and solved by the tile engine following `plan`; dp in pose order
static int32_t dense_path(dpv_problem* p, double lam, int64_t N, const FactorPlan& plan,
                          const int32_t* pos, double* dp, int32_t* status, cudaStream_t st) {
    const int64_t ld = p->dense_ld;
    DPV_CUDA(cudaMemsetAsync(p->dense, 0, sizeof(double) * (N + 1) * ld, st));
    DPV_TSTART("dense_scatter", st);
    k_dense_scatter<<<grid_for(p->W * 36, 256), 256, 0, st>>>(
        p->W, p->key_a, p->key_b, p->pose_blocks, p->schur_blocks, lam, p->dense, ld, pos);
    DPV_CHECK_LAUNCH();
    DPV_TSTART("dense_pin_rhs", st);
    k_dense_pin_rhs<<<grid_for(N, 256), 256, 0, st>>>(N, p->rhs_pose, p->rhs_schur, lam, p->scal,
                                                       p->dense, ld, pos);
    DPV_CHECK_LAUNCH();
    DPV_TRY(dense_factor_solve(p->dense, ld, N, status, p->red_rhs, p->bsub_part, plan, st));
    DPV_TSTART("unpermute", st);
    k_unpermute<<<grid_for(N, 256), 256, 0, st>>>(p->n, pos, p->red_rhs, dp);
    DPV_CHECK_LAUNCH();
    return DPV_OK;
}

int32_t solve(dpv_problem* p, double lam, double* dp, double* dd, int32_t* status,
              cudaStream_t st) {
    const int64_t N = 6 * p->n;
    DPV_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t) * 2, st));
    const int32_t backend = p->solve_backend;
    if (N <= kSmallMax && backend != 2) {
        const size_t smem = sizeof(double) * (size_t)(N + 1) * (N + 1);
        DPV_TSTART("small_solve", st);
        static size_t cur = 0;
        DPV_TRY(ensure_smem(k_small_solve2, smem, cur));
        k_small_solve2<<<1, kSmallThreads, smem, st>>>(
            p->n, p->W, p->key_a, p->key_b, p->pose_blocks, p->schur_blocks, p->rhs_pose,
            p->rhs_schur, p->scal, lam, dp, status);
        DPV_CHECK_LAUNCH();
    } else if (backend == 1) {
        // ba.solve_dense (ba.py:451-472): S scattered into a dense matrix in
        // natural pose order, every-tile right-looking Cholesky (cholesky.cu)
        DPV_TRY(ensure_dense_full(p, N, st));
        DPV_TRY(dense_path(p, lam, N, *p->dplan, p->ident_pos, dp, status, st));
    } else if (!p->spd_failed) {
        // banded + border sparse factorisation (spd.cu)
        if (!p->spd && p->plan_thread.joinable()) {
            p->plan_thread.join();           // built beside the first edge pass
            p->spd = p->spd_pending;
            p->spd_pending = nullptr;
            if (p->plan_status != DPV_OK || !p->spd) {
                p->spd = nullptr;
                p->spd_failed = 1;
                return solve(p, lam, dp, dd, status, st);
            }
        }
        if (!p->spd) {
            std::vector<int32_t> ka(p->W), kb(p->W);
            DPV_CUDA(cudaMemcpyAsync(ka.data(), p->key_a, sizeof(int32_t) * p->W,
                                     cudaMemcpyDeviceToHost, st));
            DPV_CUDA(cudaMemcpyAsync(kb.data(), p->key_b, sizeof(int32_t) * p->W,
                                     cudaMemcpyDeviceToHost, st));
            DPV_CUDA(cudaStreamSynchronize(st));
            if (spd_plan_build(ka.data(), kb.data(), p->W, p->n, &p->spd, st) != DPV_OK) {
                // e.g. a border too large for one co-resident factor grid: the
                // tile-plan factorisation below handles any pattern
                clear_error();
                p->spd = nullptr;
                p->spd_failed = 1;
                return solve(p, lam, dp, dd, status, st);
            }
        }
        // S(lam) and its rhs are formed by the scatter into the solver's storage
        SpdSysInput sys;
        sys.pose = p->pose_blocks;
        sys.schur = p->schur_blocks;
        sys.rhs_pose = p->rhs_pose;
        sys.rhs_schur = p->rhs_schur;
        sys.scal = p->scal;
        sys.lam = lam;
        DPV_TRY(spd_factor_solve(p->spd, p->key_a, p->key_b, nullptr, nullptr, dp, status, st,
                                 &sys));
    } else {
        DPV_TRY(ensure_dense(p, N, st));
        DPV_TRY(dense_path(p, lam, N, *p->plan, p->perm_pos, dp, status, st));
    }
    return back_substitute(p, lam, dp, dd, st);
}

int32_t back_substitute(dpv_problem* p, double lam, const double* dp, double* dd,
                        cudaStream_t st) {
    if (p->P == 0) return DPV_OK;
    DPV_TSTART("back_substitute", st);
    if (p->P < (int64_t)sm_count() * 64)   // few rows: a warp each (cfg3: 0.19 vs 0.07 ms)
        k_back_substitute_warp<<<grid_for(p->P * 32, 256), 256, 0, st>>>(
            p->P, p->rinc_ptr, p->rinc, p->inc_var, p->inc_block, p->rhs_depth, p->depth_diag,
            p->active, lam, dp, dd);
    else
        k_back_substitute<<<grid_for(p->P, 256), 256, 0, st>>>(
            p->P, p->rinc_ptr, p->rinc, p->inc_var, p->inc_block, p->rhs_depth, p->depth_diag,
            p->active, lam, dp, dd);
    DPV_CHECK_LAUNCH();
    return DPV_OK;
}

int32_t cholesky_solve(double* a, int64_t lda, double* b, int64_t n, int32_t* status,
                       double* work, cudaStream_t st) {
    // a: augmented (n+1) x lda buffer with the rhs already in row n; x -> b
    static FactorPlan dense_plan;   // every tile (the matrix pattern is unknown)
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (dense_plan.N != n) DPV_TRY(build_factor_plan(n, nullptr, dense_plan));
    DPV_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t) * 2, st));
    return dense_factor_solve(a, lda, n, status, b, work, dense_plan, st);
}

int32_t apply_step(dpv_problem* p, const double* q, const double* t, const double* d,
                   const double* dp, const double* dd, double* q2, double* t2, double* d2,
                   cudaStream_t st) {
    DPV_TSTART("apply_step", st);
    k_apply_step<<<grid_for(p->F + p->P, 256), 256, 0, st>>>(p->F, p->first, p->last, p->P, q, t,
                                                              d, dp, dd, q2, t2, d2);
    DPV_CHECK_LAUNCH();
    return DPV_OK;
}

}  // namespace dpv
