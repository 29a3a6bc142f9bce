// Sim(3) pose-graph optimisation (posegraph.py:121-196, the adjacent backend
// of the loop closure) on the device.
//
// Nodes are camera-to-world similarities x -> s R x + t stored as 8 doubles
// [tx ty tz | qx qy qz qw | s] (the g2o field order, posegraph.py:12-14);
// constraints are (a, b, M) with residual r = log(M S_a^-1 S_b) in the Sim(3)
// tangent (rho, phi, sigma) (posegraph.py:99-104).  Per LM iteration:
//   k_pgo_linearize  one thread per constraint: compose, log, the inverse
//                    right Jacobian Jr^-1(r) = J_l(-r)^-1 with J_l(x) =
//                    phi1(ad_x) (the reference's 14x14 block expm,
//                    geometry.py:363-375, evaluated by scaling and squaring
//                    of (e^A, phi1(A))), J_b = Jr^-1 Adj(S_b^-1);
//   k_pgo_blocks     warp per 7x7 block of H: the block's JtJ contributions
//                    in constraint order (the reference accumulates the
//                    dense h in that order, posegraph.py:141-155) into the
//                    lower triangle of a dense (7(n-1))^2 matrix;
//   k_pgo_grad       one thread per gradient entry, constraint order;
//   damped dense solve on the K4c engine (cholesky_solve: FP64 DMMA tiles);
//   k_pgo_apply      candidate nodes exp(delta_i) S_i (node 0 = the gauge);
// with the LM control flow of posegraph.py:121-196 on the host and one
// scalar read-back per damping attempt.  All reductions have a fixed order
// (bit-identical reruns, test_posegraph.py:163-179).
#include <algorithm>
#include <cmath>
#include <vector>

#include "problem.cuh"

namespace dpv {
namespace {

constexpr double kSmallAngle = 1e-8;     // geometry.py:26
constexpr double kLamGrow = 10.0, kLamShrink = 0.5, kLamMax = 1e10;   // posegraph.py:40-43

struct Sim {
    double q[4];   // x y z w
    double t[3];
    double s;
};

__device__ __forceinline__ Sim load_sim(const double* p) {
    Sim a;
    a.t[0] = p[0];
    a.t[1] = p[1];
    a.t[2] = p[2];
    a.q[0] = p[3];
    a.q[1] = p[4];
    a.q[2] = p[5];
    a.q[3] = p[6];
    a.s = p[7];
    return a;
}
__device__ __forceinline__ void store_sim(double* p, const Sim& a) {
    p[0] = a.t[0];
    p[1] = a.t[1];
    p[2] = a.t[2];
    p[3] = a.q[0];
    p[4] = a.q[1];
    p[5] = a.q[2];
    p[6] = a.q[3];
    p[7] = a.s;
}

// geometry.py:174-180: renormalise only on drift
__device__ __forceinline__ void renorm(double* q) {
    const double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (fabs(n - 1.0) > 1e-12)
        for (int k = 0; k < 4; ++k) q[k] /= n;
}
// Hamilton product (geometry.py:41-53)
__device__ __forceinline__ void qmul(const double* a, const double* b, double* o) {
    o[0] = a[3] * b[0] + a[0] * b[3] + a[1] * b[2] - a[2] * b[1];
    o[1] = a[3] * b[1] - a[0] * b[2] + a[1] * b[3] + a[2] * b[0];
    o[2] = a[3] * b[2] + a[0] * b[1] - a[1] * b[0] + a[2] * b[3];
    o[3] = a[3] * b[3] - a[0] * b[0] - a[1] * b[1] - a[2] * b[2];
}
__device__ __forceinline__ void cross(const double* a, const double* b, double* o) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}
// v + w t + xyz x t, t = 2 xyz x v (geometry.py:62-67)
__device__ __forceinline__ void qrot(const double* q, const double* v, double* o) {
    double t[3], c[3];
    cross(q, v, t);
    for (int k = 0; k < 3; ++k) t[k] *= 2.0;
    cross(q, t, c);
    for (int k = 0; k < 3; ++k) o[k] = v[k] + q[3] * t[k] + c[k];
}
// Similarity.__mul__ / inverse (geometry.py:263-272)
__device__ __forceinline__ Sim compose(const Sim& a, const Sim& b) {
    Sim o;
    qmul(a.q, b.q, o.q);
    renorm(o.q);
    double r[3];
    qrot(a.q, b.t, r);
    for (int k = 0; k < 3; ++k) o.t[k] = a.s * r[k] + a.t[k];
    o.s = a.s * b.s;
    return o;
}
__device__ __forceinline__ Sim inverse(const Sim& a) {
    Sim o;
    o.q[0] = -a.q[0];
    o.q[1] = -a.q[1];
    o.q[2] = -a.q[2];
    o.q[3] = a.q[3];
    renorm(o.q);
    double r[3];
    qrot(o.q, a.t, r);
    for (int k = 0; k < 3; ++k) o.t[k] = -r[k] / a.s;
    o.s = 1.0 / a.s;
    return o;
}
// geometry.py:70-86
__device__ __forceinline__ void qmat(const double* q, double* m) {
    const double x = q[0], y = q[1], z = q[2], w = q[3];
    const double xx = x * x, yy = y * y, zz = z * z;
    const double xy = x * y, xz = x * z, yz = y * z, wx = w * x, wy = w * y, wz = w * z;
    m[0] = 1 - 2 * (yy + zz);
    m[1] = 2 * (xy - wz);
    m[2] = 2 * (xz + wy);
    m[3] = 2 * (xy + wz);
    m[4] = 1 - 2 * (xx + zz);
    m[5] = 2 * (yz - wx);
    m[6] = 2 * (xz - wy);
    m[7] = 2 * (yz + wx);
    m[8] = 1 - 2 * (xx + yy);
}
// rotation-vector log / exp of unit quaternions (geometry.py:89-117)
__device__ __forceinline__ void quat_to_rotvec(const double* q0, double* phi) {
    double q[4];
    const double sg = q0[3] < 0 ? -1.0 : 1.0;
    for (int k = 0; k < 4; ++k) q[k] = sg * q0[k];
    const double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2]);
    const double theta = 2.0 * atan2(n, q[3]);
    const double k = n < kSmallAngle ? 2.0 / q[3] : theta / n;
    for (int c = 0; c < 3; ++c) phi[c] = q[c] * k;
}
__device__ __forceinline__ void rotvec_to_quat(const double* phi, double* q) {
    const double theta = sqrt(phi[0] * phi[0] + phi[1] * phi[1] + phi[2] * phi[2]);
    const double half = 0.5 * theta;
    const double k = theta < kSmallAngle ? 0.5 - theta * theta / 48.0 : sin(half) / theta;
    for (int c = 0; c < 3; ++c) q[c] = phi[c] * k;
    q[3] = cos(half);
}

// (e^A, phi1(A) = sum A^k/(k+1)!) of a D x D matrix (row-major) by scaling
// and squaring: ||A/2^s||_1 <= 1/4, 18-term Taylor, then s times
// phi1(2B) = phi1(B) (e^B + I) / 2, e^(2B) = (e^B)^2 - the [:D, D:] block of
// expm([[A, I], [0, 0]]) the reference takes (geometry.py:151-157, 363-369)
template <int D>
__device__ void phi1(const double* A, double* P) {
    double nrm = 0.0;
    for (int j = 0; j < D; ++j) {
        double c = 0.0;
        for (int i = 0; i < D; ++i) c += fabs(A[i * D + j]);
        nrm = fmax(nrm, c);
    }
    int s = 0;
    while (nrm > 0.25 && s < 64) {
        nrm *= 0.5;
        ++s;
    }
    const double sc = ldexp(1.0, -s);
    double B[D * D], T[D * D], E[D * D], W[D * D];
    for (int x = 0; x < D * D; ++x) {
        B[x] = A[x] * sc;
        const double id = (x / D == x % D) ? 1.0 : 0.0;
        T[x] = id;
        E[x] = id;
        P[x] = id;
    }
    for (int k = 1; k <= 18; ++k) {
        // T <- T B / k
        for (int i = 0; i < D; ++i)
            for (int j = 0; j < D; ++j) {
                double v = 0.0;
                for (int m = 0; m < D; ++m) v += T[i * D + m] * B[m * D + j];
                W[i * D + j] = v / k;
            }
        for (int x = 0; x < D * D; ++x) {
            T[x] = W[x];
            E[x] += W[x];
            P[x] += W[x] / (k + 1);
        }
    }
    for (int r = 0; r < s; ++r) {
        // P <- P (E + I) / 2, E <- E E
        for (int i = 0; i < D; ++i)
            for (int j = 0; j < D; ++j) {
                double v = 0.0;
                for (int m = 0; m < D; ++m) v += P[i * D + m] * (E[m * D + j] + (m == j ? 1.0 : 0.0));
                W[i * D + j] = 0.5 * v;
            }
        for (int x = 0; x < D * D; ++x) P[x] = W[x];
        for (int i = 0; i < D; ++i)
            for (int j = 0; j < D; ++j) {
                double v = 0.0;
                for (int m = 0; m < D; ++m) v += E[i * D + m] * E[m * D + j];
                W[i * D + j] = v;
            }
        for (int x = 0; x < D * D; ++x) E[x] = W[x];
    }
}

// Gauss-Jordan with partial pivoting: X = A^-1 (A destroyed); D x D
template <int D>
__device__ void invert(double* A, double* X) {
    for (int x = 0; x < D * D; ++x) X[x] = (x / D == x % D) ? 1.0 : 0.0;
    for (int c = 0; c < D; ++c) {
        int p = c;
        for (int r = c + 1; r < D; ++r)
            if (fabs(A[r * D + c]) > fabs(A[p * D + c])) p = r;
        if (p != c)
            for (int k = 0; k < D; ++k) {
                double t = A[c * D + k];
                A[c * D + k] = A[p * D + k];
                A[p * D + k] = t;
                t = X[c * D + k];
                X[c * D + k] = X[p * D + k];
                X[p * D + k] = t;
            }
        const double inv = 1.0 / A[c * D + c];
        for (int k = 0; k < D; ++k) {
            A[c * D + k] *= inv;
            X[c * D + k] *= inv;
        }
        for (int r = 0; r < D; ++r) {
            if (r == c) continue;
            const double f = A[r * D + c];
            if (f == 0.0) continue;
            for (int k = 0; k < D; ++k) {
                A[r * D + k] -= f * A[c * D + k];
                X[r * D + k] -= f * X[c * D + k];
            }
        }
    }
}

// coupling matrix phi1(sigma I + [phi]x) (geometry.py:143-157)
__device__ __forceinline__ void coupling(const double* phi, double sigma, double* V) {
    double A[9] = {sigma, -phi[2], phi[1], phi[2], sigma, -phi[0], -phi[1], phi[0], sigma};
    phi1<3>(A, V);
}

// sim3_exp / sim3_log (geometry.py:303-321)
__device__ Sim sim3_exp(const double* v) {
    Sim o;
    rotvec_to_quat(v + 3, o.q);
    renorm(o.q);
    double V[9];
    coupling(v + 3, v[6], V);
    for (int i = 0; i < 3; ++i) o.t[i] = V[3 * i] * v[0] + V[3 * i + 1] * v[1] + V[3 * i + 2] * v[2];
    o.s = exp(v[6]);
    return o;
}
__device__ void sim3_log(const Sim& a, double* v) {
    double phi[3];
    quat_to_rotvec(a.q, phi);
    const double sigma = log(a.s);
    double V[9], Vi[9];
    coupling(phi, sigma, V);
    invert<3>(V, Vi);
    for (int i = 0; i < 3; ++i) v[i] = Vi[3 * i] * a.t[0] + Vi[3 * i + 1] * a.t[1] + Vi[3 * i + 2] * a.t[2];
    v[3] = phi[0];
    v[4] = phi[1];
    v[5] = phi[2];
    v[6] = sigma;
}

// inverse right Jacobian Jr^-1(x) = J_l(-x)^-1, J_l(y) = phi1(ad_y)
// (geometry.py:324-375)
__device__ void jr_inv(const double* x, double* Jri) {
    double ad[49];
    for (int k = 0; k < 49; ++k) ad[k] = 0.0;
    const double rho[3] = {-x[0], -x[1], -x[2]}, phi[3] = {-x[3], -x[4], -x[5]};
    const double sigma = -x[6];
    auto put_skew = [&](int r0, int c0, const double* w, double diag) {
        ad[(r0 + 0) * 7 + c0 + 0] = diag;
        ad[(r0 + 0) * 7 + c0 + 1] = -w[2];
        ad[(r0 + 0) * 7 + c0 + 2] = w[1];
        ad[(r0 + 1) * 7 + c0 + 0] = w[2];
        ad[(r0 + 1) * 7 + c0 + 1] = diag;
        ad[(r0 + 1) * 7 + c0 + 2] = -w[0];
        ad[(r0 + 2) * 7 + c0 + 0] = -w[1];
        ad[(r0 + 2) * 7 + c0 + 1] = w[0];
        ad[(r0 + 2) * 7 + c0 + 2] = diag;
    };
    put_skew(0, 0, phi, sigma);
    put_skew(0, 3, rho, 0.0);
    for (int i = 0; i < 3; ++i) ad[i * 7 + 6] = -rho[i];
    put_skew(3, 3, phi, 0.0);
    double Jl[49];
    phi1<7>(ad, Jl);
    invert<7>(Jl, Jri);
}

// Similarity.adjoint (geometry.py:289-297)
__device__ void adjoint(const Sim& a, double* ad) {
    double R[9];
    qmat(a.q, R);
    for (int k = 0; k < 49; ++k) ad[k] = 0.0;
    const double* t = a.t;
    const double S[9] = {0.0, -t[2], t[1], t[2], 0.0, -t[0], -t[1], t[0], 0.0};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            ad[i * 7 + j] = a.s * R[i * 3 + j];
            double v = 0.0;
            for (int m = 0; m < 3; ++m) v += S[i * 3 + m] * R[m * 3 + j];
            ad[i * 7 + 3 + j] = v;
            ad[(3 + i) * 7 + 3 + j] = R[i * 3 + j];
        }
    for (int i = 0; i < 3; ++i) ad[i * 7 + 6] = -t[i];
    ad[6 * 7 + 6] = 1.0;
}

// residual r = log(M S_a^-1 S_b) and J_b = Jr^-1(r) Adj(S_b^-1)
// (posegraph.py:99-104); J == nullptr: residual only
__global__ void k_pgo_linearize(int64_t C, const int32_t* __restrict__ ca,
                                const int32_t* __restrict__ cb, const double* __restrict__ cm,
                                const double* __restrict__ nodes, double* __restrict__ r,
                                double* __restrict__ J, double* __restrict__ rr,
                                double* __restrict__ rn) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
         c += (int64_t)gridDim.x * blockDim.x) {
        const Sim m = load_sim(cm + 8 * c);
        const Sim sa = load_sim(nodes + 8 * (int64_t)ca[c]);
        const Sim sb = load_sim(nodes + 8 * (int64_t)cb[c]);
        const Sim x = compose(compose(m, inverse(sa)), sb);
        double v[7];
        sim3_log(x, v);
        double s2 = 0.0;
        for (int k = 0; k < 7; ++k) {
            r[7 * c + k] = v[k];
            s2 += v[k] * v[k];
        }
        rr[c] = s2;
        if (rn) rn[c] = sqrt(s2);
        if (J) {
            double Ji[49], Ad[49];
            jr_inv(v, Ji);
            adjoint(inverse(sb), Ad);
            for (int i = 0; i < 7; ++i)
                for (int j = 0; j < 7; ++j) {
                    double a = 0.0;
                    for (int m2 = 0; m2 < 7; ++m2) a += Ji[i * 7 + m2] * Ad[m2 * 7 + j];
                    J[49 * c + i * 7 + j] = a;
                }
        }
    }
}

// H block (p, q), p >= q, lower storage: sum over the block's contributions
// (constraint code c * 2 + negative) of +- J_c^T J_c, in constraint order.
// One warp per block, lane = entry (i, j) of the 7x7 block (49 -> 2 passes).
__global__ void k_pgo_blocks(int64_t nb, const int2* __restrict__ keys,
                             const int32_t* __restrict__ ptr, const int32_t* __restrict__ con,
                             const double* __restrict__ J, double* __restrict__ H, int64_t ld) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = warp; b < nb; b += nw) {
        const int2 k = keys[b];
        for (int e = lane; e < 49; e += 32) {
            const int i = e / 7, j = e % 7;
            double v = 0.0;
            for (int32_t x = ptr[b]; x < ptr[b + 1]; ++x) {
                const int32_t code = con[x];
                const double* Jc = J + 49 * (int64_t)(code >> 1);
                double d = 0.0;
                for (int m = 0; m < 7; ++m) d += Jc[m * 7 + i] * Jc[m * 7 + j];
                v += (code & 1) ? -d : d;
            }
            const int64_t row = 7 * (int64_t)k.x + i, col = 7 * (int64_t)k.y + j;
            if (k.x != k.y || j <= i) H[row * ld + col] = v;
        }
    }
}

// gradient entry (v, i): sum over the var's contributions of -+ J_c^T r_c
// (posegraph.py:146-152: b side -J^T r, a side +J^T r), constraint order
__global__ void k_pgo_grad(int64_t nvar, const int32_t* __restrict__ ptr,
                           const int32_t* __restrict__ con, const double* __restrict__ J,
                           const double* __restrict__ r, double* __restrict__ g) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < 7 * nvar;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = x / 7;
        const int i = (int)(x % 7);
        double acc = 0.0;
        for (int32_t e = ptr[v]; e < ptr[v + 1]; ++e) {
            const int32_t code = con[e];
            const int64_t c = code >> 1;
            double d = 0.0;
            for (int m = 0; m < 7; ++m) d += J[49 * c + m * 7 + i] * r[7 * c + m];
            acc += (code & 1) ? -d : d;
        }
        g[x] = acc;
    }
}

// out[0] = sum rr (fixed-order: strided partials, xor tree, warp order),
// out[1] = max rn, out[2] = max |g|; one 1024-thread block
__global__ void __launch_bounds__(1024) k_pgo_stats(int64_t C, const double* rr, const double* rn,
                                                    int64_t N, const double* g, double* out) {
    __shared__ double sh[3][32];
    double s = 0.0, mr = 0.0, mg = 0.0;
    for (int64_t c = threadIdx.x; c < C; c += blockDim.x) {
        s += rr[c];
        if (rn) mr = fmax(mr, rn[c]);
    }
    if (g)
        for (int64_t x = threadIdx.x; x < N; x += blockDim.x) mg = fmax(mg, fabs(g[x]));
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        mr = fmax(mr, __shfl_xor_sync(0xffffffffu, mr, o));
        mg = fmax(mg, __shfl_xor_sync(0xffffffffu, mg, o));
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        sh[0][w] = s;
        sh[1][w] = mr;
        sh[2][w] = mg;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0, c2 = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
            a += sh[0][k];
            b = fmax(b, sh[1][k]);
            c2 = fmax(c2, sh[2][k]);
        }
        out[0] = a;
        out[1] = b;
        out[2] = c2;
    }
}

// augmented damped system for cholesky_solve: rows 0..N-1 lower of
// H with diag * (1 + lam) + 1e-300 (posegraph.py:160-163), row N = g
__global__ void k_pgo_damp(int64_t N, const double* __restrict__ H, int64_t ld,
                           const double* __restrict__ g, double lam, double* __restrict__ aug,
                           int64_t lda) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < (N + 1) * N;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = x / N, j = x % N;
        if (i == N) {
            aug[N * lda + j] = g[j];
        } else if (j < i) {
            aug[i * lda + j] = H[i * ld + j];
        } else if (j == i) {
            aug[i * lda + j] = H[i * ld + j] * (1.0 + lam) + 1e-300;
        }
    }
}

// candidate nodes: exp(delta_i) S_i for i >= 1, node 0 unchanged
// (posegraph.py:171-173)
__global__ void k_pgo_apply(int64_t n, const double* __restrict__ nodes,
                            const double* __restrict__ delta, double* __restrict__ cand) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i == 0) {
            for (int k = 0; k < 8; ++k) cand[k] = nodes[k];
            continue;
        }
        double v[7];
        for (int k = 0; k < 7; ++k) v[k] = delta[7 * (i - 1) + k];
        store_sim(cand + 8 * i, compose(sim3_exp(v), load_sim(nodes + 8 * i)));
    }
}

__global__ void k_sim3_exp(int64_t n, const double* v, double* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        store_sim(out + 8 * i, sim3_exp(v + 7 * i));
}
__global__ void k_sim3_log(int64_t n, const double* s, double* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        sim3_log(load_sim(s + 8 * i), out + 7 * i);
}

struct DevBuf {
    std::vector<void*> ptrs;
    cudaStream_t st;
    explicit DevBuf(cudaStream_t s) : st(s) {}
    template <typename T>
    int32_t get(T** p, int64_t count) {
        void* q = nullptr;
        DPV_CUDA(cudaMallocAsync(&q, sizeof(T) * (size_t)std::max<int64_t>(count, 1), st));
        ptrs.push_back(q);
        *p = reinterpret_cast<T*>(q);
        return DPV_OK;
    }
    ~DevBuf() {
        for (void* q : ptrs) cudaFreeAsync(q, st);
    }
};

}  // namespace
}  // namespace dpv

using namespace dpv;

extern "C" {

int32_t dpv_pgo_linearize(int64_t n_nodes, const double* nodes, int64_t n_cons, const int32_t* ca,
                          const int32_t* cb, const double* cm, double* r, double* J,
                          double* objective, void* stream) {
    DPV_ABI_TRY
    clear_error();
    DPV_ARG(n_nodes >= 1 && n_cons >= 0 && nodes && (n_cons == 0 || (ca && cb && cm && r)),
            "bad pgo_linearize args");
    cudaStream_t st = as_stream(stream);
    DevBuf buf(st);
    double *rr = nullptr, *stats = nullptr;
    DPV_TRY(buf.get(&rr, n_cons));
    DPV_TRY(buf.get(&stats, 4));
    if (n_cons > 0) {
        DPV_TSTART("pgo_linearize", st);
        k_pgo_linearize<<<grid_for(n_cons, 128), 128, 0, st>>>(n_cons, ca, cb, cm, nodes, r, J, rr,
                                                               nullptr);
        DPV_CHECK_LAUNCH();
    }
    if (objective) {
        k_pgo_stats<<<1, 1024, 0, st>>>(n_cons, rr, nullptr, 0, nullptr, stats);
        DPV_CHECK_LAUNCH();
        DPV_CUDA(cudaMemcpyAsync(objective, stats, sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    DPV_CUDA(cudaStreamSynchronize(st));   // rr is freed with buf
    return DPV_OK;
    DPV_ABI_CATCH
}

int32_t dpv_sim3_exp(int64_t n, const double* tangents, double* sims, void* stream) {
    DPV_ABI_TRY
    clear_error();
    DPV_ARG(n >= 0 && (n == 0 || (tangents && sims)), "bad sim3_exp args");
    if (n == 0) return DPV_OK;
    k_sim3_exp<<<grid_for(n, 128), 128, 0, as_stream(stream)>>>(n, tangents, sims);
    DPV_CHECK_LAUNCH();
    return DPV_OK;
    DPV_ABI_CATCH
}

int32_t dpv_sim3_log(int64_t n, const double* sims, double* tangents, void* stream) {
    DPV_ABI_TRY
    clear_error();
    DPV_ARG(n >= 0 && (n == 0 || (tangents && sims)), "bad sim3_log args");
    if (n == 0) return DPV_OK;
    k_sim3_log<<<grid_for(n, 128), 128, 0, as_stream(stream)>>>(n, sims, tangents);
    DPV_CHECK_LAUNCH();
    return DPV_OK;
    DPV_ABI_CATCH
}

int32_t dpv_pgo_optimize(int64_t n_nodes, double* nodes, int64_t n_cons, const int32_t* ca_h,
                         const int32_t* cb_h, const int32_t* ca, const int32_t* cb,
                         const double* cm, int32_t max_iterations, double tolerance,
                         double damping, dpv_pgo_report* rep, void* stream) {
    DPV_ABI_TRY
    clear_error();
    DPV_ARG(n_nodes >= 1 && n_cons >= 0 && nodes && rep && max_iterations >= 0 &&
                (n_cons == 0 || (ca_h && cb_h && ca && cb && cm)),
            "bad pgo_optimize args");
    cudaStream_t st = as_stream(stream);
    const int64_t n = n_nodes, nv = n - 1, N = 7 * nv, C = n_cons;
    // ---- host: block pattern of H and per-var contribution lists, in
    // constraint order (posegraph.py:141-155); var(i) = i - 1, node 0 fixed
    std::vector<std::vector<int32_t>> var_con(nv);
    std::vector<std::pair<int64_t, std::vector<int32_t>>> blocks;   // key p*nv+q (p >= q)
    std::vector<int64_t> key_of;
    {
        std::vector<std::pair<int64_t, int32_t>> items;   // (key, code), stable by constraint
        for (int64_t c = 0; c < C; ++c) {
            const int64_t a = ca_h[c], b = cb_h[c];
            DPV_ARG(0 <= a && a < n && 0 <= b && b < n && a != b, "constraint references invalid nodes");
            const int64_t va = a - 1, vb = b - 1;
            if (vb >= 0) {
                items.push_back({vb * nv + vb, (int32_t)(2 * c)});
                var_con[vb].push_back((int32_t)(2 * c + 1));   // -J^T r
            }
            if (va >= 0) {
                items.push_back({va * nv + va, (int32_t)(2 * c)});
                var_con[va].push_back((int32_t)(2 * c));       // +J^T r
            }
            if (va >= 0 && vb >= 0) {
                const int64_t p = std::max(va, vb), q = std::min(va, vb);
                items.push_back({p * nv + q, (int32_t)(2 * c + 1)});
            }
        }
        std::stable_sort(items.begin(), items.end(),
                         [](const auto& x, const auto& y) { return x.first < y.first; });
        for (const auto& it : items) {
            if (blocks.empty() || blocks.back().first != it.first) blocks.push_back({it.first, {}});
            blocks.back().second.push_back(it.second);
        }
    }
    std::vector<int2> h_keys;
    std::vector<int32_t> h_bptr{0}, h_bcon, h_vptr{0}, h_vcon;
    for (const auto& b : blocks) {
        h_keys.push_back(make_int2((int)(b.first / std::max<int64_t>(nv, 1)),
                                   (int)(b.first % std::max<int64_t>(nv, 1))));
        h_bcon.insert(h_bcon.end(), b.second.begin(), b.second.end());
        h_bptr.push_back((int32_t)h_bcon.size());
    }
    for (int64_t v = 0; v < nv; ++v) {
        h_vcon.insert(h_vcon.end(), var_con[v].begin(), var_con[v].end());
        h_vptr.push_back((int32_t)h_vcon.size());
    }
    const int64_t nb = (int64_t)h_keys.size();
    const int64_t ld = N > 0 ? ((N + 7) / 8) * 8 : 8;
    const int64_t lda = ((N + 1 + 7) / 8) * 8;
    DevBuf buf(st);
    int2* d_keys;
    int32_t *d_bptr, *d_bcon, *d_vptr, *d_vcon, *d_status;
    double *d_r, *d_J, *d_rr, *d_rn, *d_H, *d_g, *d_aug, *d_work, *d_x, *d_cand, *d_stats, *d_cstats;
    DPV_TRY(buf.get(&d_keys, nb));
    DPV_TRY(buf.get(&d_bptr, nb + 1));
    DPV_TRY(buf.get(&d_bcon, (int64_t)h_bcon.size()));
    DPV_TRY(buf.get(&d_vptr, nv + 1));
    DPV_TRY(buf.get(&d_vcon, (int64_t)h_vcon.size()));
    DPV_TRY(buf.get(&d_status, 4));
    DPV_TRY(buf.get(&d_r, 7 * C));
    DPV_TRY(buf.get(&d_J, 49 * C));
    DPV_TRY(buf.get(&d_rr, C));
    DPV_TRY(buf.get(&d_rn, C));
    DPV_TRY(buf.get(&d_H, N * ld));
    DPV_TRY(buf.get(&d_g, N));
    DPV_TRY(buf.get(&d_aug, (N + 1) * lda));
    DPV_TRY(buf.get(&d_work, N > 0 ? cholesky_work_doubles(N) : 1));
    DPV_TRY(buf.get(&d_x, N));
    DPV_TRY(buf.get(&d_cand, 8 * n));
    DPV_TRY(buf.get(&d_stats, 4));
    DPV_TRY(buf.get(&d_cstats, 4));
    auto h2d = [&](void* d, const void* h, size_t bytes) -> int32_t {
        if (bytes) DPV_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st));
        return DPV_OK;
    };
    DPV_TRY(h2d(d_keys, h_keys.data(), sizeof(int2) * nb));
    DPV_TRY(h2d(d_bptr, h_bptr.data(), sizeof(int32_t) * h_bptr.size()));
    DPV_TRY(h2d(d_bcon, h_bcon.data(), sizeof(int32_t) * h_bcon.size()));
    DPV_TRY(h2d(d_vptr, h_vptr.data(), sizeof(int32_t) * h_vptr.size()));
    DPV_TRY(h2d(d_vcon, h_vcon.data(), sizeof(int32_t) * h_vcon.size()));
    if (N > 0) DPV_CUDA(cudaMemsetAsync(d_H, 0, sizeof(double) * N * ld, st));

    double host[4];
    auto read = [&](const double* d, int k) -> int32_t {
        DPV_CUDA(cudaMemcpyAsync(host, d, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
        DPV_CUDA(cudaStreamSynchronize(st));
        return DPV_OK;
    };
    // objective at `x` -> dev out[0]
    auto objective_at = [&](const double* x, double* out) -> int32_t {
        if (C > 0) {
            DPV_TSTART("pgo_objective", st);
            k_pgo_linearize<<<grid_for(C, 128), 128, 0, st>>>(C, ca, cb, cm, x, d_r, nullptr, d_rr,
                                                               nullptr);
            DPV_CHECK_LAUNCH();
        }
        k_pgo_stats<<<1, 1024, 0, st>>>(C, d_rr, nullptr, 0, nullptr, out);
        DPV_CHECK_LAUNCH();
        return DPV_OK;
    };
    DPV_TRY(objective_at(nodes, d_stats));
    DPV_TRY(read(d_stats, 1));
    double obj = host[0];
    rep->iterations = 0;
    rep->converged = 0;
    rep->initial_objective = obj;
    rep->final_objective = obj;
    rep->max_residual_norm = 0.0;
    double lam = damping;
    for (int it = 0; it < max_iterations; ++it) {
        // linearise at the current nodes
        if (C > 0) {
            DPV_TSTART("pgo_linearize", st);
            k_pgo_linearize<<<grid_for(C, 128), 128, 0, st>>>(C, ca, cb, cm, nodes, d_r, d_J, d_rr,
                                                               d_rn);
            DPV_CHECK_LAUNCH();
        }
        if (nb > 0) {
            DPV_TSTART("pgo_blocks", st);
            k_pgo_blocks<<<grid_for(nb * 32, 128), 128, 0, st>>>(nb, d_keys, d_bptr, d_bcon, d_J,
                                                                  d_H, ld);
            DPV_CHECK_LAUNCH();
        }
        if (N > 0) {
            k_pgo_grad<<<grid_for(N, 128), 128, 0, st>>>(nv, d_vptr, d_vcon, d_J, d_r, d_g);
            DPV_CHECK_LAUNCH();
        }
        k_pgo_stats<<<1, 1024, 0, st>>>(C, d_rr, d_rn, N, d_g, d_stats);
        DPV_CHECK_LAUNCH();
        DPV_TRY(read(d_stats, 3));
        rep->max_residual_norm = host[1];
        const double grad_norm = host[2];
        bool accepted = false;
        while (lam <= kLamMax) {
            int32_t singular = 0;
            if (N > 0) {
                DPV_CUDA(cudaMemsetAsync(d_aug, 0, sizeof(double) * (N + 1) * lda, st));
                k_pgo_damp<<<grid_for((N + 1) * N, 256), 256, 0, st>>>(N, d_H, ld, d_g, lam, d_aug,
                                                                       lda);
                DPV_CHECK_LAUNCH();
                DPV_TRY(cholesky_solve(d_aug, lda, d_x, N, d_status, d_work, st));
                int32_t hs = 0;
                DPV_CUDA(cudaMemcpyAsync(&hs, d_status, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
                DPV_CUDA(cudaStreamSynchronize(st));
                singular = hs;
            }
            if (singular) {
                // np.linalg.solve failure (posegraph.py:164-168)
                lam *= kLamGrow;
                if (lam > kLamMax) {
                    set_error("pose graph normal equations stayed singular");
                    return DPV_SINGULAR;
                }
                continue;
            }
            k_pgo_apply<<<grid_for(n, 128), 128, 0, st>>>(n, nodes, d_x, d_cand);
            DPV_CHECK_LAUNCH();
            DPV_TRY(objective_at(d_cand, d_cstats));
            DPV_TRY(read(d_cstats, 1));
            const double cand = host[0];
            if (cand <= obj * (1 + 1e-12) + 1e-300) {
                DPV_CUDA(cudaMemcpyAsync(nodes, d_cand, sizeof(double) * 8 * n,
                                         cudaMemcpyDeviceToDevice, st));
                obj = std::min(cand, obj);
                lam = std::max(lam * kLamShrink, 1e-12);
                accepted = true;
                break;
            }
            lam *= kLamGrow;
        }
        if (!accepted) break;
        rep->iterations += 1;
        rep->final_objective = obj;
        if (grad_norm < tolerance) {
            rep->converged = 1;
            break;
        }
    }
    DPV_CUDA(cudaStreamSynchronize(st));
    rep->final_objective = obj;
    rep->final_damping = lam;
    if (obj < 1e-24) rep->converged = 1;
    return DPV_OK;
    DPV_ABI_CATCH
}

}  // extern "C"
