// K2 + K3 + K4a: fused per-edge reprojection / Jacobians / whitened Gram,
// deterministic segmented reductions into the block-sparse normal equations,
// and the Schur elimination of the inverse depths.
//
// Restates ba.residuals/objective (ba.py:219-253) and ba.assemble
// (ba.py:328-440) with geometry.reproject_grid (geometry.py:478-529) inlined.
// Every reduction runs over a fixed, index-sorted list (no float atomics), so
// results are bit-identical run to run.
#include <cstdlib>

#include "problem.cuh"

namespace dpv {
namespace {

struct Frame {
    double R[9];
    double t[3];
};

__device__ __forceinline__ void load_frame(const double* Rall, const double* tall, int f,
                                           Frame& fr) {
#pragma unroll
    for (int k = 0; k < 9; ++k) fr.R[k] = __ldg(Rall + 9 * f + k);
#pragma unroll
    for (int k = 0; k < 3; ++k) fr.t[k] = __ldg(tall + 3 * f + k);
}

// One patch cell: world point, target-camera point, validity and pixel.
struct Cell {
    double xw[3];
    double xt[3];
    double zs;
    double iz;      // 1 / zs
    bool valid;
    double u, v;
};

__device__ __forceinline__ void reproject_cell(double rx, double ry, double inv_d_recip,
                                               const Frame& fi, const Frame& fj,
                                               const double* intr, Cell& c) {
    // x_cam = ray / d  (ray z = 1)
    const double xc0 = rx * inv_d_recip, xc1 = ry * inv_d_recip, xc2 = inv_d_recip;
    // x_w = R_i x_c + t_i
#pragma unroll
    for (int r = 0; r < 3; ++r)
        c.xw[r] = fi.R[3 * r] * xc0 + fi.R[3 * r + 1] * xc1 + fi.R[3 * r + 2] * xc2 + fi.t[r];
    const double e0 = c.xw[0] - fj.t[0], e1 = c.xw[1] - fj.t[1], e2 = c.xw[2] - fj.t[2];
    // x_t = R_j^T (x_w - t_j)
#pragma unroll
    for (int k = 0; k < 3; ++k) c.xt[k] = fj.R[k] * e0 + fj.R[3 + k] * e1 + fj.R[6 + k] * e2;
    c.valid = c.xt[2] > kDepthEps;
    c.zs = c.valid ? c.xt[2] : 1.0;
    // one reciprocal per cell instead of two divisions (results agree with
    // the reference's fx * x / z to a few ulp; parity is tolerance-based)
    c.iz = __drcp_rn(c.zs);
    c.u = intr[0] * c.xt[0] * c.iz + intr[2];
    c.v = intr[1] * c.xt[1] * c.iz + intr[3];
}

// same, frames read from shared memory (per-warp uniform, broadcast loads)
struct FrameP {
    const double* R;
    const double* t;
};

__device__ __forceinline__ void reproject_cell(double rx, double ry, double inv_d_recip,
                                               const FrameP& fi, const FrameP& fj,
                                               const double* intr, Cell& c) {
    const double xc0 = rx * inv_d_recip, xc1 = ry * inv_d_recip, xc2 = inv_d_recip;
#pragma unroll
    for (int r = 0; r < 3; ++r)
        c.xw[r] = fi.R[3 * r] * xc0 + fi.R[3 * r + 1] * xc1 + fi.R[3 * r + 2] * xc2 + fi.t[r];
    const double e0 = c.xw[0] - fj.t[0], e1 = c.xw[1] - fj.t[1], e2 = c.xw[2] - fj.t[2];
#pragma unroll
    for (int k = 0; k < 3; ++k) c.xt[k] = fj.R[k] * e0 + fj.R[3 + k] * e1 + fj.R[6 + k] * e2;
    c.valid = c.xt[2] > kDepthEps;
    c.zs = c.valid ? c.xt[2] : 1.0;
    c.iz = __drcp_rn(c.zs);
    c.u = intr[0] * c.xt[0] * c.iz + intr[2];
    c.v = intr[1] * c.xt[1] * c.iz + intr[3];
}

// ---------------------------------------------------------------------------
// K2 objective: sum_e sum_cells w_comp * valid * r^2 (ba.py:248-253)

__global__ void __launch_bounds__(256) k_objective(
    int64_t E, int m, int64_t P, const int32_t* __restrict__ a_src,
    const int32_t* __restrict__ a_dst, const int32_t* __restrict__ a_row,
    const double* __restrict__ a_tgt, const double* __restrict__ a_w,
    const double* __restrict__ r_ray, const double* __restrict__ Rall,
    const double* __restrict__ tall, const double* __restrict__ d, double fx, double fy,
    double cx, double cy, double* __restrict__ part) {
    const double intr[4] = {fx, fy, cx, cy};
    double acc = 0.0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        Frame fi, fj;
        load_frame(Rall, tall, a_src[e], fi);
        load_frame(Rall, tall, a_dst[e], fj);
        const int32_t row = a_row[e];
        const double id = __drcp_rn(__ldg(d + row));
        const double w0 = a_w[e], w1 = a_w[E + e];
        double s = 0.0;
        for (int c = 0; c < m; ++c) {
            Cell cl;
            reproject_cell(__ldg(r_ray + (int64_t)(2 * c) * P + row),
                           __ldg(r_ray + (int64_t)(2 * c + 1) * P + row), id, fi, fj, intr, cl);
            if (cl.valid) {
                const double r0 = cl.u - a_tgt[(int64_t)(2 * c) * E + e];
                const double r1 = cl.v - a_tgt[(int64_t)(2 * c + 1) * E + e];
                s += w0 * r0 * r0 + w1 * r1 * r1;
            }
        }
        acc += s;
    }
    // fixed-order block reduction
    __shared__ double sh[8];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
        part[blockIdx.x] = t;
    }
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
    asm volatile("prefetch.global.L1 [%0];\n" ::"l"(p));
}

// same sum, one warp per (src, dst) segment: the two frames are loaded once
// per segment into shared memory, lanes stride over the segment's edges.
template <int M, int U, int MINB, bool PF>
__global__ void __launch_bounds__(256, MINB) k_objective_seg(
    int64_t S, int64_t E, int64_t P, const int32_t* __restrict__ seg_ptr,
    const int32_t* __restrict__ seg_src, const int32_t* __restrict__ seg_dst,
    const int32_t* __restrict__ a_row, const double* __restrict__ a_tgt,
    const double* __restrict__ a_w, const double* __restrict__ r_ray,
    const double* __restrict__ Rall, const double* __restrict__ tall,
    const double* __restrict__ d, double fx, double fy, double cx, double cy,
    double* __restrict__ part) {
    const double intr[4] = {fx, fy, cx, cy};
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    __shared__ double sfr[8][24];
    double* fr = sfr[threadIdx.x >> 5];
    const FrameP fi{fr, fr + 9}, fj{fr + 12, fr + 21};
    double acc = 0.0;
    for (int64_t s = warp; s < S; s += nwarps) {
        const int32_t e0 = seg_ptr[s], e1 = seg_ptr[s + 1];
        __syncwarp();
        if (lane < 12) {
            const int32_t f = seg_src[s];
            fr[lane] = lane < 9 ? __ldg(Rall + 9 * f + lane) : __ldg(tall + 3 * f + lane - 9);
        } else if (lane < 24) {
            const int32_t f = seg_dst[s];
            fr[lane] = lane < 21 ? __ldg(Rall + 9 * f + lane - 12) : __ldg(tall + 3 * f + lane - 21);
        }
        __syncwarp();
        int32_t rn1 = (PF && e0 + lane + 32 < e1) ? a_row[e0 + lane + 32] : 0;
        for (int32_t e = e0 + lane; e < e1; e += 32) {
            if (PF) {          // next edge's inputs into L1 (see k_assemble_edges)
                const int32_t en = e + 32;
                int32_t rn2 = 0;
                if (en < e1) {
#pragma unroll
                    for (int c = 0; c < 2 * M; ++c) {
                        prefetch_l1(a_tgt + (int64_t)c * E + en);
                        prefetch_l1(r_ray + (int64_t)c * P + rn1);
                    }
                    prefetch_l1(a_w + en);
                    prefetch_l1(a_w + E + en);
                    prefetch_l1(d + rn1);
                    if (en + 32 < e1) rn2 = a_row[en + 32];
                }
                rn1 = rn2;
            }
            const int32_t row = a_row[e];
            const double id = __drcp_rn(__ldg(d + row));
            const double w0 = a_w[e], w1 = a_w[E + e];
            double sum = 0.0;
#pragma unroll U
            for (int c = 0; c < M; ++c) {
                Cell cl;
                reproject_cell(__ldg(r_ray + (int64_t)(2 * c) * P + row),
                               __ldg(r_ray + (int64_t)(2 * c + 1) * P + row), id, fi, fj, intr,
                               cl);
                const double r0 = cl.u - a_tgt[(int64_t)(2 * c) * E + e];
                const double r1 = cl.v - a_tgt[(int64_t)(2 * c + 1) * E + e];
                sum += cl.valid ? w0 * r0 * r0 + w1 * r1 * r1 : 0.0;
            }
            acc += sum;
        }
    }
    __shared__ double sh[8];
    acc = warp_sum(acc);
    if (lane == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
        part[blockIdx.x] = t;
    }
}

// block b sums the contiguous slice [b*n/B, (b+1)*n/B) in a fixed order
__global__ void k_slice_sums(int64_t n, const double* v, double* part) {
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t lo = (int64_t)blockIdx.x * per, hi = min(n, lo + per);
    double acc = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) acc += v[i];
    __shared__ double sh[32];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
        part[blockIdx.x] = t;
    }
}

__global__ void k_sum_parts(int n, const double* part, double* out) {
    __shared__ double sh[32];
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc += part[i];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
        out[0] = t;
    }
}

// residual export in problem-edge order (ba.py:219-245)
__global__ void k_residuals(int64_t E, int m, int64_t P, const int32_t* a_src,
                            const int32_t* a_dst, const int32_t* a_row, const int32_t* a_pidx,
                            const double* a_tgt, const double* r_ray, const double* Rall,
                            const double* tall, const double* d, double fx, double fy, double cx,
                            double cy, double* res, uint8_t* valid) {
    const double intr[4] = {fx, fy, cx, cy};
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        Frame fi, fj;
        load_frame(Rall, tall, a_src[e], fi);
        load_frame(Rall, tall, a_dst[e], fj);
        const int32_t row = a_row[e];
        const double id = 1.0 / d[row];
        const int64_t p = a_pidx[e];
        for (int c = 0; c < m; ++c) {
            Cell cl;
            reproject_cell(r_ray[(int64_t)(2 * c) * P + row], r_ray[(int64_t)(2 * c + 1) * P + row],
                           id, fi, fj, intr, cl);
            res[(p * m + c) * 2] = cl.u - a_tgt[(int64_t)(2 * c) * E + e];
            res[(p * m + c) * 2 + 1] = cl.v - a_tgt[(int64_t)(2 * c + 1) * E + e];
            valid[p * m + c] = cl.valid ? 1 : 0;
        }
    }
}

// reprojected pixels * scale in problem-edge order (coordinates for K1)
__global__ void k_coords(int64_t E, int m, int64_t P, const int32_t* a_src,
                         const int32_t* a_dst, const int32_t* a_row, const int32_t* a_pidx,
                         const double* r_ray, const double* Rall, const double* tall,
                         const double* d, double fx, double fy, double cx, double cy,
                         double scale, double* coords) {
    const double intr[4] = {fx, fy, cx, cy};
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        Frame fi, fj;
        load_frame(Rall, tall, a_src[e], fi);
        load_frame(Rall, tall, a_dst[e], fj);
        const int32_t row = a_row[e];
        const double id = __drcp_rn(__ldg(d + row));
        const int64_t p = a_pidx[e];
        for (int c = 0; c < m; ++c) {
            Cell cl;
            reproject_cell(__ldg(r_ray + (int64_t)(2 * c) * P + row),
                           __ldg(r_ray + (int64_t)(2 * c + 1) * P + row), id, fi, fj, intr, cl);
            coords[(p * m + c) * 2] = cl.u * scale;
            coords[(p * m + c) * 2 + 1] = cl.v * scale;
        }
    }
}

// K2 pixels of a selection of problem edges (the correlation edges), output
// in selection order
__global__ void k_coords_sel(int64_t n_sel, const int64_t* sel, const int32_t* p_pos, int m,
                             int64_t P, const int32_t* a_src, const int32_t* a_dst,
                             const int32_t* a_row, const double* r_ray, const double* Rall,
                             const double* tall, const double* d, double fx, double fy,
                             double cx, double cy, double scale, double* coords) {
    const double intr[4] = {fx, fy, cx, cy};
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n_sel * m;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = x / m;
        const int c = (int)(x % m);
        const int64_t e = p_pos[sel[i]];
        Frame fi, fj;
        load_frame(Rall, tall, a_src[e], fi);
        load_frame(Rall, tall, a_dst[e], fj);
        const int32_t row = a_row[e];
        const double id = __drcp_rn(__ldg(d + row));
        Cell cl;
        reproject_cell(__ldg(r_ray + (int64_t)(2 * c) * P + row),
                       __ldg(r_ray + (int64_t)(2 * c + 1) * P + row), id, fi, fj, intr, cl);
        coords[x * 2] = cl.u * scale;
        coords[x * 2 + 1] = cl.v * scale;
    }
}

// new flow targets / confidences (problem order) -> assembly-order SoA
__global__ void k_update_targets(int64_t E, int m, const int32_t* p_pos, const double* tgt,
                                 const double* conf, double* a_tgt, double* a_w) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < E;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = p_pos[p];
        for (int c = 0; c < 2 * m; ++c) a_tgt[(int64_t)c * E + e] = tgt[p * 2 * m + c];
        if (conf) {
            a_w[e] = conf[2 * p];
            a_w[E + e] = conf[2 * p + 1];
        }
    }
}

// ---------------------------------------------------------------------------
// K2+K3 fused: one warp per segment (same source/target frame, <= kSegMax
// edges), one lane per edge.  Per edge it writes e_pd (6), c_dd, g_d; per
// segment the warp-reduced sum of J^T W J (21, upper) and J^T W r (6).

__device__ __forceinline__ int utri(int a, int b) {  // a <= b < 6
    return a * 6 - (a * (a - 1)) / 2 + (b - a);
}

// Same pass in the TARGET camera's frame (default).  With B = diag(R_j, R_j)
// the world Jacobian row is J_r = B k_r, k_r = [jp_r ; y x jp_r] where jp_r is
// row r of Jproj and y = R_j^T x_w (rotation commutes with the cross
// product), so per segment Sum w J^T J = B (Sum w k k^T) B^T.  k_0 has no
// y-component (k_0[1] = 0) and k_1 no x-component (k_1[0] = 0): 15 instead of
// 21 Gram FMAs per residual row.  The point chain uses Rrel = R_j^T R_i and
// u = R_j^T (t_i - t_j) (x_t = Rrel x_c + u; J_depth = -jp_r . Rrel x_c / d,
// since t_i - x_w = -R_i x_c).  The per-edge e_pd and the per-segment sums
// are rotated back to world coordinates, so the outputs keep their meaning
// (ba.py:355-366); values agree with the world-frame pass to rounding.
template <int Z>
__device__ __forceinline__ void gram_row(const double (&k)[6], double wv, double rr, double jd,
                                         double (&acc)[28], double (&ep)[6], double& cdd,
                                         double& gd) {
    // acc: 0..20 Sum w k k^T (upper, utri order), 21..26 Sum w k r, 27 objective
    double wk[6];
#pragma unroll
    for (int a = 0; a < 6; ++a) wk[a] = (a == Z) ? 0.0 : k[a] * wv;
#pragma unroll
    for (int a = 0; a < 6; ++a) {
        if (a == Z) continue;
#pragma unroll
        for (int b = a; b < 6; ++b) {
            if (b == Z) continue;
            acc[utri(a, b)] += wk[a] * k[b];
        }
        acc[21 + a] += wk[a] * rr;
        ep[a] += wk[a] * jd;
    }
    const double wjd = jd * wv;
    cdd += wjd * jd;
    gd += wjd * rr;
    acc[27] += wv * rr * rr;
}

// The local-frame edge pass with its inputs staged through shared memory:
// per warp a double-buffered ring of 32-edge items (one lane per edge).
// While item i computes, item i+1's targets, weights, rays and depth are in
// flight as 8-byte cp.async copies (its rows were loaded one item earlier),
// so the FP64 chain no longer waits on global-load latency.  Segments are cut
// into items of <= 32 edges; the Gram sums run across a segment's items and
// are reduced / rotated to world coordinates after its last item.
constexpr int kStgVals = 39;                  // 18 targets, 18 rays, 2 weights, depth
constexpr int kStgFrames = kStgVals * 32;     // + the segment's two frames (24) when it starts
constexpr int kStgDoubles = kStgVals * 32 + 32;

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait1() {
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
}

// 1/x for a positive normal x without __drcp_rn's special-case branch: the
// library call's slow-path test splits the unrolled 9-cell loop of the edge
// pass into ~10 basic blocks the scheduler cannot interleave.  MUFU seed +
// two Newton steps (within 1 ulp of the correctly rounded reciprocal).
__device__ __forceinline__ double rcp_pos(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}

// a segment's bounds and frames, loaded one segment ahead of its first item
struct SegDesc {
    int64_t s;        // >= S: none
    int32_t e0, se1, fs, fd;
};

struct EdgeItem {
    int64_t s;        // segment (>= S: none)
    int32_t e0, e1;   // this item's edge range
    int32_t se1;      // segment end
    int32_t fs, fd;   // source / target frame (first item only)
    bool first;       // first item of its segment
};

// Warp reduce-scatter of 32 per-lane values (recursive halving: 31 shuffles
// instead of 5 per value): afterwards v[0] of lane l is the warp total of
// value l.  Fixed tree, so the sums are reproducible run to run.
template <int O>
__device__ __forceinline__ void halve(double (&v)[32], int lane) {
    const bool up = lane & O;
#pragma unroll
    for (int i = 0; i < O; ++i) {
        const double send = up ? v[i] : v[i + O];
        const double keep = up ? v[i + O] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, O);
    }
}

template <int NW, int MINB>
__global__ void __launch_bounds__(32 * NW, MINB) k_assemble_edges_stg(
    int64_t S, int64_t E, int64_t P, const int32_t* __restrict__ seg_ptr,
    const int32_t* __restrict__ seg_src, const int32_t* __restrict__ seg_dst,
    const int32_t* __restrict__ a_row, const double* __restrict__ a_tgt,
    const double* __restrict__ a_w, const double* __restrict__ r_ray,
    const double* __restrict__ Rall, const double* __restrict__ tall,
    const double* __restrict__ d, double fx, double fy, double cx, double cy,
    double* __restrict__ e_terms, double* __restrict__ seg_h, double* __restrict__ seg_g,
    double* __restrict__ seg_obj) {
    extern __shared__ double stg_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double* ring = stg_raw + (int64_t)wib * 2 * kStgDoubles;
    __shared__ double sfr[NW][82];
    double* fr = sfr[wib];
    const double* Ri = fr;
    const double* ti = fr + 9;
    const double* Rj = fr + 12;
    const double* tj = fr + 21;
    const double* Rr = fr + 24;
    const double* uu = fr + 33;
    const double* cc = fr + 36;
    double* Hs = fr + 40;
    double* Gs = fr + 76;

    // Segment descriptors are loaded a whole segment ahead and items two
    // items ahead, so no global load sits on the dependency chain of an item
    // (the per-segment seg_ptr -> a_row and seg_src -> frame chains were the
    // kernel's long-scoreboard stalls).
    auto load_seg = [&](int64_t s) {
        SegDesc g;
        g.s = s;
        if (s < S) {
            g.e0 = __ldg(seg_ptr + s);
            g.se1 = __ldg(seg_ptr + s + 1);
            g.fs = __ldg(seg_src + s);
            g.fd = __ldg(seg_dst + s);
        } else {
            g.e0 = g.se1 = g.fs = g.fd = 0;
        }
        return g;
    };
    SegDesc pend = load_seg(warp);
    auto start_item = [&]() {
        EdgeItem it;
        it.s = pend.s;
        it.e0 = pend.e0;
        it.se1 = pend.se1;
        it.e1 = min(it.e0 + 32, it.se1);
        it.fs = pend.fs;
        it.fd = pend.fd;
        it.first = true;
        if (pend.s < S) pend = load_seg(pend.s + nwarps);
        return it;
    };
    auto next_item = [&](const EdgeItem& it) {
        if (it.s < S && it.e1 < it.se1) {
            EdgeItem n = it;
            n.e0 = it.e1;
            n.e1 = min(n.e0 + 32, it.se1);
            n.first = false;
            return n;
        }
        return start_item();
    };
    auto row_of = [&](const EdgeItem& it) -> int32_t {
        const int32_t e = it.e0 + lane;
        return (it.s < S && e < it.e1) ? __ldg(a_row + e) : 0;
    };
    auto issue = [&](const EdgeItem& it, int32_t row, double* b) {
        const int32_t e = it.e0 + lane;
        if (it.s < S && e < it.e1) {
#pragma unroll
            for (int c = 0; c < 18; ++c) cp_async8(b + c * 32 + lane, a_tgt + (int64_t)c * E + e);
#pragma unroll
            for (int c = 0; c < 18; ++c)
                cp_async8(b + (18 + c) * 32 + lane, r_ray + (int64_t)c * P + row);
            cp_async8(b + 36 * 32 + lane, a_w + e);
            cp_async8(b + 37 * 32 + lane, a_w + E + e);
            cp_async8(b + 38 * 32 + lane, d + row);
        }
        if (it.s < S && it.first && lane < 24) {
            const double* src = lane < 9    ? Rall + 9 * it.fs + lane
                                : lane < 12 ? tall + 3 * it.fs + lane - 9
                                : lane < 21 ? Rall + 9 * it.fd + lane - 12
                                            : tall + 3 * it.fd + lane - 21;
            cp_async8(b + kStgFrames + lane, src);
        }
        cp_async_commit();
    };

    EdgeItem cur = start_item();
    EdgeItem nx = next_item(cur);
    int32_t row_cur = row_of(cur);
    int32_t row_nx = row_of(nx);
    issue(cur, row_cur, ring);
    double acc[28];                   // per-lane Gram sums of the segment (gram_row)
    int buf = 0;
    while (cur.s < S) {
        // stage the next item, load the rows of the one after
        const EdgeItem nx2 = next_item(nx);
        const int32_t row_nx2 = row_of(nx2);
        issue(nx, row_nx, ring + (buf ^ 1) * kStgDoubles);
        cp_async_wait1();
        __syncwarp();
        const double* b = ring + buf * kStgDoubles;
        if (cur.first) {
            if (lane < 24) fr[lane] = b[kStgFrames + lane];
            __syncwarp();
            if (lane < 9) {
                const int a = lane / 3, bb = lane % 3;
                fr[24 + lane] = Rj[a] * Ri[bb] + Rj[3 + a] * Ri[3 + bb] + Rj[6 + a] * Ri[6 + bb];
            } else if (lane < 12) {
                const int a = lane - 9;
                fr[24 + lane] = Rj[a] * (ti[0] - tj[0]) + Rj[3 + a] * (ti[1] - tj[1]) +
                                Rj[6 + a] * (ti[2] - tj[2]);
            } else if (lane < 15) {
                const int a = lane - 12;
                fr[24 + lane] = Rj[a] * tj[0] + Rj[3 + a] * tj[1] + Rj[6 + a] * tj[2];
            }
#pragma unroll
            for (int k = 0; k < 28; ++k) acc[k] = 0.0;
            __syncwarp();
        }
        const int32_t e = cur.e0 + lane;
        if (e < cur.e1) {
            const double id = rcp_pos(b[38 * 32 + lane]);
            const double w0 = b[36 * 32 + lane], w1 = b[37 * 32 + lane];
            double ep[6] = {0, 0, 0, 0, 0, 0};
            double cdd = 0.0, gd = 0.0;
#pragma unroll
            for (int c = 0; c < 9; ++c) {
                const double xc0 = b[(18 + 2 * c) * 32 + lane] * id;
                const double xc1 = b[(19 + 2 * c) * 32 + lane] * id;
                double xr[3], xt[3];
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    xr[a] = Rr[3 * a] * xc0 + Rr[3 * a + 1] * xc1 + Rr[3 * a + 2] * id;
                    xt[a] = xr[a] + uu[a];
                }
                const bool valid = xt[2] > kDepthEps;
                const double iz = rcp_pos(valid ? xt[2] : 1.0);
                const double t0 = xt[0] * iz, t1 = xt[1] * iz;
                const double p0 = fx * iz, p1 = fy * iz;
                const double q0 = -p0 * t0, q1 = -p1 * t1;
                const double y0 = xt[0] + cc[0], y1 = xt[1] + cc[1], y2 = xt[2] + cc[2];
                const double k0[6] = {p0, 0.0, q0, y1 * q0, y2 * p0 - y0 * q0, -y1 * p0};
                const double k1[6] = {0.0, p1, q1, y1 * q1 - y2 * p1, -y0 * q1, y0 * p1};
                const double jd0 = -(p0 * xr[0] + q0 * xr[2]) * id;
                const double jd1 = -(p1 * xr[1] + q1 * xr[2]) * id;
                const double r0 = (fx * t0 + cx) - b[(2 * c) * 32 + lane];
                const double r1 = (fy * t1 + cy) - b[(2 * c + 1) * 32 + lane];
                gram_row<1>(k0, valid ? w0 : 0.0, r0, jd0, acc, ep, cdd, gd);
                gram_row<0>(k1, valid ? w1 : 0.0, r1, jd1, acc, ep, cdd, gd);
            }
            double ew[6];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int a = 0; a < 3; ++a)
                    ew[3 * h + a] = Rj[3 * a] * ep[3 * h] + Rj[3 * a + 1] * ep[3 * h + 1] +
                                    Rj[3 * a + 2] * ep[3 * h + 2];
            double2* et = reinterpret_cast<double2*>(e_terms + (int64_t)e * 6);
            et[0] = make_double2(ew[0], ew[1]);
            et[1] = make_double2(ew[2], ew[3]);
            et[2] = make_double2(ew[4], ew[5]);
            reinterpret_cast<double2*>(e_terms + 6 * E)[e] = make_double2(cdd, gd);
        }
        if (cur.e1 == cur.se1) {          // segment done: reduce, rotate, write
            const int64_t sg = cur.s;
            __syncwarp();
            double v[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) v[k] = k < 28 ? acc[k] : 0.0;
            halve<16>(v, lane);
            halve<8>(v, lane);
            halve<4>(v, lane);
            halve<2>(v, lane);
            halve<1>(v, lane);
            if (lane < 21) {
                int a = 0;
                while (a < 5 && utri(a + 1, a + 1) <= lane) ++a;
                const int bb = a + (lane - utri(a, a));
                Hs[a * 6 + bb] = v[0];
                Hs[bb * 6 + a] = v[0];
            } else if (lane < 27) {
                Gs[lane - 21] = v[0];
            } else if (lane == 27 && seg_obj) {
                seg_obj[sg] = v[0];
            }
            __syncwarp();
            if (lane < 21) {
                int a = 0;
                while (a < 5 && utri(a + 1, a + 1) <= lane) ++a;
                const int bb = a + (lane - utri(a, a));
                const int al = a % 3, ab = (a / 3) * 3, bl = bb % 3, bo = (bb / 3) * 3;
                double v = 0.0;
#pragma unroll
                for (int pp = 0; pp < 3; ++pp) {
                    const double* hr = Hs + (ab + pp) * 6 + bo;
                    const double inner = hr[0] * Rj[3 * bl] + hr[1] * Rj[3 * bl + 1] +
                                         hr[2] * Rj[3 * bl + 2];
                    v += Rj[3 * al + pp] * inner;
                }
                seg_h[sg * 21 + lane] = v;
            } else if (lane < 27) {
                const int a = lane - 21, al = a % 3, ab = (a / 3) * 3;
                seg_g[sg * 6 + a] = Rj[3 * al] * Gs[ab] + Rj[3 * al + 1] * Gs[ab + 1] +
                                    Rj[3 * al + 2] * Gs[ab + 2];
            }
        }
        __syncwarp();                     // buffer `buf` and the frames are free
        cur = nx;
        nx = nx2;
        row_nx = row_nx2;
        buf ^= 1;
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// depth side (ba.py:370-373): per-row sums over the row's edges
__global__ void k_rows(int64_t P, int64_t E, const int32_t* row_ptr, const int32_t* row_pos,
                       const double* e_terms, double* depth_diag, double* rhs_depth,
                       uint8_t* active, double* cinv0, unsigned long long* grad_bits,
                       unsigned long long* n_inactive) {
    // (c_dd, g_d) of edge e: the SoA tail of e_terms, 16 B per edge, so the
    // adjacent rows' edges of one segment share sectors
    const double2* e_cg = reinterpret_cast<const double2*>(e_terms + 6 * E);
    double gmax = 0.0;
    unsigned long long inact = 0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < P;
         r += (int64_t)gridDim.x * blockDim.x) {
        double c = 0.0, g = 0.0;
        const int32_t k1 = row_ptr[r + 1];
        int32_t k = row_ptr[r];
        for (; k + 1 < k1; k += 2) {       // two gathers in flight, same order
            const int32_t ea = __ldg(row_pos + k), eb = __ldg(row_pos + k + 1);
            const double2 ca = __ldg(e_cg + ea);
            const double2 cb = __ldg(e_cg + eb);
            c += ca.x;
            g += ca.y;
            c += cb.x;
            g += cb.y;
        }
        if (k < k1) {
            const double2 cg = __ldg(e_cg + __ldg(row_pos + k));
            c += cg.x;
            g += cg.y;
        }
        depth_diag[r] = c;
        rhs_depth[r] = -g;
        const bool act = c > kActiveEps;
        active[r] = act ? 1 : 0;
        cinv0[r] = act ? 1.0 / c : 0.0;
        if (act) gmax = fmax(gmax, fabs(g));
        else ++inact;
    }
    // one atomic per warp (max / count are order-independent)
    gmax = warp_max(gmax);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) inact += __shfl_xor_sync(0xffffffffu, inact, o);
    if ((threadIdx.x & 31) == 0) {
        if (gmax > 0.0) {
            const unsigned long long gb = (unsigned long long)__double_as_longlong(gmax);
            atomicMax(grad_bits, gb);
            atomicMax(grad_bits + 7, gb);   // depth-only part (sharded BA)
        }
        if (inact) atomicAdd(n_inactive, inact);
    }
}

// same sums, two contributions per step (both gathers in flight before the
// adds; same summation order) and 16-byte stores
__global__ void __launch_bounds__(256) k_incidences2(int64_t I, const int32_t* __restrict__ inc_ptr,
                                                     const int32_t* __restrict__ inc_con,
                                                     const int32_t* __restrict__ inc_row,
                                                     const double* __restrict__ e_terms,
                                                     const double* __restrict__ cinv0,
                                                     double* __restrict__ inc_block,
                                                     double* __restrict__ uinc, int sym) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < I;
         i += (int64_t)gridDim.x * blockDim.x) {
        double acc[6] = {0, 0, 0, 0, 0, 0};
        const int32_t k0 = inc_ptr[i], k1 = inc_ptr[i + 1];
        const double c0 = __ldg(cinv0 + inc_row[i]);
        int32_t k = k0;
        for (; k + 1 < k1; k += 2) {
            const int32_t ca = __ldg(inc_con + k), cb = __ldg(inc_con + k + 1);
            const double2* ea = reinterpret_cast<const double2*>(e_terms + (int64_t)(ca >> 1) * 6);
            const double2* eb = reinterpret_cast<const double2*>(e_terms + (int64_t)(cb >> 1) * 6);
            double2 va[3], vb[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                va[a] = __ldg(ea + a);
                vb[a] = __ldg(eb + a);
            }
            const double sa = (ca & 1) ? -1.0 : 1.0, sb = (cb & 1) ? -1.0 : 1.0;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                acc[2 * a] += sa * va[a].x;
                acc[2 * a + 1] += sa * va[a].y;
            }
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                acc[2 * a] += sb * vb[a].x;
                acc[2 * a + 1] += sb * vb[a].y;
            }
        }
        if (k < k1) {
            const int32_t ca = __ldg(inc_con + k);
            const double2* ea = reinterpret_cast<const double2*>(e_terms + (int64_t)(ca >> 1) * 6);
            const double sa = (ca & 1) ? -1.0 : 1.0;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const double2 v = __ldg(ea + a);
                acc[2 * a] += sa * v.x;
                acc[2 * a + 1] += sa * v.y;
            }
        }
        const double c = sym ? sqrt(c0) : c0;
        double2* ib = reinterpret_cast<double2*>(inc_block + i * 6);
        double2* ub = reinterpret_cast<double2*>(uinc + i * 6);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            ib[a] = make_double2(acc[2 * a], acc[2 * a + 1]);
            ub[a] = make_double2(acc[2 * a] * c, acc[2 * a + 1] * c);
        }
    }
}

// small problems (few rows): one warp per row, lanes over the row's edges,
// xor-tree reduction (fixed order)
__global__ void k_rows_warp(int64_t P, int64_t E, const int32_t* row_ptr, const int32_t* row_pos,
                            const double* e_terms, double* depth_diag, double* rhs_depth,
                            uint8_t* active, double* cinv0, unsigned long long* grad_bits,
                            unsigned long long* n_inactive) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double gmax = 0.0;
    unsigned long long inact = 0;
    for (int64_t r = warp; r < P; r += nwarps) {
        double c = 0.0, g = 0.0;
        for (int32_t k = row_ptr[r] + lane; k < row_ptr[r + 1]; k += 32) {
            const double2 cg = __ldg(reinterpret_cast<const double2*>(e_terms + 6 * E) +
                                     __ldg(row_pos + k));
            c += cg.x;
            g += cg.y;
        }
        c = warp_sum(c);
        g = warp_sum(g);
        if (lane == 0) {
            depth_diag[r] = c;
            rhs_depth[r] = -g;
            const bool act = c > kActiveEps;
            active[r] = act ? 1 : 0;
            cinv0[r] = act ? 1.0 / c : 0.0;
            if (act) gmax = fmax(gmax, fabs(g));
            else ++inact;
        }
    }
    gmax = warp_max(gmax);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) inact += __shfl_xor_sync(0xffffffffu, inact, o);
    if (lane == 0) {
        if (gmax > 0.0) {
            const unsigned long long gb = (unsigned long long)__double_as_longlong(gmax);
            atomicMax(grad_bits, gb);
            atomicMax(grad_bits + 7, gb);
        }
        if (inact) atomicAdd(n_inactive, inact);
    }
}

__device__ __forceinline__ void dmma_f64(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// pose blocks (ba.py:389-394) and Schur blocks E C0^-1 E^T (ba.py:405-413):
// one warp per union key, fixed lane-strided order + xor-tree reduction
template <int UNR, int MINB>
__global__ void __launch_bounds__(128, MINB) k_key_blocks(
    int64_t W, const int32_t* key_seg_ptr, const int32_t* key_seg, const double* seg_h,
    const int32_t* __restrict__ key_run_ptr, const int32_t* __restrict__ run_l,
    const int32_t* __restrict__ run_r, const int32_t* __restrict__ run_len,
    const double* __restrict__ uinc, const double* __restrict__ inc_block,
    double* __restrict__ pose_blocks, double* __restrict__ schur_blocks, int pose_only) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t w = warp; w < W; w += nwarps) {
        // lane q < 21 sums upper entry q over the key's segments in segment
        // order (most keys have two segments, i->j and j->i; a frame's
        // diagonal key ~2x the odometry radius), 4 loads in flight, and
        // writes it and its mirror: no cross-lane reduction
        {
            const int32_t k0 = key_seg_ptr[w], k1 = key_seg_ptr[w + 1];
            const int q = lane;
            double hq = 0.0;
            int32_t k = k0;
            for (; k + 4 <= k1; k += 4) {
                double v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int32_t code = __ldg(key_seg + k + u);
                    const double x = lane < 21 ? __ldg(seg_h + (int64_t)(code >> 1) * 21 + q) : 0.0;
                    v[u] = (code & 1) ? -x : x;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) hq += v[u];
            }
            for (; k < k1; ++k) {
                const int32_t code = __ldg(key_seg + k);
                const double x = lane < 21 ? __ldg(seg_h + (int64_t)(code >> 1) * 21 + q) : 0.0;
                hq += (code & 1) ? -x : x;
            }
            if (lane < 21) {
                int a = 0;
                while (a < 5 && utri(a + 1, a + 1) <= lane) ++a;
                const int b = a + (lane - utri(a, a));
                pose_blocks[w * 36 + a * 6 + b] = hq;
                if (a != b) pose_blocks[w * 36 + b * 6 + a] = hq;
            }
        }
        if (pose_only) continue;
        // Schur block = U^T V over the key's pair runs (l+t, r+t) on the FP64
        // tensor cores: per m8n8k4 step 4 pairs; lane (k = lane&3, i = lane>>2)
        // loads component i of pair k of both sides, so a quad reads 4
        // consecutive 48-byte incidence blocks (coalesced).  4 independent
        // accumulators break the DMMA dependency chain.
        const int kq = lane & 3, ci = lane >> 2;
        double c[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
        for (int32_t q = key_run_ptr[w]; q < key_run_ptr[w + 1]; ++q) {
            const int32_t len = run_len[q];
            const double* ub = uinc + (int64_t)run_l[q] * 6;
            const double* vb = inc_block + (int64_t)run_r[q] * 6;
            // UNR steps (4*UNR pairs) of loads in flight, then UNR DMMAs
            for (int32_t t0 = 0; t0 < len; t0 += 4 * UNR) {
                double a[UNR], b[UNR];
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const int32_t t = t0 + 4 * u + kq;
                    const bool ok = t < len && ci < 6;
                    a[u] = ok ? __ldg(ub + (int64_t)t * 6 + ci) : 0.0;
                    b[u] = ok ? __ldg(vb + (int64_t)t * 6 + ci) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < UNR; ++u) dmma_f64(c[u & 3][0], c[u & 3][1], a[u], b[u]);
            }
        }
        // C[i][j] at lane (i = lane>>2, j = 2*(lane&3) + h)
        const int oi = lane >> 2;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int oj = 2 * (lane & 3) + h;
            const double v = (c[0][h] + c[1][h]) + (c[2][h] + c[3][h]);
            if (oi < 6 && oj < 6) schur_blocks[w * 36 + oi * 6 + oj] = v;
        }
    }
}

// Grouped Schur complement: per chunk of rows sharing one incidence-var list
// (v_0 < ... < v_{m-1}), stage W (6m x nr: var j's 6 components on rows
// 6j..6j+5, columns = rows of the chunk) in shared memory and form the upper
// triangle of W W^T on DMMA (m8n8k4, K = rows) over 8x8 tiles of the packed
// 6m rows; every element lands in its 6x6 var block (j1 <= j2), the chunk's
// contribution to schur_blocks[key(v_j1, v_j2)] (ba.py:405-413).
__global__ void __launch_bounds__(256) k_group_syrk(const int4* __restrict__ chunks,
                                                     const int32_t* __restrict__ rows,
                                                     const int32_t* __restrict__ rinc_ptr,
                                                     const int32_t* __restrict__ rinc,
                                                     const double* __restrict__ w,
                                                     double* __restrict__ sbuf) {
    extern __shared__ double Ws[];
    const int4 ch = chunks[blockIdx.x];
    const int nr = ch.y, m = ch.z;
    const int n6 = 6 * m, TR = (n6 + 7) / 8;
    // K padded to the m8n8k4 step; row stride = 4 (mod 16) doubles
    const int ldt = ((((nr + 3) & ~3) + 11) / 16) * 16 + 4;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int x = tid; x < m * ldt; x += blockDim.x) {
        const int j = x / ldt, t = x % ldt;
        double v[6] = {0, 0, 0, 0, 0, 0};
        if (t < nr) {
            const int32_t r = rows[ch.x + t];
            const double2* src =
                reinterpret_cast<const double2*>(w + (int64_t)rinc[rinc_ptr[r] + j] * 6);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const double2 u = __ldg(src + q);
                v[2 * q] = u.x;
                v[2 * q + 1] = u.y;
            }
        }
#pragma unroll
        for (int c = 0; c < 6; ++c) Ws[(6 * j + c) * ldt + t] = v[c];
    }
    // zero rows up to a whole 2 x 2 block of tiles (16 rows)
    const int TB2 = (TR + 1) / 2;
    for (int x = tid; x < (16 * TB2 - n6) * ldt; x += blockDim.x) Ws[n6 * ldt + x] = 0.0;
    __syncthreads();
    // upper triangle of 2 x 2 blocks of 8 x 8 tiles, one block per warp and
    // round: 4 operand loads feed 4 DMMAs (the 1 x 2 form was bound by the
    // shared-memory operand loads, 4 per 2 DMMAs)
    const int nb = TB2 * (TB2 + 1) / 2;
    const int lr = lane >> 2, lc = lane & 3;
    const int kend = (nr + 3) & ~3;
    for (int q = warp; q < nb; q += 8) {
        int bi = 0, rem = q;
        while (rem >= TB2 - bi) {
            rem -= TB2 - bi;
            ++bi;
        }
        const int bj = bi + rem;
        double c[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};
        const double* a0 = Ws + (16 * bi + lr) * ldt + lc;
        const double* a1 = a0 + 8 * ldt;
        const double* b0 = Ws + (16 * bj + lr) * ldt + lc;
        const double* b1 = b0 + 8 * ldt;
#pragma unroll 4
        for (int k = 0; k < kend; k += 4) {
            const double x0 = a0[k], x1 = a1[k], y0 = b0[k], y1 = b1[k];
            dmma_f64(c[0][0][0], c[0][0][1], x0, y0);
            dmma_f64(c[0][1][0], c[0][1][1], x0, y1);
            dmma_f64(c[1][0][0], c[1][0][1], x1, y0);
            dmma_f64(c[1][1][0], c[1][1][1], x1, y1);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int tr = 2 * bi + u, tc = 2 * bj + v;
                if (tr > tc || tc >= TR) continue;
                const int r = 8 * tr + lr;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int cc = 8 * tc + 2 * lc + h;
                    if (r >= n6 || cc >= n6) continue;
                    const int vr = r / 6, vc = cc / 6, i = r % 6, jj = cc % 6;
                    if (vr > vc) continue;          // mirror of an element of this tile
                    const int blk = vr * m - vr * (vr - 1) / 2 + (vc - vr);
                    double* dst = sbuf + ((int64_t)ch.w + blk) * 36;
                    dst[i * 6 + jj] = c[u][v][h];
                    if (vr == vc) dst[jj * 6 + i] = c[u][v][h];   // symmetric diagonal block
                }
            }
    }
}

// schur_blocks[key] = sum of the key's chunk blocks in chunk order (warp per key)
__global__ void k_key_schur_sum(int64_t W, const int32_t* __restrict__ key_blk_ptr,
                                const int32_t* __restrict__ key_blk,
                                const double* __restrict__ sbuf, double* __restrict__ schur) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = warp; k < W; k += nwarps) {
        double s0 = 0.0, s1 = 0.0;
        for (int32_t q = key_blk_ptr[k]; q < key_blk_ptr[k + 1]; ++q) {
            const double* b = sbuf + (int64_t)key_blk[q] * 36;
            s0 += __ldg(b + lane);
            if (lane < 4) s1 += __ldg(b + 32 + lane);
        }
        schur[k * 36 + lane] = s0;
        if (lane < 4) schur[k * 36 + 32 + lane] = s1;
    }
}

// Small problems (few keys / vars, e.g. a 22-frame window): the same sums
// with one 4-warp CTA per key / var, so each key's segments and pair runs are
// split over 4 warps instead of one; partial results combine in a fixed
// warp order (deterministic).
template <int UNR>
__global__ void __launch_bounds__(128) k_key_blocks_cta(
    int64_t W, const int32_t* key_seg_ptr, const int32_t* key_seg, const double* seg_h,
    const int32_t* __restrict__ key_run_ptr, const int32_t* __restrict__ run_l,
    const int32_t* __restrict__ run_r, const int32_t* __restrict__ run_len,
    const double* __restrict__ uinc, const double* __restrict__ inc_block,
    double* __restrict__ pose_blocks, double* __restrict__ schur_blocks, int pose_only) {
    __shared__ double hp[4][21];
    __shared__ double sp[4][64];
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    for (int64_t w = blockIdx.x; w < W; w += gridDim.x) {
        double h[21];
#pragma unroll
        for (int k = 0; k < 21; ++k) h[k] = 0.0;
        for (int32_t k = key_seg_ptr[w] + wi * 32 + lane; k < key_seg_ptr[w + 1]; k += 128) {
            const int32_t code = key_seg[k];
            const double sgn = (code & 1) ? -1.0 : 1.0;
            const double* src = seg_h + (int64_t)(code >> 1) * 21;
#pragma unroll
            for (int q = 0; q < 21; ++q) h[q] += sgn * src[q];
        }
#pragma unroll
        for (int q = 0; q < 21; ++q) h[q] = warp_sum(h[q]);
        if (lane < 21) {
            double v = 0.0;
#pragma unroll
            for (int q = 0; q < 21; ++q) v = (q == lane) ? h[q] : v;
            hp[wi][lane] = v;
        }
        const int kq = lane & 3, ci = lane >> 2;
        double c[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
        if (!pose_only) {
            for (int32_t q = key_run_ptr[w]; q < key_run_ptr[w + 1]; ++q) {
                const int32_t len = run_len[q];
                const double* ub = uinc + (int64_t)run_l[q] * 6;
                const double* vb = inc_block + (int64_t)run_r[q] * 6;
                for (int32_t t0 = wi * 4 * UNR; t0 < len; t0 += 16 * UNR) {
                    double a[UNR], b[UNR];
#pragma unroll
                    for (int u = 0; u < UNR; ++u) {
                        const int32_t t = t0 + 4 * u + kq;
                        const bool ok = t < len && ci < 6;
                        a[u] = ok ? __ldg(ub + (int64_t)t * 6 + ci) : 0.0;
                        b[u] = ok ? __ldg(vb + (int64_t)t * 6 + ci) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < UNR; ++u) dmma_f64(c[u & 3][0], c[u & 3][1], a[u], b[u]);
                }
            }
        }
        sp[wi][2 * lane] = (c[0][0] + c[1][0]) + (c[2][0] + c[3][0]);
        sp[wi][2 * lane + 1] = (c[0][1] + c[1][1]) + (c[2][1] + c[3][1]);
        __syncthreads();
        if (threadIdx.x < 36) {
            const int idx = threadIdx.x, a = idx / 6, b = idx % 6;
            const int t = a <= b ? utri(a, b) : utri(b, a);
            pose_blocks[w * 36 + idx] = ((hp[0][t] + hp[1][t]) + hp[2][t]) + hp[3][t];
            if (!pose_only) {
                // fragment element (i, j) sits at lane 4 i + j / 2, slot j % 2
                const int e = 2 * (4 * a + b / 2) + (b & 1);
                schur_blocks[w * 36 + idx] = ((sp[0][e] + sp[1][e]) + sp[2][e]) + sp[3][e];
            }
        }
        __syncthreads();
    }
}

// scale pin direction (ba.py:419-426)
__device__ __forceinline__ void pin_direction(const double* t, int32_t first_free,
                                              int32_t anchor, double* scal) {
    double u[3];
    for (int k = 0; k < 3; ++k) u[k] = t[3 * first_free + k] - (anchor >= 0 ? t[3 * anchor + k] : 0.0);
    const double nrm = sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
    if (nrm > 1e-9) {
        scal[1] = 1.0;
        for (int k = 0; k < 3; ++k) scal[2 + k] = u[k] / nrm;
    } else {
        scal[1] = 0.0;
    }
}

__global__ void __launch_bounds__(128) k_var_rhs_cta(
    int64_t n, const int32_t* var_seg_ptr, const int32_t* var_seg, const double* seg_g,
    const int32_t* var_inc_ptr, const int32_t* inc_row, const double* inc_block,
    const double* cinv0, const double* rhs_depth, double* rhs_pose, double* rhs_schur,
    unsigned long long* grad_bits, const double* pin_t, int32_t pin_first, int32_t pin_anchor,
    double* scal) {
    __shared__ double part[4][12];
    // the scale-gauge pin (ba.py:311-319) rides along: one thread of CTA 0
    // (pin_t == nullptr: the problem's scale is not degenerate)
    if (pin_t && blockIdx.x == 0 && threadIdx.x == 0) pin_direction(pin_t, pin_first, pin_anchor, scal);
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    for (int64_t v = blockIdx.x; v < n; v += gridDim.x) {
        double g[6] = {0, 0, 0, 0, 0, 0}, sc[6] = {0, 0, 0, 0, 0, 0};
        for (int32_t k = var_seg_ptr[v] + threadIdx.x; k < var_seg_ptr[v + 1]; k += 128) {
            const int32_t code = var_seg[k];
            const double sgn = (code & 1) ? -1.0 : 1.0;
#pragma unroll
            for (int a = 0; a < 6; ++a) g[a] += sgn * seg_g[(int64_t)(code >> 1) * 6 + a];
        }
        for (int32_t i = var_inc_ptr[v] + threadIdx.x; i < var_inc_ptr[v + 1]; i += 128) {
            const int32_t row = inc_row[i];
            const double r = rhs_depth[row] * cinv0[row];
#pragma unroll
            for (int a = 0; a < 6; ++a) sc[a] += inc_block[(int64_t)i * 6 + a] * r;
        }
#pragma unroll
        for (int a = 0; a < 6; ++a) {
            g[a] = warp_sum(g[a]);
            sc[a] = warp_sum(sc[a]);
        }
        if (lane < 12) {
            double x = 0.0;
#pragma unroll
            for (int a = 0; a < 6; ++a) {
                x = (lane == a) ? g[a] : x;
                x = (lane == 6 + a) ? sc[a] : x;
            }
            part[wi][lane] = x;
        }
        __syncthreads();
        if (threadIdx.x < 12) {
            const int a = threadIdx.x;
            const double x = ((part[0][a] + part[1][a]) + part[2][a]) + part[3][a];
            if (a < 6) {
                rhs_pose[v * 6 + a] = x;
                atomicMax(grad_bits, (unsigned long long)__double_as_longlong(fabs(x)));
            } else {
                rhs_schur[v * 6 + a - 6] = x;
            }
        }
        __syncthreads();
    }
}

}  // namespace

int32_t objective(dpv_problem* p, const double* q, const double* t, const double* d, double* out,
                  cudaStream_t st) {
    DPV_TRY(frame_rotations(p, q, st));
    DPV_TSTART("objective", st);
    if (p->m == 9 && p->S > 0)
    {
        k_objective_seg<9, 3, 4, true><<<kObjBlocks, 256, 0, st>>>(
            p->S, p->E, p->P, p->seg_ptr, p->seg_src, p->seg_dst, p->a_row, p->a_tgt, p->a_w,
            p->r_ray, p->frame_R, t, d, p->intr[0], p->intr[1], p->intr[2], p->intr[3],
            p->obj_part);
    }
    else
        k_objective<<<kObjBlocks, 256, 0, st>>>(p->E, p->m, p->P, p->a_src, p->a_dst, p->a_row,
                                                p->a_tgt, p->a_w, p->r_ray, p->frame_R, t, d,
                                                p->intr[0], p->intr[1], p->intr[2], p->intr[3],
                                                p->obj_part);
    DPV_CHECK_LAUNCH();
    DPV_TSTART("sum_parts", st);
    k_sum_parts<<<1, 1024, 0, st>>>(kObjBlocks, p->obj_part, out);
    DPV_CHECK_LAUNCH();
    return DPV_OK;
}

int32_t residuals(dpv_problem* p, const double* q, const double* t, const double* d, double* res,
                  uint8_t* valid, cudaStream_t st) {
    DPV_TRY(frame_rotations(p, q, st));
    if (p->E == 0) return DPV_OK;
    DPV_TSTART("residuals", st);
    k_residuals<<<grid_for(p->E, 256), 256, 0, st>>>(p->E, p->m, p->P, p->a_src, p->a_dst,
                                                      p->a_row, p->a_pidx, p->a_tgt, p->r_ray,
                                                      p->frame_R, t, d, p->intr[0], p->intr[1],
                                                      p->intr[2], p->intr[3], res, valid);
    DPV_CHECK_LAUNCH();
    return DPV_OK;
}

int32_t coords(dpv_problem* p, const double* q, const double* t, const double* d, double scale,
               double* out, cudaStream_t st) {
    DPV_TRY(frame_rotations(p, q, st));
    if (p->E == 0) return DPV_OK;
    DPV_TSTART("coords", st);
    k_coords<<<grid_for(p->E, 256), 256, 0, st>>>(p->E, p->m, p->P, p->a_src, p->a_dst, p->a_row,
                                                   p->a_pidx, p->r_ray, p->frame_R, t, d,
                                                   p->intr[0], p->intr[1], p->intr[2], p->intr[3],
                                                   scale, out);
    DPV_CHECK_LAUNCH();
    return DPV_OK;
}

int32_t coords_sel(dpv_problem* p, const double* q, const double* t, const double* d,
                   double scale, const int64_t* sel, int64_t n_sel, double* out,
                   cudaStream_t st) {
    DPV_TRY(frame_rotations(p, q, st));
    if (n_sel == 0) return DPV_OK;
    DPV_TSTART("coords", st);
    k_coords_sel<<<grid_for(n_sel * p->m, 256), 256, 0, st>>>(
        n_sel, sel, p->p_pos, p->m, p->P, p->a_src, p->a_dst, p->a_row, p->r_ray, p->frame_R, t,
        d, p->intr[0], p->intr[1], p->intr[2], p->intr[3], scale, out);
    DPV_CHECK_LAUNCH();
    return DPV_OK;
}

int32_t update_targets(dpv_problem* p, const double* tgt, const double* conf, cudaStream_t st) {
    if (p->E == 0) return DPV_OK;
    DPV_TSTART("update_targets", st);
    k_update_targets<<<grid_for(p->E, 256), 256, 0, st>>>(p->E, p->m, p->p_pos, tgt, conf,
                                                           p->a_tgt, p->a_w);
    DPV_CHECK_LAUNCH();
    return DPV_OK;
}

// K2+K3 edge pass at (q, t, d): per-edge terms, per-segment Gram sums and,
// when obj != nullptr, the objective at that state (fixed-order sum of the
// per-segment sums) - the LM driver evaluates every candidate this way, so an
// accepted candidate's edge pass is already done (speculative assembly).
int32_t assemble_edges_pass(dpv_problem* p, const double* q, const double* t, const double* d,
                            double* obj, cudaStream_t st) {
    DPV_TRY(frame_rotations(p, q, st));
    if (p->S > 0) {
        DPV_ARG(p->m == 9, "assembly kernel is instantiated for 3x3 patches");
        // persistent: every warp walks many segments so the staging pipeline
        // stays full; 4 warps x 2 blocks per SM (225 registers): 0.50 ms at
        // cfg3 (register-capped 3x3 / 2x5 / 1x10 shapes spill: 0.83-0.86 ms)
        constexpr int kNW = 4, kMinB = 2;
        const size_t smem = sizeof(double) * 2 * kStgDoubles * kNW;
        static size_t cur = 0;
        DPV_TRY(ensure_smem(k_assemble_edges_stg<kNW, kMinB>, smem, cur));
        const int pblocks = (int)std::min<int64_t>((p->S + kNW - 1) / kNW,
                                                   (int64_t)sm_count() * kMinB);
        DPV_TSTART("assemble_edges", st);
        k_assemble_edges_stg<kNW, kMinB><<<pblocks, 32 * kNW, smem, st>>>(
            p->S, p->E, p->P, p->seg_ptr, p->seg_src, p->seg_dst, p->a_row, p->a_tgt, p->a_w,
            p->r_ray, p->frame_R, t, d, p->intr[0], p->intr[1], p->intr[2], p->intr[3],
            p->e_terms, p->seg_h, p->seg_g, obj ? p->seg_obj : nullptr);
        DPV_CHECK_LAUNCH();
    }
    if (obj) {
        if (p->S > 0) {
            // fixed-order two-level sum: contiguous slices per block, then the
            // block partials (deterministic)
            const int nb = (int)std::min<int64_t>(kObjBlocks, (p->S + 255) / 256);
            DPV_TSTART("sum_parts", st);
            k_slice_sums<<<nb, 256, 0, st>>>(p->S, p->seg_obj, p->obj_part);
            DPV_CHECK_LAUNCH();
            k_sum_parts<<<1, 1024, 0, st>>>(nb, p->obj_part, obj);
            DPV_CHECK_LAUNCH();
        } else {
            DPV_CUDA(cudaMemsetAsync(obj, 0, sizeof(double), st));
        }
    }
    return DPV_OK;
}

// the rest of the assembly (rows, incidences, Schur, rhs, pin) from the
// edge pass's terms; t = the state's translations (scale pin)
int32_t assemble_rest(dpv_problem* p, const double* t, cudaStream_t st) {
    DPV_CUDA(cudaMemsetAsync(p->scal, 0, sizeof(double) * 8, st));
    auto* grad_bits = reinterpret_cast<unsigned long long*>(p->scal);
    auto* n_inactive = reinterpret_cast<unsigned long long*>(p->scal + 6);
    if (p->P > 0) {
        DPV_TSTART("rows", st);
        if (p->P < (int64_t)sm_count() * 64)      // few rows: a warp each
            k_rows_warp<<<grid_for(p->P * 32, 256), 256, 0, st>>>(
                p->P, p->E, p->row_ptr, p->row_pos, p->e_terms, p->depth_diag, p->rhs_depth,
                p->active, p->cinv0, grad_bits, n_inactive);
        else
            k_rows<<<grid_for(p->P, 256), 256, 0, st>>>(p->P, p->E, p->row_ptr, p->row_pos,
                                                         p->e_terms, p->depth_diag, p->rhs_depth,
                                                         p->active, p->cinv0, grad_bits,
                                                         n_inactive);
        DPV_CHECK_LAUNCH();
    }
    if (p->I > 0) {
        DPV_TSTART("incidences", st);
        k_incidences2<<<grid_for(p->I, 256), 256, 0, st>>>(p->I, p->inc_ptr, p->inc_con,
                                                            p->inc_row, p->e_terms, p->cinv0,
                                                            p->inc_block, p->uinc, p->grouped);
        DPV_CHECK_LAUNCH();
    }
    // few keys / vars: one CTA each (a warp each would leave most SMs idle)
    // (at cfg3 the per-key CTA form loses: 0.98 vs 0.51 ms)
    const bool small = p->W < (int64_t)sm_count() * 8 && !p->grouped;
    if (p->W > 0 && small) {
        DPV_TSTART("key_blocks", st);
        k_key_blocks_cta<4><<<(int)p->W, 128, 0, st>>>(
            p->W, p->key_seg_ptr, p->key_seg, p->seg_h, p->key_run_ptr, p->run_l, p->run_r,
            p->run_len, p->uinc, p->inc_block, p->pose_blocks, p->schur_blocks, 0);
        DPV_CHECK_LAUNCH();
    } else if (p->W > 0) {
        int blocks = (int)std::min<int64_t>((p->W + 3) / 4, (int64_t)sm_count() * 64);
        DPV_TSTART("key_blocks", st);
        k_key_blocks<16, 3><<<blocks, 128, 0, st>>>(p->W, p->key_seg_ptr, p->key_seg, p->seg_h,
                                                    p->key_run_ptr, p->run_l, p->run_r,
                                                    p->run_len, p->uinc, p->inc_block,
                                                    p->pose_blocks, p->schur_blocks, p->grouped);
        DPV_CHECK_LAUNCH();
        if (p->grouped) {
            static size_t cur = 0;
            const size_t smem = sizeof(double) * kSyrkSmemDoubles + 2048;
            DPV_TRY(ensure_smem(k_group_syrk, smem, cur));
            DPV_TSTART("group_syrk", st);
            k_group_syrk<<<(int)p->n_chunks, 256, smem, st>>>(p->g_chunks, p->g_rows, p->rinc_ptr,
                                                              p->rinc, p->uinc, p->g_sbuf);
            DPV_CHECK_LAUNCH();
            DPV_TSTART("key_schur_sum", st);
            k_key_schur_sum<<<grid_for(p->W * 32, 256), 256, 0, st>>>(
                p->W, p->key_blk_ptr, p->key_blk, p->g_sbuf, p->schur_blocks);
            DPV_CHECK_LAUNCH();
        }
    }
    if (p->n > 0) {
        DPV_TSTART("var_rhs", st);
        // one 4-warp CTA per var at every size (cfg3: 0.078 -> 0.058 ms
        // against a warp per var)
        k_var_rhs_cta<<<(int)std::min<int64_t>(p->n, 65535), 128, 0, st>>>(
            p->n, p->var_seg_ptr, p->var_seg, p->seg_g, p->var_inc_ptr, p->inc_row,
            p->inc_block, p->cinv0, p->rhs_depth, p->rhs_pose, p->rhs_schur, grad_bits,
            p->scale_degenerate ? t : nullptr, p->first, p->touched0, p->scal);
        DPV_CHECK_LAUNCH();
    }
    return DPV_OK;
}

int32_t assemble(dpv_problem* p, const double* q, const double* t, const double* d,
                 cudaStream_t st) {
    DPV_TRY(assemble_edges_pass(p, q, t, d, nullptr, st));
    return assemble_rest(p, t, st);
}

}  // namespace dpv
