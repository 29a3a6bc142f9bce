// Flow oracle on the device (reference synthetic.py:222-287, fill_flow; SURVEY
// 8(f) rank 1): per selected edge the ground-truth reprojection of the source
// patch grid into the target frame, the Gaussian shift, the seeded gross
// outliers and the observability mask, written as flow targets and
// confidences.  The random draws come from the host generator (numpy's
// default_rng stream, drawn in the reference's order) so the inputs stay
// bit-identical; every floating-point operation below is an explicit
// round-to-nearest intrinsic in the order numpy evaluates the reference
// expressions (measured on this image's numpy):
//   * np.einsum("eb,eb->e", R[:, :, 2], L - t) with a strided operand:
//     ((a0 b0 + a1 b1) + a2 b2), no fused multiply-add;
//   * batched matmul (E,9,3) @ (E,3,3): fma(a2, b2, fma(a1, b1, a0 b0));
//   * separate ufuncs for every other operator (no contraction).
#include "problem.cuh"

namespace dpv {
namespace {

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dadd_rn(a, -b); }
__device__ __forceinline__ double dvd(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double mm3(double a0, double b0, double a1, double b1, double a2,
                                      double b2) {
    return __fma_rn(a2, b2, __fma_rn(a1, b1, mul(a0, b0)));
}

// pinhole_rays + _np_reproject_exact (package synthetic.py:101-115, the
// reference expression of geometry.py:478-529 without Jacobians)
struct Reproj {
    double px, py;
    bool valid;
};
__device__ __forceinline__ Reproj reproject_cell(double gx, double gy, double inv_depth,
                                                 const double* Ri, const double* ti,
                                                 const double* Rj, const double* tj,
                                                 const double* intr) {
    const double rx = dvd(sub(gx, intr[2]), intr[0]);
    const double ry = dvd(sub(gy, intr[3]), intr[1]);
    const double c0 = dvd(rx, inv_depth), c1 = dvd(ry, inv_depth), c2 = dvd(1.0, inv_depth);
    double w[3], d[3], x[3];
    for (int a = 0; a < 3; ++a)   // x_cam @ R_i^T + t_i
        w[a] = add(mm3(c0, Ri[3 * a], c1, Ri[3 * a + 1], c2, Ri[3 * a + 2]), ti[a]);
    for (int a = 0; a < 3; ++a) d[a] = sub(w[a], tj[a]);
    for (int a = 0; a < 3; ++a)   // (x_world - t_j) @ R_j
        x[a] = mm3(d[0], Rj[a], d[1], Rj[3 + a], d[2], Rj[6 + a]);
    Reproj r;
    r.valid = x[2] > 1e-8;
    const double zs = r.valid ? x[2] : 1.0;
    r.px = add(dvd(mul(intr[0], x[0]), zs), intr[2]);
    r.py = add(dvd(mul(intr[1], x[1]), zs), intr[3]);
    return r;
}

__global__ void k_fill_flow(int64_t n, const int64_t* __restrict__ sel,
                            const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                            const int32_t* __restrict__ gpatch, const double* __restrict__ grid,
                            const double* __restrict__ rot, const double* __restrict__ trans,
                            const double* __restrict__ lms, const int64_t* __restrict__ plm,
                            const double* __restrict__ shift, const uint8_t* __restrict__ outlier,
                            const double* __restrict__ gross, double low_conf, double w, double h,
                            double slack, double fx, double fy, double cx, double cy, int m,
                            double* __restrict__ target, double* __restrict__ conf) {
    const double intr[4] = {fx, fy, cx, cy};
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = sel ? sel[k] : k;
        const int s = src[e], t = dst[e];
        const int64_t g = gpatch[e];
        const double* Ri = rot + 9 * s;
        const double* ti = trans + 3 * s;
        const double* L = lms + 3 * plm[g];
        // cam_z = R_s[:, 2] . (L - t_s)  (einsum, strided operand)
        const double z = add(add(mul(Ri[2], sub(L[0], ti[0])), mul(Ri[5], sub(L[1], ti[1]))),
                             mul(Ri[8], sub(L[2], ti[2])));
        const double inv_depth = dvd(1.0, z);
        bool obs = true;
        double* out = target + k * m * 2;
        for (int c = 0; c < m; ++c) {
            const Reproj r = reproject_cell(grid[(g * m + c) * 2], grid[(g * m + c) * 2 + 1],
                                            inv_depth, Ri, ti, rot + 9 * t, trans + 3 * t, intr);
            obs = obs && r.valid && r.px > -slack && r.px < w + slack && r.py > -slack &&
                  r.py < h + slack;
            out[2 * c] = r.px;
            out[2 * c + 1] = r.py;
        }
        const double s0 = shift[2 * k], s1 = shift[2 * k + 1];
        const bool bad = outlier[k] && obs;
        for (int c = 0; c < m; ++c) {
            double u = add(out[2 * c], s0), v = add(out[2 * c + 1], s1);
            if (bad) {
                u = add(u, gross[2 * k]);
                v = add(v, gross[2 * k + 1]);
            }
            out[2 * c] = u;
            out[2 * c + 1] = v;
        }
        const double cf = !obs ? 0.0 : (bad ? low_conf : 1.0);
        conf[2 * k] = cf;
        conf[2 * k + 1] = cf;
    }
}

// initial targets = reprojection at the current state (graph.py:152-164,
// package synthetic._reproject_targets): patch inverse depths given
__global__ void k_reproject_exact(int64_t n, const int64_t* __restrict__ sel,
                                  const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                                  const int32_t* __restrict__ gpatch,
                                  const double* __restrict__ grid, const double* __restrict__ rot,
                                  const double* __restrict__ trans,
                                  const double* __restrict__ depth, double fx, double fy,
                                  double cx, double cy, int m, double* __restrict__ pix) {
    const double intr[4] = {fx, fy, cx, cy};
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = sel ? sel[k] : k;
        const int s = src[e], t = dst[e];
        const int64_t g = gpatch[e];
        for (int c = 0; c < m; ++c) {
            const Reproj r = reproject_cell(grid[(g * m + c) * 2], grid[(g * m + c) * 2 + 1],
                                            depth[g], rot + 9 * s, trans + 3 * s, rot + 9 * t,
                                            trans + 3 * t, intr);
            pix[(k * m + c) * 2] = r.px;
            pix[(k * m + c) * 2 + 1] = r.py;
        }
    }
}

// visible_landmarks for every frame at once (synthetic.py:68-79): camera
// points inv_pose.act(L) = L + w t + u x t (t = 2 u x L) + inv_t with
// numpy's np.cross (a1 b2 - a2 b1, no contraction), projection, the depth /
// margin tests.  One thread per (frame, landmark); flags (F, L) uint8.
__global__ void k_visible(int64_t F, int64_t L, const double* __restrict__ inv_q,
                          const double* __restrict__ inv_t, const double* __restrict__ lms,
                          double fx, double fy, double cx, double cy, double margin, double umax,
                          double vmax, uint8_t* __restrict__ flags) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < F * L;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = x / L, l = x % L;
        const double* q = inv_q + 4 * f;
        const double v0 = lms[3 * l], v1 = lms[3 * l + 1], v2 = lms[3 * l + 2];
        const double u0 = q[0], u1 = q[1], u2 = q[2], w = q[3];
        const double t0 = mul(2.0, sub(mul(u1, v2), mul(u2, v1)));
        const double t1 = mul(2.0, sub(mul(u2, v0), mul(u0, v2)));
        const double t2 = mul(2.0, sub(mul(u0, v1), mul(u1, v0)));
        const double c0 = sub(mul(u1, t2), mul(u2, t1));
        const double c1 = sub(mul(u2, t0), mul(u0, t2));
        const double c2 = sub(mul(u0, t1), mul(u1, t0));
        const double* it = inv_t + 3 * f;
        const double px = add(add(add(v0, mul(w, t0)), c0), it[0]);
        const double py = add(add(add(v1, mul(w, t1)), c1), it[1]);
        const double pz = add(add(add(v2, mul(w, t2)), c2), it[2]);
        const bool valid = pz > 1e-8;
        const double zs = valid ? pz : 1.0;
        const double u = add(dvd(mul(fx, px), zs), cx);
        const double v = add(dvd(mul(fy, py), zs), cy);
        flags[x] = (valid && pz > 0.5 && u >= margin && u <= umax && v >= margin && v <= vmax)
                       ? 1 : 0;
    }
}

}  // namespace
}  // namespace dpv

using namespace dpv;

extern "C" {

int32_t dpv_fill_flow(const dpv_graph* g, const double* rot, const double* trans,
                      const double* landmarks, const int64_t* patch_landmark, const int64_t* sel,
                      int64_t n, const double* shift, const uint8_t* outlier, const double* gross,
                      double low_confidence, double width, double height, double* target,
                      double* conf, void* stream) {
    DPV_ABI_TRY
    clear_error();
    DPV_ARG(g && n >= 0 && g->cells > 0, "bad fill_flow args");
    if (n == 0) return DPV_OK;
    DPV_ARG(rot && trans && landmarks && patch_landmark && shift && outlier && gross && target &&
                conf && g->edge_src && g->edge_dst && g->edge_gpatch && g->patch_grid,
            "NULL fill_flow argument");
    cudaStream_t st = as_stream(stream);
    const double slack = 0.25 * (width > height ? width : height);   // synthetic.py:255
    DPV_TSTART("fill_flow", st);
    k_fill_flow<<<grid_for(n, 128), 128, 0, st>>>(
        n, sel, g->edge_src, g->edge_dst, g->edge_gpatch, g->patch_grid, rot, trans, landmarks,
        patch_landmark, shift, outlier, gross, low_confidence, width, height, slack, g->intr[0],
        g->intr[1], g->intr[2], g->intr[3], g->cells, target, conf);
    DPV_CHECK_LAUNCH();
    return DPV_OK;
    DPV_ABI_CATCH
}

int32_t dpv_reproject_exact(const dpv_graph* g, const double* rot, const double* trans,
                            const double* patch_depth, const int64_t* sel, int64_t n, double* pix,
                            void* stream) {
    DPV_ABI_TRY
    clear_error();
    DPV_ARG(g && n >= 0 && g->cells > 0, "bad reproject_exact args");
    if (n == 0) return DPV_OK;
    DPV_ARG(rot && trans && patch_depth && pix && g->edge_src && g->edge_dst && g->edge_gpatch &&
                g->patch_grid,
            "NULL reproject_exact argument");
    cudaStream_t st = as_stream(stream);
    DPV_TSTART("reproject_exact", st);
    k_reproject_exact<<<grid_for(n, 128), 128, 0, st>>>(n, sel, g->edge_src, g->edge_dst,
                                                        g->edge_gpatch, g->patch_grid, rot, trans,
                                                        patch_depth, g->intr[0], g->intr[1],
                                                        g->intr[2], g->intr[3], g->cells, pix);
    DPV_CHECK_LAUNCH();
    return DPV_OK;
    DPV_ABI_CATCH
}

int32_t dpv_visible_landmarks(int64_t n_frames, int64_t n_landmarks, const double* inv_q,
                              const double* inv_t, const double* landmarks, const double* intr,
                              double margin, double u_max, double v_max, uint8_t* flags,
                              void* stream) {
    DPV_ABI_TRY
    clear_error();
    DPV_ARG(n_frames >= 0 && n_landmarks >= 0 && intr, "bad visible_landmarks args");
    if (n_frames == 0 || n_landmarks == 0) return DPV_OK;
    DPV_ARG(inv_q && inv_t && landmarks && flags, "NULL visible_landmarks argument");
    cudaStream_t st = as_stream(stream);
    DPV_TSTART("visible_landmarks", st);
    k_visible<<<grid_for(n_frames * n_landmarks, 256), 256, 0, st>>>(
        n_frames, n_landmarks, inv_q, inv_t, landmarks, intr[0], intr[1], intr[2], intr[3], margin,
        u_max, v_max, flags);
    DPV_CHECK_LAUNCH();
    return DPV_OK;
    DPV_ABI_CATCH
}

}  // extern "C"
