// K2 standalone: geometry.quat_to_matrix (geometry.py:70-86) and
// geometry.reproject_grid (geometry.py:478-529) over caller arrays.  The BA
// kernels inline the same arithmetic (assemble.cu); this entry point serves
// the drop-in reproject_grid used by graph construction and the flow oracle.
#include "problem.cuh"

namespace dpv {
namespace {

__global__ void k_quat_to_matrix(int64_t n, const double* q, double* r) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        quat_to_rot(q + 4 * i, r + 9 * i);
}

// one thread per (edge, cell)
__global__ void k_reproject_grid(int64_t E, int m, const double* __restrict__ rays,
                                 const double* __restrict__ inv_depth,
                                 const double* __restrict__ rot_i, const double* __restrict__ t_i,
                                 const double* __restrict__ rot_j, const double* __restrict__ t_j,
                                 double fx, double fy, double cx, double cy,
                                 double* __restrict__ pix, uint8_t* __restrict__ valid,
                                 double* __restrict__ j_pose, double* __restrict__ j_depth) {
    const int64_t total = E * m;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = x / m;
        const double d = inv_depth[e];
        const double* ray = rays + 3 * x;
        const double* Ri = rot_i + 9 * e;
        const double* Rj = rot_j + 9 * e;
        const double* ti = t_i + 3 * e;
        const double* tj = t_j + 3 * e;
        const double xc[3] = {ray[0] / d, ray[1] / d, ray[2] / d};
        double xw[3], xt[3];
#pragma unroll
        for (int r = 0; r < 3; ++r)
            xw[r] = xc[0] * Ri[3 * r] + xc[1] * Ri[3 * r + 1] + xc[2] * Ri[3 * r + 2] + ti[r];
        const double e0 = xw[0] - tj[0], e1 = xw[1] - tj[1], e2 = xw[2] - tj[2];
#pragma unroll
        for (int k = 0; k < 3; ++k) xt[k] = e0 * Rj[k] + e1 * Rj[3 + k] + e2 * Rj[6 + k];
        const bool ok = xt[2] > kDepthEps;
        const double zs = ok ? xt[2] : 1.0;
        pix[2 * x] = fx * xt[0] / zs + cx;
        pix[2 * x + 1] = fy * xt[1] / zs + cy;
        valid[x] = ok ? 1 : 0;
        if (j_pose) {
            const double p0 = fx / zs, q0 = -fx * xt[0] / (zs * zs);
            const double p1 = fy / zs, q1 = -fy * xt[1] / (zs * zs);
            double a[2][3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                a[0][k] = p0 * Rj[3 * k] + q0 * Rj[3 * k + 2];
                a[1][k] = p1 * Rj[3 * k + 1] + q1 * Rj[3 * k + 2];
            }
            const double g[3] = {(ti[0] - xw[0]) / d, (ti[1] - xw[1]) / d, (ti[2] - xw[2]) / d};
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                double* J = j_pose + (2 * x + r) * 6;
                J[0] = a[r][0];
                J[1] = a[r][1];
                J[2] = a[r][2];
                J[3] = xw[1] * a[r][2] - xw[2] * a[r][1];
                J[4] = xw[2] * a[r][0] - xw[0] * a[r][2];
                J[5] = xw[0] * a[r][1] - xw[1] * a[r][0];
                j_depth[2 * x + r] = a[r][0] * g[0] + a[r][1] * g[1] + a[r][2] * g[2];
            }
        }
    }
}

}  // namespace

int32_t quat_to_matrix(const double* q, int64_t n, double* r, cudaStream_t st) {
    if (n <= 0) return DPV_OK;
    k_quat_to_matrix<<<grid_for(n, 256), 256, 0, st>>>(n, q, r);
    DPV_CHECK_LAUNCH();
    return DPV_OK;
}

int32_t reproject_grid(const double* rays, const double* inv_depth, const double* rot_i,
                       const double* t_i, const double* rot_j, const double* t_j,
                       const double* intr, int64_t E, int m, double* pix, uint8_t* valid,
                       double* j_pose, double* j_depth, cudaStream_t st) {
    if (E <= 0) return DPV_OK;
    DPV_ARG((j_pose == nullptr) == (j_depth == nullptr), "j_pose and j_depth go together");
    k_reproject_grid<<<grid_for(E * m, 256), 256, 0, st>>>(E, m, rays, inv_depth, rot_i, t_i,
                                                           rot_j, t_j, intr[0], intr[1], intr[2],
                                                           intr[3], pix, valid, j_pose, j_depth);
    DPV_CHECK_LAUNCH();
    return DPV_OK;
}

}  // namespace dpv
