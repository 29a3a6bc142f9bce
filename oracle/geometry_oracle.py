"""Float64 numpy restatement of the reference geometry used on the hot path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Each function cites the
reference definition it restates (paths under /root/reference/pkg/src/patchslam).
"""

from __future__ import annotations

import numpy as np

DEPTH_EPS = 1e-8            # geometry.py:24
SMALL_ANGLE = 1e-8          # geometry.py:26
INVERSE_DEPTH_FLOOR = 1e-6  # geometry.py:28


def quat_to_rot(q: np.ndarray) -> np.ndarray:
    """Unit quaternion (x, y, z, w) -> rotation matrix.  geometry.py:70-86."""
    x, y, z, w = (q[..., i] for i in range(4))
    r = np.empty(q.shape[:-1] + (3, 3))
    r[..., 0, 0] = 1 - 2 * (y * y + z * z)
    r[..., 0, 1] = 2 * (x * y - w * z)
    r[..., 0, 2] = 2 * (x * z + w * y)
    r[..., 1, 0] = 2 * (x * y + w * z)
    r[..., 1, 1] = 1 - 2 * (x * x + z * z)
    r[..., 1, 2] = 2 * (y * z - w * x)
    r[..., 2, 0] = 2 * (x * z - w * y)
    r[..., 2, 1] = 2 * (y * z + w * x)
    r[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return r


def hamilton(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Hamilton product a*b in (x, y, z, w) order.  geometry.py:41-53."""
    ax, ay, az, aw = (a[..., i] for i in range(4))
    bx, by, bz, bw = (b[..., i] for i in range(4))
    out = np.empty(np.broadcast_shapes(a.shape, b.shape))
    out[..., 0] = aw * bx + ax * bw + ay * bz - az * by
    out[..., 1] = aw * by - ax * bz + ay * bw + az * bx
    out[..., 2] = aw * bz + ax * by - ay * bx + az * bw
    out[..., 3] = aw * bw - ax * bx - ay * by - az * bz
    return out


def rotate(q: np.ndarray, v: np.ndarray) -> np.ndarray:
    """v + w*t + xyz x t with t = 2 xyz x v.  geometry.py:62-67."""
    u = q[..., :3]
    t = 2.0 * np.cross(u, v)
    return v + q[..., 3:] * t + np.cross(u, t)


def exp_rotation(phi: np.ndarray) -> np.ndarray:
    """Rotation vector -> quaternion, Taylor branch below 1e-8.  geometry.py:89-101."""
    phi = np.asarray(phi, dtype=float)
    theta = np.sqrt((phi * phi).sum(-1, keepdims=True))
    small = theta < SMALL_ANGLE
    with np.errstate(invalid="ignore", divide="ignore"):
        k = np.where(small, 0.5 - theta * theta / 48.0,
                     np.sin(0.5 * theta) / np.where(small, 1.0, theta))
    q = np.empty(phi.shape[:-1] + (4,))
    q[..., :3] = phi * k
    q[..., 3] = np.cos(0.5 * theta)[..., 0]
    return q


def normalize(q: np.ndarray) -> np.ndarray:
    """geometry.py:37-38."""
    return q / np.linalg.norm(q, axis=-1, keepdims=True)


def rays_from_grid(grid: np.ndarray, intr) -> np.ndarray:
    """Unit-depth rays ((x-cx)/fx, (y-cy)/fy, 1).  geometry.py:386-391."""
    fx, fy, cx, cy = (float(v) for v in intr)
    out = np.empty(grid.shape[:-1] + (3,))
    out[..., 0] = (grid[..., 0] - cx) / fx
    out[..., 1] = (grid[..., 1] - cy) / fy
    out[..., 2] = 1.0
    return out


def reproject(rays, inv_depth, rot_i, t_i, rot_j, t_j, intr, jacobians=False):
    """Per-edge patch-grid reprojection i -> j.  geometry.py:478-529.

    Returns pix (E,m,2), valid (E,m) and, with jacobians, J_pose (E,m,2,6)
    (left-multiplicative source tangent (rho, phi); target is its negation)
    and J_depth (E,m,2).  Invalid cells use z=1 and keep finite Jacobians.
    """
    fx, fy, cx, cy = (float(v) for v in intr)
    xc = rays / inv_depth[:, None, None]
    xw = np.einsum("emk,eck->emc", xc, rot_i) + t_i[:, None, :]
    rel = xw - t_j[:, None, :]
    xt = np.einsum("emk,ekc->emc", rel, rot_j)
    z = xt[..., 2]
    valid = z > DEPTH_EPS
    zs = np.where(valid, z, 1.0)
    pix = np.empty(xt.shape[:-1] + (2,))
    pix[..., 0] = fx * xt[..., 0] / zs + cx
    pix[..., 1] = fy * xt[..., 1] / zs + cy
    if not jacobians:
        return pix, valid
    # A = Jproj R_j^T: row 0 = (fx/z) R_j[:,0] - (fx x/z^2) R_j[:,2], row 1 likewise
    a = np.empty(xt.shape[:-1] + (2, 3))
    c0 = fx / zs
    c1 = fy / zs
    d0 = -fx * xt[..., 0] / (zs * zs)
    d1 = -fy * xt[..., 1] / (zs * zs)
    rj0 = rot_j[:, None, :, 0]
    rj1 = rot_j[:, None, :, 1]
    rj2 = rot_j[:, None, :, 2]
    a[..., 0, :] = c0[..., None] * rj0 + d0[..., None] * rj2
    a[..., 1, :] = c1[..., None] * rj1 + d1[..., None] * rj2
    jp = np.empty(xt.shape[:-1] + (2, 6))
    jp[..., :3] = a
    jp[..., 3:] = np.cross(xw[:, :, None, :], a)
    dxw = (t_i[:, None, :] - xw) / inv_depth[:, None, None]
    jd = (a * dxw[:, :, None, :]).sum(-1)
    return pix, valid, jp, jd
