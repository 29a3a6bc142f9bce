"""Geometry of the hot path: value types on the host, reprojection on the B200.

Value types (``Intrinsics``, ``Pose``, ``Patch``) and the small quaternion
helpers keep the reference's conventions (patchslam/geometry.py:1-12):
quaternions (x, y, z, w), world-from-camera poses x_w = R x_c + t, tangent
(rho, phi).  They are host-side bookkeeping for a handful of frames and are
written to produce bit-identical values to the reference (the synthetic-input
generator relies on that).

``reproject_grid`` — the per-edge reprojection + Jacobian kernel K2
(geometry.py:478-529) — runs only on the GPU through the C-ABI
``dpv_reproject_grid``; there is no CPU implementation in this package.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

from . import _lib
from .errors import BehindCamera, NonPositiveDepth

DEPTH_EPS = 1e-8              # geometry.py:24
SMALL_ANGLE = 1e-8            # geometry.py:26
INVERSE_DEPTH_FLOOR = 1e-6    # geometry.py:28
DEFAULT_PATCH_SIZE = 3        # geometry.py:30


# ---------------------------------------------------------------------------
# quaternion helpers (host, value types only)


def quat_normalize(q):
    return q / np.linalg.norm(q, axis=-1, keepdims=True)


def quat_mul(a, b):
    """Hamilton product, (x, y, z, w) order (geometry.py:41-53)."""
    ax, ay, az, aw = np.moveaxis(a, -1, 0)
    bx, by, bz, bw = np.moveaxis(b, -1, 0)
    return np.stack([aw * bx + ax * bw + ay * bz - az * by,
                     aw * by - ax * bz + ay * bw + az * bx,
                     aw * bz + ax * by - ay * bx + az * bw,
                     aw * bw - ax * bx - ay * by - az * bz], axis=-1)


def quat_conj(q):
    out = np.array(q, copy=True)
    out[..., :3] *= -1.0
    return out


def quat_rotate(q, v):
    """v + w t + u x t, t = 2 u x v (geometry.py:62-67)."""
    u = q[..., :3]
    t = 2.0 * np.cross(u, v)
    return v + q[..., 3:] * t + np.cross(u, t)


def quat_to_matrix(q):
    """Host rotation matrices for value types (device twin: dpv_quat_to_matrix)."""
    x, y, z, w = np.moveaxis(q, -1, 0)
    xx, yy, zz = x * x, y * y, z * z
    xy, xz, yz = x * y, x * z, y * z
    wx, wy, wz = w * x, w * y, w * z
    m = np.empty(np.shape(q)[:-1] + (3, 3))
    m[..., 0, 0] = 1 - 2 * (yy + zz)
    m[..., 0, 1] = 2 * (xy - wz)
    m[..., 0, 2] = 2 * (xz + wy)
    m[..., 1, 0] = 2 * (xy + wz)
    m[..., 1, 1] = 1 - 2 * (xx + zz)
    m[..., 1, 2] = 2 * (yz - wx)
    m[..., 2, 0] = 2 * (xz - wy)
    m[..., 2, 1] = 2 * (yz + wx)
    m[..., 2, 2] = 1 - 2 * (xx + yy)
    return m


def rotvec_to_quat(phi):
    """Quaternion exponential, Taylor branch below SMALL_ANGLE (geometry.py:89-101)."""
    phi = np.asarray(phi, dtype=float)
    theta = np.linalg.norm(phi, axis=-1, keepdims=True)
    half = 0.5 * theta
    small = theta < SMALL_ANGLE
    with np.errstate(invalid="ignore", divide="ignore"):
        k = np.where(small, 0.5 - theta * theta / 48.0,
                     np.sin(half) / np.where(small, 1.0, theta))
    q = np.empty(phi.shape[:-1] + (4,))
    q[..., :3] = phi * k
    q[..., 3] = np.cos(half)[..., 0]
    return q


def matrix_to_quat(m):
    """Shepperd's method (geometry.py:117-137)."""
    m = np.asarray(m, dtype=float)
    tr = np.trace(m)
    if tr > 0:
        s = np.sqrt(tr + 1.0) * 2.0
        q = np.array([(m[2, 1] - m[1, 2]) / s, (m[0, 2] - m[2, 0]) / s,
                      (m[1, 0] - m[0, 1]) / s, 0.25 * s])
    elif m[0, 0] >= m[1, 1] and m[0, 0] >= m[2, 2]:
        s = np.sqrt(1.0 + m[0, 0] - m[1, 1] - m[2, 2]) * 2.0
        q = np.array([0.25 * s, (m[0, 1] + m[1, 0]) / s,
                      (m[0, 2] + m[2, 0]) / s, (m[2, 1] - m[1, 2]) / s])
    elif m[1, 1] >= m[2, 2]:
        s = np.sqrt(1.0 + m[1, 1] - m[0, 0] - m[2, 2]) * 2.0
        q = np.array([(m[0, 1] + m[1, 0]) / s, 0.25 * s,
                      (m[1, 2] + m[2, 1]) / s, (m[0, 2] - m[2, 0]) / s])
    else:
        s = np.sqrt(1.0 + m[2, 2] - m[0, 0] - m[1, 1]) * 2.0
        q = np.array([(m[0, 2] + m[2, 0]) / s, (m[1, 2] + m[2, 1]) / s,
                      0.25 * s, (m[1, 0] - m[0, 1]) / s])
    return quat_normalize(q)


def skew(v):
    x, y, z = np.moveaxis(np.asarray(v, dtype=float), -1, 0)
    zero = np.zeros_like(x)
    return np.stack([zero, -z, y, z, zero, -x, -y, x, zero], axis=-1).reshape(
        np.shape(v)[:-1] + (3, 3))


def _se3_v_matrix(phi):
    """SE(3) V matrix as the phi_1 block of expm (geometry.py:149-161, sigma = 0)."""
    blk = np.zeros((6, 6))
    blk[:3, :3] = 0.0 * np.eye(3) + skew(np.asarray(phi, dtype=float))
    blk[:3, 3:] = np.eye(3)
    return scipy.linalg.expm(blk)[:3, 3:]


def _frozen(a, shape):
    out = np.array(a, dtype=float).reshape(shape)
    out.flags.writeable = False
    return out


def _renormalized(q):
    q = np.asarray(q, dtype=float)
    norm = np.linalg.norm(q)
    return q / norm if abs(norm - 1.0) > 1e-12 else q


@dataclass(frozen=True, eq=False)
class Pose:
    """World-from-camera rigid transform (geometry.py:183-242)."""

    q: np.ndarray = field(default_factory=lambda: np.array([0.0, 0.0, 0.0, 1.0]))
    t: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        object.__setattr__(self, "q", _frozen(_renormalized(self.q), (4,)))
        object.__setattr__(self, "t", _frozen(self.t, (3,)))

    @staticmethod
    def identity() -> "Pose":
        return Pose()

    @staticmethod
    def exp(xi) -> "Pose":
        xi = np.asarray(xi, dtype=float).reshape(6)
        return Pose(rotvec_to_quat(xi[3:]), _se3_v_matrix(xi[3:]) @ xi[:3])

    def __mul__(self, other: "Pose") -> "Pose":
        return Pose(quat_mul(self.q, other.q), quat_rotate(self.q, other.t) + self.t)

    def inverse(self) -> "Pose":
        qc = quat_conj(self.q)
        return Pose(qc, -quat_rotate(qc, self.t))

    def act(self, points):
        return quat_rotate(self.q, np.asarray(points, dtype=float)) + self.t

    def rotation_matrix(self):
        return quat_to_matrix(self.q)

    def as_array(self):
        return np.concatenate([self.t, self.q])

    @staticmethod
    def from_array(a) -> "Pose":
        a = np.asarray(a, dtype=float).reshape(7)
        return Pose(a[3:], a[:3])

    def __repr__(self):
        return f"Pose(t={self.t.tolist()}, q={self.q.tolist()})"


@dataclass(frozen=True)
class Intrinsics:
    """Pinhole intrinsics (geometry.py:350-362)."""

    fx: float
    fy: float
    cx: float
    cy: float

    def __post_init__(self):
        if not (self.fx > 0 and self.fy > 0):
            raise ValueError(f"focal lengths must be positive, got fx={self.fx} fy={self.fy}")

    def as_array(self):
        return np.array([self.fx, self.fy, self.cx, self.cy])


def square_grids(centers, patch_size: int = DEFAULT_PATCH_SIZE):
    """square_grid of many keypoints at once (n, p*p, 2); the same additions,
    so bit-identical to stacking square_grid per keypoint."""
    centers = np.asarray(centers, dtype=float).reshape(-1, 2)
    offs = np.arange(patch_size) - (patch_size - 1) / 2.0
    gy, gx = np.meshgrid(offs, offs, indexing="ij")
    return np.stack([gx.ravel()[None, :] + centers[:, 0:1], gy.ravel()[None, :] + centers[:, 1:2]],
                    axis=-1)


def square_grid(center, patch_size: int = DEFAULT_PATCH_SIZE):
    """Row-major p x p unit grid around a keypoint (geometry.py:398-407)."""
    center = np.asarray(center, dtype=float).reshape(2)
    offs = np.arange(patch_size) - (patch_size - 1) / 2.0
    gy, gx = np.meshgrid(offs, offs, indexing="ij")
    return np.stack([gx.ravel() + center[0], gy.ravel() + center[1]], axis=-1)


def pinhole_rays(pixels, intr: Intrinsics):
    """Unit-depth rays (geometry.py:386-391); computed on the device for BA."""
    pixels = np.asarray(pixels, dtype=float)
    x = (pixels[..., 0] - intr.cx) / intr.fx
    y = (pixels[..., 1] - intr.cy) / intr.fy
    return np.stack([x, y, np.ones_like(x)], axis=-1)


@dataclass(frozen=True, eq=False)
class Patch:
    """p x p pixel grid with one inverse depth (geometry.py:410-461)."""

    frame_id: int
    grid: np.ndarray
    inverse_depth: float
    landmark_id: int | None = None

    def __post_init__(self):
        grid = np.array(self.grid, dtype=float).reshape(-1, 2)
        p = int(round(np.sqrt(grid.shape[0])))
        if p * p != grid.shape[0]:
            raise ValueError(f"patch grid must have p*p cells, got {grid.shape[0]}")
        if not np.allclose(grid, square_grid(grid.mean(axis=0), p), atol=1e-6):
            raise ValueError("patch grid is not an axis-aligned unit-spacing square")
        if not self.inverse_depth > 0:
            raise NonPositiveDepth(f"patch inverse depth must be positive, got {self.inverse_depth}")
        grid.flags.writeable = False
        object.__setattr__(self, "grid", grid)
        object.__setattr__(self, "inverse_depth", float(self.inverse_depth))

    @staticmethod
    def square(frame_id, center, inverse_depth, patch_size=DEFAULT_PATCH_SIZE,
               landmark_id=None) -> "Patch":
        return Patch(frame_id, square_grid(center, patch_size), inverse_depth, landmark_id)

    @property
    def size(self) -> int:
        return int(round(np.sqrt(self.grid.shape[0])))

    @property
    def center(self):
        return self.grid.mean(axis=0)

    def with_inverse_depth(self, d: float) -> "Patch":
        if not d > 0:
            raise NonPositiveDepth(f"patch inverse depth must be positive, got {d}")
        out = object.__new__(Patch)
        object.__setattr__(out, "frame_id", self.frame_id)
        object.__setattr__(out, "grid", self.grid)
        object.__setattr__(out, "inverse_depth", float(d))
        object.__setattr__(out, "landmark_id", self.landmark_id)
        return out


# ---------------------------------------------------------------------------
# K2 on the device


def _as_device(x, torch):
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=torch.float64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device="cuda")


def reproject_grid(rays, inverse_depth, rot_i, t_i, rot_j, t_j, intr, jacobians=False):
    """Drop-in for patchslam.geometry.reproject_grid (geometry.py:478-529) on the B200.

    Same shapes and semantics: pixels (E,m,2), valid (E,m) and, with
    ``jacobians``, J_pose (E,m,2,6) w.r.t. the source-pose tangent (the target
    pose's is the negation) and J_depth (E,m,2).  numpy in -> numpy out;
    CUDA tensors in -> CUDA tensors out.
    """
    import torch
    lib = _lib.lib()
    as_numpy = not isinstance(rays, torch.Tensor)
    r = _as_device(rays, torch)
    e = r.shape[0]
    m = r.shape[1] if r.dim() == 3 else 0
    dev = [r, _as_device(inverse_depth, torch).reshape(-1), _as_device(rot_i, torch),
           _as_device(t_i, torch), _as_device(rot_j, torch), _as_device(t_j, torch)]
    pix = torch.empty((e, m, 2), dtype=torch.float64, device="cuda")
    valid = torch.empty((e, m), dtype=torch.uint8, device="cuda")
    jp = torch.empty((e, m, 2, 6), dtype=torch.float64, device="cuda") if jacobians else None
    jd = torch.empty((e, m, 2), dtype=torch.float64, device="cuda") if jacobians else None
    iv = intr.as_array() if hasattr(intr, "as_array") else np.asarray(intr, dtype=float)
    intr4 = (C.c_double * 4)(*[float(v) for v in iv])
    if e and m:
        _lib.check(lib.dpv_reproject_grid(*[_lib.ptr(x) for x in dev], intr4, e, m, _lib.ptr(pix),
                                          _lib.ptr(valid), _lib.ptr(jp), _lib.ptr(jd),
                                          _lib.stream_ptr()), "reproject_grid")
    out = [pix, valid.bool()] + ([jp, jd] if jacobians else [])
    if as_numpy:
        out = [o.cpu().numpy() for o in out]
    return tuple(out)


def reproject_patch(patch: Patch, pose_i: Pose, pose_j: Pose, intr: Intrinsics, strict=False):
    """One patch through the device kernel (geometry.py:532-556)."""
    rays = pinhole_rays(patch.grid, intr)[None]
    pix, valid = reproject_grid(rays, np.array([patch.inverse_depth]),
                                pose_i.rotation_matrix()[None], pose_i.t[None],
                                pose_j.rotation_matrix()[None], pose_j.t[None], intr)
    if strict and not valid.all():
        raise BehindCamera(f"{int((~valid).sum())} patch cell(s) reprojected behind the camera")
    return pix[0], valid[0]
