"""Sim(3) pose-graph optimisation on the B200 (reference posegraph.py:121-196).

The host side keeps the reference's interface -- ``PoseGraphProblem``,
``PGOReport``, ``objective``, ``residual_smooth``, ``residual_loop``,
``residual_and_jacobian``, ``optimize`` -- and binds the C-ABI of
``csrc/pgo.cu`` (``dpv_pgo_linearize`` / ``dpv_pgo_optimize``): residuals,
Jacobians, the dense normal equations, the damped solve (the K4c Cholesky
engine) and the LM candidate evaluation all run on the device; the host only
packs the similarities into (n, 8) float64 arrays [t | q | s] and reads back
one report.  Nodes may be this module's ``Similarity`` or any value type with
the reference's (q, t, s) fields (the drop-in path hands in
``patchslam.geometry.Similarity``); results come back as the same type.
There is no CPU fallback: without the library a ``NativeUnavailable`` is
raised.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .geometry import quat_conj, quat_mul, quat_rotate

LM_LAMBDA_INIT = 1e-4            # posegraph.py:40-43
LM_LAMBDA_GROW = 10.0
LM_LAMBDA_SHRINK = 0.5
LM_LAMBDA_MAX = 1e10


def _renormalized(q):
    """Renormalise only on drift (reference geometry.py:174-180)."""
    q = np.asarray(q, dtype=float)
    n = np.linalg.norm(q)
    return q / n if abs(n - 1.0) > 1e-12 else q


@dataclass(frozen=True, eq=False)
class Similarity:
    """x -> s R x + t (reference geometry.py:246-300): host value type."""

    q: np.ndarray = field(default_factory=lambda: np.array([0.0, 0.0, 0.0, 1.0]))
    t: np.ndarray = field(default_factory=lambda: np.zeros(3))
    s: float = 1.0

    def __post_init__(self):
        if not self.s > 0:
            raise ValueError(f"similarity scale must be positive, got {self.s}")
        object.__setattr__(self, "q", _renormalized(self.q).reshape(4))
        object.__setattr__(self, "t", np.array(self.t, dtype=float).reshape(3))
        object.__setattr__(self, "s", float(self.s))

    @staticmethod
    def identity():
        return Similarity()

    @staticmethod
    def from_pose(pose, scale: float = 1.0):
        return Similarity(pose.q, pose.t, scale)

    def __mul__(self, other):
        return type(self)(quat_mul(self.q, other.q), self.s * quat_rotate(self.q, other.t) + self.t,
                          self.s * other.s)

    def inverse(self):
        qc = quat_conj(self.q)
        return type(self)(qc, -quat_rotate(qc, self.t) / self.s, 1.0 / self.s)


@dataclass
class PoseGraphProblem:
    """Reference posegraph.py:46-72 (nodes, odometry per (i, i+1), loops)."""

    nodes: list
    odometry: list
    loops: list
    damping: float = LM_LAMBDA_INIT

    def __post_init__(self):
        n = len(self.nodes)
        if len(self.odometry) != n - 1:
            raise ValueError(
                f"{n} nodes need {n - 1} odometry constraints, got {len(self.odometry)}")
        for j, k, _ in self.loops:
            if not (0 <= j < n and 0 <= k < n) or j == k:
                raise ValueError(f"loop ({j}, {k}) references invalid nodes")

    @staticmethod
    def from_poses(poses, loops=()):
        nodes = [Similarity.from_pose(p) for p in poses]
        odometry = [nodes[i].inverse() * nodes[i + 1] for i in range(len(nodes) - 1)]
        return PoseGraphProblem(nodes, odometry, list(loops))


@dataclass
class PGOReport:
    """Reference posegraph.py:75-82."""

    iterations: int
    initial_objective: float
    final_objective: float
    max_residual_norm: float
    scale_corrections: np.ndarray
    converged: bool = False


# ---------------------------------------------------------------------------
# packing


def _pack(sims) -> np.ndarray:
    out = np.empty((len(sims), 8))
    for i, s in enumerate(sims):
        out[i, 0:3] = s.t
        out[i, 3:7] = s.q
        out[i, 7] = s.s
    return out


def _constraints(problem):
    """(a, b, M) with r = log(M S_a^-1 S_b): odometry (i, i+1, odo_i^-1)
    first, then the loops (posegraph.py:91-96)."""
    cons = [(i, i + 1, problem.odometry[i].inverse()) for i in range(len(problem.nodes) - 1)]
    cons.extend((j, k, d) for j, k, d in problem.loops)
    return cons


class _Device:
    """The problem's arrays on the device (torch tensors own the memory)."""

    def __init__(self, nodes, cons):
        import torch
        self.torch = torch
        self.n = len(nodes)
        self.C = len(cons)
        self.nodes = torch.as_tensor(_pack(nodes), device="cuda")
        self.ca_h = np.ascontiguousarray([c[0] for c in cons], dtype=np.int32)
        self.cb_h = np.ascontiguousarray([c[1] for c in cons], dtype=np.int32)
        self.ca = torch.as_tensor(self.ca_h, device="cuda")
        self.cb = torch.as_tensor(self.cb_h, device="cuda")
        self.cm = torch.as_tensor(_pack([c[2] for c in cons]).reshape(-1, 8), device="cuda")

    def linearize(self, jacobians: bool):
        torch = self.torch
        r = torch.empty((self.C, 7), dtype=torch.float64, device="cuda")
        J = torch.empty((self.C, 7, 7), dtype=torch.float64, device="cuda") if jacobians else None
        obj = torch.empty(1, dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().dpv_pgo_linearize(
            self.n, _lib.ptr(self.nodes), self.C, _lib.ptr(self.ca), _lib.ptr(self.cb),
            _lib.ptr(self.cm), _lib.ptr(r), _lib.ptr(J) if J is not None else None, _lib.ptr(obj),
            _lib.stream_ptr()), "pgo_linearize")
        return r, J, obj


def _unpack(arr, cls):
    return [cls(row[3:7].copy(), row[0:3].copy(), float(row[7])) for row in arr]


# ---------------------------------------------------------------------------
# reference API


def objective(problem, nodes=None) -> float:
    """Sum of squared Sim(3) residuals (posegraph.py:99-105), on the device."""
    nodes = problem.nodes if nodes is None else nodes
    dev = _Device(nodes, _constraints(problem))
    _, _, obj = dev.linearize(False)
    return float(obj.item())


def residual_and_jacobian(m, s_a, s_b):
    """r = log(M S_a^-1 S_b) and d r / d (left tangent of S_b)
    (posegraph.py:108-116); the S_a derivative is its negation."""
    dev = _Device([s_a, s_b], [(0, 1, m)])
    r, J, _ = dev.linearize(True)
    return r[0].cpu().numpy(), J[0].cpu().numpy()


def residual_smooth(problem, i: int) -> np.ndarray:
    """Smoothness residual between keyframes i and i+1 (posegraph.py:85-88)."""
    dev = _Device(problem.nodes, [(i, i + 1, problem.odometry[i].inverse())])
    r, _, _ = dev.linearize(False)
    return r[0].cpu().numpy()


def residual_loop(problem, pair) -> np.ndarray:
    """Loop residual of a detected pair (j, k) (posegraph.py:91-96)."""
    for j, k, delta in problem.loops:
        if (j, k) == tuple(pair):
            dev = _Device(problem.nodes, [(j, k, delta)])
            r, _, _ = dev.linearize(False)
            return r[0].cpu().numpy()
    raise KeyError(f"no loop constraint {pair}")


def optimize(problem, max_iterations: int = 50, tolerance: float = 1e-12) -> PGOReport:
    """Levenberg-Marquardt over node tangents with node 0 held fixed
    (posegraph.py:121-196): the whole loop runs natively (dpv_pgo_optimize);
    problem.nodes and problem.damping are updated as the reference does."""
    cls = type(problem.nodes[0])
    dev = _Device(problem.nodes, _constraints(problem))
    rep = _lib.DpvPgoReport()
    code = _lib.lib().dpv_pgo_optimize(
        dev.n, _lib.ptr(dev.nodes), dev.C,
        dev.ca_h.ctypes.data_as(C.c_void_p), dev.cb_h.ctypes.data_as(C.c_void_p),
        _lib.ptr(dev.ca), _lib.ptr(dev.cb), _lib.ptr(dev.cm), int(max_iterations),
        float(tolerance), float(problem.damping), C.byref(rep), _lib.stream_ptr())
    _lib.check(code, "pgo_optimize")      # DPV_SINGULAR -> SingularSystem
    nodes = _unpack(dev.nodes.cpu().numpy(), cls)
    problem.nodes = nodes
    problem.damping = float(rep.final_damping)
    return PGOReport(int(rep.iterations), float(rep.initial_objective),
                     float(rep.final_objective), float(rep.max_residual_norm),
                     np.array([s.s for s in nodes]), bool(rep.converged))
