"""Synthetic scenes and the flow oracle: the inputs of the hot path.

Restates the reference's input generator (pkg/src/patchslam/synthetic.py:
``SceneSpec`` 34-54, ``generate`` 179-215, ``fill_flow`` 222-287) and the
perturbation helper of its tests (pkg/tests/conftest.py:28-32) so that the
B200 path runs on *bit-identical* inputs without importing the reference
(``tests/golden/synth_hashes.json`` pins the SHA-256 of every array against
the reference at configs 1-3).  It draws the same random numbers in the same
order and evaluates the same floating-point expressions, vectorised over
frames/edges and writing straight into the structure-of-arrays graph.

This module prepares inputs; it is not the hot path.  The ground-truth
reprojection used for flow targets is the reference's numpy expression
(kept private as ``_np_reproject_exact``) because bit-identical targets are
the point; the BA/correlation kernels never call it.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import ctypes as C

import numpy as np

from .errors import InfeasibleVisibility
from .geometry import Intrinsics, Pose, matrix_to_quat, pinhole_rays, quat_to_matrix, square_grids
from .graph import LOOP, ODOMETRY, PatchGraph

DEFAULT_INTRINSICS = Intrinsics(320.0, 320.0, 256.0, 192.0)   # synthetic.py:28
DEFAULT_IMAGE_SIZE = (512, 384)                               # synthetic.py:29
TRAJECTORY_KINDS = ("line", "circle", "square-loop", "random-walk-with-revisit")
_CHUNK = 1 << 18


@dataclass(frozen=True)
class SceneSpec:
    kind: str = "circle"
    n_frames: int = 50
    seed: int = 0
    n_landmarks: int = 4000
    extent: float = 10.0
    frame_dt: float = 0.1
    shell: tuple = (1.0, 20.0)
    image_size: tuple = DEFAULT_IMAGE_SIZE
    intrinsics: Intrinsics = field(default_factory=lambda: DEFAULT_INTRINSICS)
    overshoot: float = 0.15
    look: str = "forward"

    def __post_init__(self):
        if self.kind not in TRAJECTORY_KINDS:
            raise ValueError(f"unknown trajectory kind {self.kind!r}")
        if self.look not in ("forward", "inward"):
            raise ValueError(f"unknown look mode {self.look!r}")
        if self.n_frames < 1:
            raise ValueError("need at least one frame")


@dataclass
class SyntheticScene:
    spec: SceneSpec
    gt_poses: list
    landmarks: np.ndarray
    intrinsics: Intrinsics

    def camera_points(self, frame_id, ids=None):
        pts = self.landmarks if ids is None else self.landmarks[ids]
        return self.gt_poses[frame_id].inverse().act(pts)

    def visible_landmarks(self, frame_id, margin=2.0):
        """synthetic.py:68-79."""
        cam = self.camera_points(frame_id)
        pix, valid = _project(cam, self.intrinsics)
        w, h = self.spec.image_size
        ok = (valid & (cam[:, 2] > 0.5)
              & (pix[:, 0] >= margin) & (pix[:, 0] <= w - 1 - margin)
              & (pix[:, 1] >= margin) & (pix[:, 1] <= h - 1 - margin))
        return np.nonzero(ok)[0]


@dataclass(frozen=True)
class OracleConfig:
    pixel_noise_sigma: float = 0.0
    outlier_fraction: float = 0.0
    outlier_magnitude: float = 40.0
    low_confidence: float = 0.05

    def __post_init__(self):
        if not 0.0 <= self.outlier_fraction < 1.0:
            raise ValueError("outlier fraction must lie in [0, 1)")


def _project(points, intr):
    """project_array (geometry.py:468-475)."""
    z = points[..., 2]
    valid = z > 1e-8
    zs = np.where(valid, z, 1.0)
    u = intr.fx * points[..., 0] / zs + intr.cx
    v = intr.fy * points[..., 1] / zs + intr.cy
    return np.stack([u, v], axis=-1), valid


def _np_reproject_exact(rays, inv_depth, rot_i, t_i, rot_j, t_j, intr):
    """The reference's numpy reprojection expression, for bit-identical targets."""
    x_cam = rays / inv_depth[:, None, None]
    x_world = x_cam @ rot_i.swapaxes(-1, -2) + t_i[:, None, :]
    x_tgt = (x_world - t_j[:, None, :]) @ rot_j
    z = x_tgt[..., 2]
    valid = z > 1e-8
    zs = np.where(valid, z, 1.0)
    pix = np.stack([intr.fx * x_tgt[..., 0] / zs + intr.cx,
                    intr.fy * x_tgt[..., 1] / zs + intr.cy], axis=-1)
    return pix, valid


# ---------------------------------------------------------------------------
# trajectories (synthetic.py:98-172)


def _look_rotation(forward):
    f = forward / np.linalg.norm(forward)
    up = np.array([0.0, 1.0, 0.0])
    if abs(f @ up) > 0.99:
        up = np.array([0.0, 0.0, 1.0])
    right = np.cross(f, up)
    right /= np.linalg.norm(right)
    down = np.cross(f, right)
    return np.stack([right, down, f], axis=1)


def _positions(spec, rng):
    n = spec.n_frames
    if spec.kind == "line":
        s = np.linspace(0.0, spec.extent, n)
        return np.stack([s, np.zeros(n), np.zeros(n)], axis=1)
    if spec.kind == "circle":
        r = spec.extent / 2.0
        ang = np.linspace(0.0, 2 * np.pi * (1 + spec.overshoot), n)
        return np.stack([r * np.cos(ang), np.zeros(n), r * np.sin(ang)], axis=1)
    if spec.kind == "square-loop":
        side = spec.extent
        s = np.linspace(0.0, 4.0 * side * (1 + spec.overshoot), n) % (4.0 * side)
        pos = np.zeros((n, 3))
        for i, dist in enumerate(s):
            leg, rem = int(dist // side) % 4, dist % side
            pos[i] = [(rem, 0.0, 0.0), (side, 0.0, rem), (side - rem, 0.0, side),
                      (0.0, 0.0, side - rem)][leg]
        return pos
    step = spec.extent / max(n - 1, 1)
    heading = rng.uniform(0, 2 * np.pi)
    pos = [np.zeros(3)]
    n_out = max(int(0.7 * n), 1)
    for _ in range(n_out - 1):
        heading += rng.normal(0.0, 0.25)
        pos.append(pos[-1] + step * np.array([np.cos(heading), 0.0, np.sin(heading)]))
    far = pos[-1]
    for i in range(n - n_out):
        a = (i + 1) / max(n - n_out, 1)
        pos.append((1 - a) * far)
    return np.stack(pos[:n])


def _gt_poses(spec, rng):
    pos = _positions(spec, rng)
    centroid = pos.mean(axis=0)
    out = []
    for i in range(len(pos)):
        if spec.look == "inward":
            fwd = centroid - pos[i]
        else:
            fwd = pos[min(len(pos) - 1, i + 1)] - pos[max(0, i - 1)]
        if np.linalg.norm(fwd) < 1e-12:
            fwd = np.array([1.0, 0.0, 0.0])
        out.append(Pose(matrix_to_quat(_look_rotation(fwd)), pos[i]))
    return out


def _landmarks(spec, pos, rng):
    lo, hi = spec.shell
    anchor = pos[rng.integers(0, len(pos), size=spec.n_landmarks)]
    direction = rng.normal(size=(spec.n_landmarks, 3))
    direction /= np.linalg.norm(direction, axis=1, keepdims=True)
    radius = rng.uniform(lo, hi, size=spec.n_landmarks)
    return anchor + direction * radius[:, None]


# ---------------------------------------------------------------------------
# scene + graph (synthetic.py:179-215)


def generate(spec: SceneSpec, patches_per_frame: int = 96, odometry_radius: int = 13,
             patch_size: int = 3, initial_targets: bool = True):
    """Ground-truth scene + patch graph at the truth (bit-identical to the reference).

    ``initial_targets=False`` skips the (later overwritten) initial-reprojection
    targets of the odometry edges (graph.py:159-164) and leaves them at 0.
    """
    rng = np.random.default_rng(spec.seed)
    gt = _gt_poses(spec, rng)
    lms = _landmarks(spec, np.stack([p.t for p in gt]), rng)
    scene = SyntheticScene(spec, gt, lms, spec.intrinsics)
    graph = PatchGraph(spec.intrinsics, patch_size)
    margin = (patch_size - 1) / 2.0 + 0.5
    m = patch_size * patch_size
    counts = np.zeros(spec.n_frames, dtype=np.int64)
    vis_all = _visible_all(scene, margin) if _device_available() else None
    for fid in range(spec.n_frames):
        vis = vis_all[fid] if vis_all is not None else scene.visible_landmarks(fid, margin)
        if len(vis) < patches_per_frame:
            raise InfeasibleVisibility(
                f"frame {fid} sees {len(vis)} landmarks < {patches_per_frame};"
                " increase n_landmarks or shrink the shell")
        chosen = rng.choice(vis, size=patches_per_frame, replace=False)
        cam = scene.camera_points(fid, chosen)
        pix, _ = _project(cam, spec.intrinsics)
        grids = square_grids(pix, patch_size)
        depths = 1.0 / cam[:, 2]
        graph.add_frame_arrays(gt[fid].q, gt[fid].t, fid * spec.frame_dt, grids, depths,
                               chosen.astype(np.int64))
        counts[fid] = patches_per_frame
        if odometry_radius > 0:
            tri = PatchGraph.odometry_triples(fid, odometry_radius, counts)
            if len(tri):
                graph.add_edge_arrays(tri[:, 0], tri[:, 1], tri[:, 2], np.zeros((len(tri), m, 2)),
                                      np.ones((len(tri), 2)), ODOMETRY)
    if initial_targets and graph.n_edges:
        reproject_targets(graph, np.arange(graph.n_edges))
    return scene, graph


def reproject_targets(graph, idx, device=None):
    """Initial targets of edges idx = the current reprojection of their source
    patch grids (graph.py:152-164), bit-identical to the reference's numpy
    expression: on the device (dpv_reproject_exact) when CUDA is available,
    else the host restatement."""
    idx = np.asarray(idx, dtype=np.int64)
    if len(idx) == 0:
        return
    if device is None:
        device = _device_available()
    if not device:
        return _reproject_targets(graph, idx, graph._q.view, graph._t.view, graph._depth.view)
    import torch

    from . import _lib
    g = graph.dpv_view()
    mir = graph.device()
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")   # noqa: E731
    rot_d = T(quat_to_matrix(graph._q.view).reshape(-1, 9))
    sel_d = T(idx)
    pix = torch.empty((len(idx), graph.patch_size ** 2, 2), dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().dpv_reproject_exact(C.byref(g), _lib.ptr(rot_d), _lib.ptr(mir["t"]),
                                              _lib.ptr(mir["patch_depth"]), _lib.ptr(sel_d),
                                              len(idx), _lib.ptr(pix), _lib.stream_ptr()),
               "reproject_exact")
    mir["edge_target"][sel_d] = pix
    graph._tgt.view[idx] = pix.cpu().numpy()


def _reproject_targets(graph, idx, q, t, patch_depth):
    """Initial targets = current reprojection (graph.py:152-164), exact numpy."""
    rot = quat_to_matrix(q)
    off = graph.patch_offset()
    for lo in range(0, len(idx), _CHUNK):
        sel = idx[lo:lo + _CHUNK]
        src = graph._src.view[sel].astype(np.int64)
        dst = graph._dst.view[sel].astype(np.int64)
        gid = off[src] + graph._pat.view[sel]
        rays = pinhole_rays(graph._grid.view[gid], graph.intrinsics)
        pix, _ = _np_reproject_exact(rays, patch_depth[gid], rot[src], t[src], rot[dst], t[dst],
                                     graph.intrinsics)
        graph._tgt.view[sel] = pix
    graph._edge_clean = min(graph._edge_clean, int(idx.min()) if len(idx) else graph._edge_clean)


def add_loop_edges(graph, n_poses: int, patches: int, seed: int = 0):
    """Long-range LOOP edges, the bench-ba recipe (cli.py:103-110)."""
    rng = np.random.default_rng(seed)
    tri = []
    for _ in range(max(2, n_poses // 60)):
        old = int(rng.integers(0, max(1, n_poses // 4)))
        recent = int(rng.integers(3 * n_poses // 4, n_poses))
        tri.extend((old, k, recent) for k in range(min(patches, 32)))
    tri = np.asarray(tri, dtype=np.int64)
    m = graph.patch_size ** 2
    return graph.add_edge_arrays(tri[:, 0], tri[:, 1], tri[:, 2], np.zeros((len(tri), m, 2)),
                                 np.ones((len(tri), 2)), LOOP)


# ---------------------------------------------------------------------------
# flow oracle (synthetic.py:222-300)


def _visible_all(scene, margin):
    """visible_landmarks (synthetic.py:68-79) of every frame in one device
    pass (dpv_visible_landmarks, bit-identical tests); per frame the sorted
    landmark ids, as np.nonzero returns them."""
    import torch

    from . import _lib
    invs = [p.inverse() for p in scene.gt_poses]
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")  # noqa
    inv_q, inv_t = T(np.stack([p.q for p in invs])), T(np.stack([p.t for p in invs]))
    lms = T(scene.landmarks)
    F, L = len(invs), len(scene.landmarks)
    w, h = scene.spec.image_size
    intr = np.ascontiguousarray(scene.intrinsics.as_array(), dtype=np.float64)
    flags = torch.empty((F, L), dtype=torch.uint8, device="cuda")
    _lib.check(_lib.lib().dpv_visible_landmarks(
        F, L, _lib.ptr(inv_q), _lib.ptr(inv_t), _lib.ptr(lms), intr.ctypes.data_as(C.c_void_p),
        float(margin), float(w - 1 - margin), float(h - 1 - margin), _lib.ptr(flags),
        _lib.stream_ptr()), "visible_landmarks")
    counts = flags.sum(dim=1, dtype=torch.int64).cpu().numpy()
    ids = torch.nonzero(flags)[:, 1].cpu().numpy()
    return np.split(ids, np.cumsum(counts)[:-1])


def _device_available() -> bool:
    try:
        import torch
        return bool(torch.cuda.is_available())
    except Exception:       # torch missing: host generator
        return False


def _draws(rng, config: OracleConfig, n: int):
    """The flow oracle's random draws, in the reference's order
    (synthetic.py:263-268)."""
    shift = (rng.normal(0.0, config.pixel_noise_sigma, size=(n, 2))
             if config.pixel_noise_sigma > 0 else np.zeros((n, 2)))
    outlier = rng.random(n) < config.outlier_fraction
    ang = rng.uniform(0, 2 * np.pi, size=n)
    gross = config.outlier_magnitude * np.stack([np.cos(ang), np.sin(ang)], axis=1)
    return shift, outlier, gross


def _fill_flow_device(graph, scene, config, idx, rng):
    """fill_flow with the reprojection / observability / target assembly on
    the device (dpv_fill_flow, csrc/synth.cu; bit-identical to the host
    expressions) and the draws from the host generator."""
    import torch

    from . import _lib
    n = len(idx)
    shift, outlier, gross = _draws(rng, config, n)
    rot = quat_to_matrix(np.stack([p.q for p in scene.gt_poses])).reshape(-1, 9)
    gt_t = np.stack([p.t for p in scene.gt_poses])
    g = graph.dpv_view()
    mir = graph.device()
    dev = "cuda"
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)   # noqa: E731
    rot_d, t_d, lms_d = T(rot), T(gt_t), T(scene.landmarks)
    plm_d = T(graph._lm.view.astype(np.int64))
    sel_d = T(idx.astype(np.int64))
    shift_d, out_d, gross_d = T(shift), T(outlier.astype(np.uint8)), T(gross)
    m = graph.patch_size ** 2
    target = torch.empty((n, m, 2), dtype=torch.float64, device=dev)
    conf = torch.empty((n, 2), dtype=torch.float64, device=dev)
    w, h = scene.spec.image_size
    _lib.check(_lib.lib().dpv_fill_flow(
        C.byref(g), _lib.ptr(rot_d), _lib.ptr(t_d), _lib.ptr(lms_d), _lib.ptr(plm_d),
        _lib.ptr(sel_d), n, _lib.ptr(shift_d), _lib.ptr(out_d), _lib.ptr(gross_d),
        float(config.low_confidence), float(w), float(h), _lib.ptr(target), _lib.ptr(conf),
        _lib.stream_ptr()), "fill_flow")
    # the mirror stays current (scatter on the device), the host truth by D2H
    mir["edge_target"][sel_d] = target
    mir["edge_conf"][sel_d] = conf
    graph._tgt.view[idx] = target.cpu().numpy()
    graph._conf.view[idx] = conf.cpu().numpy()


def fill_flow(graph, scene, config: OracleConfig = OracleConfig(), edge_indices=None,
              seed: int = 0, device: bool | None = None) -> None:
    """Ground-truth reprojection + one Gaussian shift per edge, seeded
    outliers with low confidence, unobservable edges at confidence 0.
    ``device`` (default: when CUDA is available) runs the geometry on the
    B200 (dpv_fill_flow); the result is bit-identical either way."""
    idx = (np.arange(graph.n_edges) if edge_indices is None
           else np.asarray(list(edge_indices), dtype=np.int64))
    if len(idx) == 0:
        return
    rng = np.random.default_rng(seed)
    if device is None:
        device = _device_available()
    if device:
        return _fill_flow_device(graph, scene, config, idx, rng)
    intr = graph.intrinsics
    gt_q = np.stack([p.q for p in scene.gt_poses])
    gt_t = np.stack([p.t for p in scene.gt_poses])
    rot = quat_to_matrix(gt_q)
    off = graph.patch_offset()
    w, h = scene.spec.image_size
    slack = 0.25 * max(w, h)
    n = len(idx)
    pix_all = np.empty((n, graph.patch_size ** 2, 2))
    obs = np.empty(n, dtype=bool)
    for lo in range(0, n, _CHUNK):
        sel = idx[lo:lo + _CHUNK]
        src = graph._src.view[sel].astype(np.int64)
        dst = graph._dst.view[sel].astype(np.int64)
        gid = off[src] + graph._pat.view[sel]
        rays = pinhole_rays(graph._grid.view[gid], intr)
        lm = graph._lm.view[gid]
        cam_z = np.einsum("eb,eb->e", rot[src][:, :, 2], scene.landmarks[lm] - gt_t[src])
        pix, valid = _np_reproject_exact(rays, 1.0 / cam_z, rot[src], gt_t[src], rot[dst],
                                         gt_t[dst], intr)
        obs[lo:lo + len(sel)] = (
            valid.all(axis=1)
            & (pix[..., 0] > -slack).all(axis=1) & (pix[..., 0] < w + slack).all(axis=1)
            & (pix[..., 1] > -slack).all(axis=1) & (pix[..., 1] < h + slack).all(axis=1))
        pix_all[lo:lo + len(sel)] = pix
    shift, outlier, gross = _draws(rng, config, n)
    target = pix_all + shift[:, None, :]
    bad = outlier & obs
    target[bad] = target[bad] + gross[bad][:, None, :]
    conf = np.ones((n, 2))
    conf[bad] = config.low_confidence
    conf[~obs] = 0.0
    graph._tgt.view[idx] = target
    graph._conf.view[idx] = conf
    graph._edge_clean = min(graph._edge_clean, int(idx.min()))


def make_flow_oracle(scene, config: OracleConfig, seed: int = 0):
    """Stateful oracle (graph, edge_indices) -> None (synthetic.py:290-300)."""
    counter = {"n": 0}

    def oracle(graph, edge_indices):
        fill_flow(graph, scene, config, edge_indices, seed=seed * 100003 + counter["n"])
        counter["n"] += 1
    return oracle


def perturb_poses(graph, sigma: float, seed: int, first: int = 1, frame: str = "world") -> None:
    """Left-multiply Pose.exp(N(0, sigma)) onto every frame from ``first``
    (pkg/tests/conftest.py:28-32).  ``frame="camera"`` right-multiplies the
    same draws instead (a perturbation about each camera centre), which keeps
    the perturbation local on a scene far from the world origin (cfg4: a
    world-frame 0.02 rad rotation moves a camera 440 m out by metres)."""
    if frame not in ("world", "camera"):
        raise ValueError(f"unknown perturbation frame {frame!r}")
    rng = np.random.default_rng(seed)
    for f in range(first, graph.n_frames):
        cur = Pose(graph._q.view[f], graph._t.view[f])
        noise = Pose.exp(rng.normal(0, sigma, 6))
        p = noise * cur if frame == "world" else cur * noise
        graph._q.view[f] = p.q
        graph._t.view[f] = p.t
    graph._pose_ver += 1


# ---------------------------------------------------------------------------
# benchmark configurations


CONFIGS = {
    # name: (SceneSpec kwargs, loop span or 0, free range fn)
    "cfg1": dict(spec=dict(kind="circle", n_frames=16, seed=0, n_landmarks=3000, look="inward",
                           image_size=(640, 480),
                           intrinsics=Intrinsics(320.0, 320.0, 320.0, 240.0)),
                 loops=0, free=lambda n: (1, 15)),
    "cfg2": dict(spec=dict(kind="circle", n_frames=40, seed=0, n_landmarks=6000, look="inward",
                           image_size=(752, 480),
                           intrinsics=Intrinsics(458.654, 457.296, 367.215, 248.375)),
                 loops=0, free=lambda n: (n - 22, n - 1)),
    "mid": dict(spec=dict(kind="circle", n_frames=120, seed=0, n_landmarks=8640, look="inward",
                          image_size=(640, 480), intrinsics=Intrinsics(320.0, 320.0, 320.0, 240.0),
                          extent=15.0),
                loops=120, free=lambda n: (1, n - 1)),
    "cfg3": dict(spec=dict(kind="circle", n_frames=2000, seed=0, n_landmarks=144000,
                           look="inward", image_size=(640, 480),
                           intrinsics=Intrinsics(320.0, 320.0, 320.0, 240.0), extent=250.0),
                 loops=2000, free=lambda n: (1, n - 1)),
    # TartanAir-shape sequences: 64 independent cfg2-style
    # windows, sequence s uses scene seed s (make_config(..., seed=s))
    "cfg5": dict(spec=dict(kind="circle", n_frames=40, seed=0, n_landmarks=6000, look="inward",
                           image_size=(640, 480),
                           intrinsics=Intrinsics(320.0, 320.0, 320.0, 240.0)),
                 loops=0, free=lambda n: (n - 22, n - 1)),
    # KITTI shape: forward-looking square loop, 4500 frames
    "cfg4": dict(spec=dict(kind="square-loop", n_frames=4500, seed=0, n_landmarks=324000,
                           look="forward", image_size=(1226, 370),
                           intrinsics=Intrinsics(718.856, 718.856, 607.193, 185.216),
                           extent=440.0),
                 loops=4500, free=lambda n: (1, n - 1), perturb="camera"),
}

DESCRIPTIONS = {
    "cfg1": "16-frame local window (circle, 96 patches/frame, radius 13)",
    "cfg2": "EuRoC-shape 22-frame window (752x480, 96 patches/frame, radius 13)",
    "mid": "120-frame loop graph (circle, 96 patches/frame, radius 13, loop edges)",
    "cfg3": "2000-frame global loop-closure BA (circle, 96 patches/frame, radius 13, "
            "33x32 loop edges)",
    "cfg5": "TartanAir-shape sequences (640x480), one 22-frame window step each "
            "(96 patches/frame, radius 13), 8 per GPU as replicas",
    "cfg4": "KITTI-shape 4500-frame global BA (1226x370, forward square loop, 96 patches/frame, "
            "radius 13, 75x32 loop edges)",
}


def make_config(name: str, initial_targets: bool = False, seed: int | None = None):
    """Build a benchmark configuration: (scene, graph, free_range).

    Recipe: generate(96 patches, radius 13) -> bench-ba LOOP
    edges -> fill_flow(sigma=0.3, seed=1) -> perturb_poses(0.02, seed=11).
    ``seed`` overrides the scene seed (cfg5: sequence s has seed s)."""
    cfg = CONFIGS[name]
    kw = dict(cfg["spec"])
    if seed is not None:
        kw["seed"] = int(seed)
    spec = SceneSpec(**kw)
    scene, graph = generate(spec, 96, 13, initial_targets=initial_targets)
    if cfg["loops"]:
        add_loop_edges(graph, cfg["loops"], 96, seed=0)
    fill_flow(graph, scene, OracleConfig(pixel_noise_sigma=0.3), seed=1)
    perturb_poses(graph, 0.02, seed=11, frame=cfg.get("perturb", "world"))
    return scene, graph, cfg["free"](spec.n_frames)
