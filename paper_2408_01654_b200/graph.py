"""Patch graph stored as structure-of-arrays with a device mirror.

Same public surface as the reference ``patchslam.graph.PatchGraph``
(graph.py:82-258) for the hot path — ``add_frame``, ``add_edges``,
``connect_frame``, ``patch``, ``patch_rays``, ``frames``/``patches``/``edges``
views, ``active_patch_keys`` — but frames, patches and edges live in growable
numpy arrays (host truth) mirrored on the GPU as torch tensors, so a 5M-edge
graph never materialises 5M Python objects.  The views return
light objects whose attribute writes go straight into the arrays.

Global patch id = ``patch_offset[frame] + patch``: monotone in
(frame, patch), so sorting global ids reproduces the reference's sorted
``depth_keys`` (ba.py:80-83).
"""

from __future__ import annotations

import numpy as np

from .errors import InconsistentFrameId, IndexOutOfRange
from .geometry import DEFAULT_PATCH_SIZE, Intrinsics, Patch, Pose, pinhole_rays

ODOMETRY = "odometry"   # graph.py:40
LOOP = "loop"           # graph.py:41
_KIND_CODE = {ODOMETRY: 0, LOOP: 1}
_KIND_NAME = {0: ODOMETRY, 1: LOOP}


class _Grow:
    """Growable array with amortised doubling along axis 0."""

    def __init__(self, shape_tail, dtype, cap=64):
        self.a = np.zeros((cap,) + tuple(shape_tail), dtype=dtype)
        self.n = 0

    def reserve(self, need):
        if need > len(self.a):
            cap = max(need, 2 * len(self.a))
            b = np.zeros((cap,) + self.a.shape[1:], dtype=self.a.dtype)
            b[:self.n] = self.a[:self.n]
            self.a = b

    def extend(self, rows):
        rows = np.asarray(rows, dtype=self.a.dtype)
        self.reserve(self.n + len(rows))
        self.a[self.n:self.n + len(rows)] = rows
        self.n += len(rows)

    @property
    def view(self):
        return self.a[:self.n]


class FrameView:
    """Frame record view (graph.py:44-51); pose writes land in the SoA arrays."""

    __slots__ = ("_g", "frame_id")

    def __init__(self, g, fid):
        self._g = g
        self.frame_id = fid

    @property
    def pose(self) -> Pose:
        return Pose(self._g._q.view[self.frame_id], self._g._t.view[self.frame_id])

    @pose.setter
    def pose(self, p: Pose):
        self._g._q.view[self.frame_id] = p.q
        self._g._t.view[self.frame_id] = p.t
        self._g._pose_ver += 1

    @property
    def timestamp(self):
        return float(self._g._ts.view[self.frame_id])

    @property
    def patch_count(self):
        g = self._g
        return int(g._poff[self.frame_id + 1] - g._poff[self.frame_id])

    @property
    def is_keyframe(self):
        return bool(self._g._kf.view[self.frame_id])

    @property
    def has_dense_features(self):
        return bool(self._g._feat.view[self.frame_id])

    @has_dense_features.setter
    def has_dense_features(self, v):
        self._g._feat.view[self.frame_id] = bool(v)


class EdgeView:
    """Edge record view (graph.py:54-71)."""

    __slots__ = ("_g", "_i")

    def __init__(self, g, i):
        self._g = g
        self._i = i

    src_frame = property(lambda s: int(s._g._src.view[s._i]))
    src_patch = property(lambda s: int(s._g._pat.view[s._i]))
    dst_frame = property(lambda s: int(s._g._dst.view[s._i]))
    kind = property(lambda s: _KIND_NAME[int(s._g._kind.view[s._i])])

    @property
    def target(self):
        self._g._touch_edge(self._i)
        return self._g._tgt.view[self._i]

    @target.setter
    def target(self, v):
        self._g._tgt.view[self._i] = np.asarray(v, dtype=float).reshape(-1, 2)
        self._g._touch_edge(self._i)

    @property
    def confidence(self):
        self._g._touch_edge(self._i)
        return self._g._conf.view[self._i]

    @confidence.setter
    def confidence(self, v):
        v = np.asarray(v, dtype=float).reshape(2)
        if np.any(v < 0) or np.any(v > 1):
            raise ValueError(f"confidence must lie in [0, 1], got {v}")
        self._g._conf.view[self._i] = v
        self._g._touch_edge(self._i)


class EdgeList:
    def __init__(self, g):
        self._g = g

    def __len__(self):
        return self._g._src.n

    def __getitem__(self, i):
        n = len(self)
        if isinstance(i, slice):
            return [EdgeView(self._g, k) for k in range(*i.indices(n))]
        i = int(i)
        if i < 0:
            i += n
        if not 0 <= i < n:
            raise IndexError(i)
        return EdgeView(self._g, i)

    def __iter__(self):
        return (EdgeView(self._g, k) for k in range(len(self)))


class FrameList:
    def __init__(self, g):
        self._g = g

    def __len__(self):
        return self._g._q.n

    def __getitem__(self, i):
        n = len(self)
        if isinstance(i, slice):
            return [FrameView(self._g, k) for k in range(*i.indices(n))]
        i = int(i)
        if i < 0:
            i += n
        if not 0 <= i < n:
            raise IndexError(i)
        return FrameView(self._g, i)

    def __iter__(self):
        return (FrameView(self._g, k) for k in range(len(self)))


class FramePatches:
    """graph.patches[f]: list-like of Patch values; item writes update depths."""

    def __init__(self, g, fid):
        self._g = g
        self._f = fid

    def __len__(self):
        return int(self._g._poff[self._f + 1] - self._g._poff[self._f])

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self[j] for j in range(*k.indices(len(self)))]
        k = int(k)
        if k < 0:
            k += len(self)
        if not 0 <= k < len(self):
            raise IndexError(k)
        return self._g.patch(self._f, k)

    def __setitem__(self, k, patch):
        self._g._set_patch(self._f, int(k), patch)

    def __iter__(self):
        return (self[j] for j in range(len(self)))


class PatchTable:
    def __init__(self, g):
        self._g = g

    def __len__(self):
        return self._g.n_frames

    def __getitem__(self, f):
        return FramePatches(self._g, int(f))

    def __setitem__(self, f, plist):
        plist = list(plist)
        fp = FramePatches(self._g, int(f))
        if len(plist) != len(fp):
            raise ValueError("replacing a frame's patches must keep their count")
        for k, p in enumerate(plist):
            fp[k] = p

    def __iter__(self):
        return (self[f] for f in range(len(self)))


class PatchGraph:
    """Single-writer container for frames, patches and edges (graph.py:82)."""

    def __init__(self, intrinsics: Intrinsics, patch_size: int = DEFAULT_PATCH_SIZE):
        self.intrinsics = intrinsics
        self.patch_size = patch_size
        m = patch_size * patch_size
        self._q = _Grow((4,), np.float64)
        self._t = _Grow((3,), np.float64)
        self._ts = _Grow((), np.float64)
        self._kf = _Grow((), np.bool_)
        self._feat = _Grow((), np.bool_)
        self._poff = [0]
        self._grid = _Grow((m, 2), np.float64)
        self._depth = _Grow((), np.float64)
        self._lm = _Grow((), np.int64)
        self._src = _Grow((), np.int32)
        self._pat = _Grow((), np.int32)
        self._dst = _Grow((), np.int32)
        self._tgt = _Grow((m, 2), np.float64)
        self._conf = _Grow((2,), np.float64)
        self._kind = _Grow((), np.uint8)
        self._pose_ver = 0
        self._patch_ver = 0
        self._edge_clean = 0          # edges [0, _edge_clean) mirrored and unchanged
        self._mirror = None

    # -- sizes / accessors (graph.py:93-120) ----------------------------------

    @property
    def n_frames(self) -> int:
        return self._q.n

    @property
    def n_patches(self) -> int:
        return self._depth.n

    @property
    def n_edges(self) -> int:
        return self._src.n

    @property
    def frames(self):
        return FrameList(self)

    @property
    def patches(self):
        return PatchTable(self)

    @property
    def edges(self):
        return EdgeList(self)

    def patch_offset(self) -> np.ndarray:
        return np.asarray(self._poff, dtype=np.int64)

    def _gid(self, frame_id, index) -> int:
        return self._poff[frame_id] + index

    def patch(self, frame_id: int, index: int) -> Patch:
        g = self._gid(frame_id, index)
        out = object.__new__(Patch)
        object.__setattr__(out, "frame_id", int(frame_id))
        object.__setattr__(out, "grid", self._grid.view[g])
        object.__setattr__(out, "inverse_depth", float(self._depth.view[g]))
        lm = int(self._lm.view[g])
        object.__setattr__(out, "landmark_id", None if lm < 0 else lm)
        return out

    def _set_patch(self, f, k, patch):
        g = self._gid(f, k)
        self._grid.view[g] = np.asarray(patch.grid, dtype=float).reshape(-1, 2)
        self._depth.view[g] = float(patch.inverse_depth)
        self._lm.view[g] = -1 if patch.landmark_id is None else int(patch.landmark_id)
        self._patch_ver += 1

    def patch_rays(self, frame_id: int, index: int):
        return pinhole_rays(self._grid.view[self._gid(frame_id, index)], self.intrinsics)

    def camera_centers(self):
        return self._t.view.copy()

    # -- mutation (graph.py:124-176) ------------------------------------------

    def add_frame(self, pose_init: Pose, timestamp: float, patches, is_keyframe: bool = True) -> int:
        fid = self.n_frames
        patches = list(patches)
        for p in patches:
            if p.frame_id != fid:
                raise InconsistentFrameId(f"patch carries frame id {p.frame_id}, expected {fid}")
            if p.size != self.patch_size:
                raise ValueError(f"patch size {p.size} != graph patch size {self.patch_size}")
        m = self.patch_size ** 2
        grids = np.stack([p.grid for p in patches]) if patches else np.zeros((0, m, 2))
        depths = np.array([p.inverse_depth for p in patches], dtype=float)
        lms = np.array([-1 if p.landmark_id is None else p.landmark_id for p in patches],
                       dtype=np.int64)
        return self.add_frame_arrays(pose_init.q, pose_init.t, timestamp, grids, depths, lms,
                                     is_keyframe)

    def add_frame_arrays(self, q, t, timestamp, grids, depths, landmarks=None,
                         is_keyframe=True) -> int:
        """Bulk form of add_frame: patch grids (K, m, 2), inverse depths (K,)."""
        fid = self.n_frames
        self._q.extend(np.asarray(q, dtype=float).reshape(1, 4))
        self._t.extend(np.asarray(t, dtype=float).reshape(1, 3))
        self._ts.extend([float(timestamp)])
        self._kf.extend([bool(is_keyframe)])
        self._feat.extend([True])
        k = len(depths)
        self._grid.extend(np.asarray(grids, dtype=float).reshape(k, self.patch_size ** 2, 2))
        self._depth.extend(depths)
        self._lm.extend(np.full(k, -1) if landmarks is None else landmarks)
        self._poff.append(self._poff[-1] + k)
        self._pose_ver += 1
        self._patch_ver += 1
        return fid

    def _check_edge_indices(self, i, k, j):
        nf = self.n_frames
        if not (0 <= i < nf and 0 <= j < nf):
            raise IndexOutOfRange(f"edge ({i},{k},{j}) references a nonexistent frame")
        if not 0 <= k < self._poff[i + 1] - self._poff[i]:
            raise IndexOutOfRange(f"edge ({i},{k},{j}) references a nonexistent patch")

    def add_edges(self, triples, kind: str = ODOMETRY) -> list[int]:
        """Append edges (i, k, j); targets start at the current reprojection
        with confidence (1, 1) (graph.py:144-165), computed on the GPU
        (dpv_reproject_exact, bit-identical to the reference's expression)."""
        tri = np.asarray(list(triples), dtype=np.int64).reshape(-1, 3)
        if len(tri) == 0:
            return []
        if kind not in _KIND_CODE:
            raise ValueError(f"unknown edge kind {kind!r}")
        for i, k, j in tri.tolist():
            self._check_edge_indices(i, k, j)
        if kind == LOOP and np.any(tri[:, 0] == tri[:, 2]):
            raise ValueError("loop edges must connect distinct frames")
        from .synthetic import reproject_targets
        src, pat, dst = tri[:, 0], tri[:, 1], tri[:, 2]
        m = self.patch_size ** 2
        ids = self.add_edge_arrays(src, pat, dst, np.zeros((len(tri), m, 2)),
                                   np.ones((len(tri), 2)), kind)
        reproject_targets(self, np.asarray(ids, dtype=np.int64))
        return ids

    def add_edge_arrays(self, src, patch, dst, target, conf, kind=ODOMETRY) -> list[int]:
        """Bulk edge append without reprojection (targets supplied)."""
        first = self.n_edges
        n = len(src)
        self._src.extend(src)
        self._pat.extend(patch)
        self._dst.extend(dst)
        self._tgt.extend(np.asarray(target, dtype=float).reshape(n, -1, 2))
        self._conf.extend(np.asarray(conf, dtype=float).reshape(n, 2))
        self._kind.extend(np.full(n, _KIND_CODE[kind] if isinstance(kind, str) else kind))
        return list(range(first, first + n))

    @staticmethod
    def odometry_triples(frame_id: int, radius: int, patch_counts) -> np.ndarray:
        """connect_frame's triple order (graph.py:171-175): for each earlier
        frame j, all (n, k, j) then all (j, k, n)."""
        out = []
        for j in range(max(0, frame_id - radius), frame_id):
            kn = np.arange(patch_counts[frame_id])
            kj = np.arange(patch_counts[j])
            out.append(np.stack([np.full_like(kn, frame_id), kn, np.full_like(kn, j)], 1))
            out.append(np.stack([np.full_like(kj, j), kj, np.full_like(kj, frame_id)], 1))
        return np.concatenate(out) if out else np.zeros((0, 3), dtype=np.int64)

    def connect_frame(self, frame_id: int, radius: int) -> list[int]:
        counts = np.diff(np.asarray(self._poff))
        return self.add_edges(self.odometry_triples(frame_id, radius, counts), ODOMETRY)

    def _touch_edge(self, i):
        if i < self._edge_clean:
            self._edge_clean = i

    # -- bookkeeping (graph.py:221-258) ---------------------------------------

    def dense_feature_requirement(self) -> set:
        return set(np.unique(self._dst.view).tolist())

    def active_patch_keys(self, edge_indices, confidence_gate: float = 0.5) -> set:
        idx = np.asarray(list(edge_indices), dtype=np.int64)
        if len(idx) == 0:
            return set()
        hit = idx[self._conf.view[idx].max(axis=1) > confidence_gate]
        keys = np.unique(np.stack([self._src.view[hit], self._pat.view[hit]], 1), axis=0)
        return {(int(a), int(b)) for a, b in keys}

    def check_invariants(self) -> None:
        nf = self.n_frames
        assert len(self._poff) == nf + 1
        assert np.all(self._depth.view > 0)
        src, dst, pat = self._src.view, self._dst.view, self._pat.view
        assert np.all((src >= 0) & (src < nf) & (dst >= 0) & (dst < nf))
        counts = np.diff(np.asarray(self._poff))
        assert np.all((pat >= 0) & (pat < counts[src]))
        c = self._conf.view
        assert np.all((c >= 0) & (c <= 1))

    def snapshot_poses(self):
        return [f.pose for f in self.frames]

    # -- SoA export / import ----------------------------------------------------

    def soa(self) -> dict:
        """Host arrays (views) in the oracle / fixture layout."""
        return {
            "intr": self.intrinsics.as_array(), "patch_size": np.int64(self.patch_size),
            "frame_q": self._q.view, "frame_t": self._t.view,
            "patch_offset": self.patch_offset(), "patch_grid": self._grid.view,
            "patch_depth": self._depth.view, "patch_landmark": self._lm.view,
            "edge_src": self._src.view.astype(np.int64), "edge_patch": self._pat.view.astype(np.int64),
            "edge_dst": self._dst.view.astype(np.int64), "edge_target": self._tgt.view,
            "edge_conf": self._conf.view, "edge_kind": self._kind.view,
        }

    @classmethod
    def from_soa(cls, d: dict, timestamps=None) -> "PatchGraph":
        intr = Intrinsics(*[float(v) for v in d["intr"]])
        g = cls(intr, int(d.get("patch_size", 3)))
        off = np.asarray(d["patch_offset"], dtype=np.int64)
        nf = len(d["frame_q"])
        g._q.extend(d["frame_q"])
        g._t.extend(d["frame_t"])
        g._ts.extend(timestamps if timestamps is not None else np.zeros(nf))
        g._kf.extend(np.ones(nf, dtype=bool))
        g._feat.extend(np.ones(nf, dtype=bool))
        g._poff = off.tolist()
        g._grid.extend(d["patch_grid"])
        g._depth.extend(d["patch_depth"])
        g._lm.extend(d.get("patch_landmark", np.full(len(d["patch_depth"]), -1)))
        kind = np.asarray(d.get("edge_kind", np.zeros(len(d["edge_src"]), np.uint8)))
        g._src.extend(d["edge_src"])
        g._pat.extend(d["edge_patch"])
        g._dst.extend(d["edge_dst"])
        g._tgt.extend(d["edge_target"])
        g._conf.extend(d["edge_conf"])
        g._kind.extend(kind)
        return g

    @classmethod
    def from_reference(cls, ref) -> "PatchGraph":
        """Copy a reference ``patchslam.graph.PatchGraph`` (object form) into SoA."""
        intr = Intrinsics(ref.intrinsics.fx, ref.intrinsics.fy, ref.intrinsics.cx,
                          ref.intrinsics.cy)
        g = cls(intr, ref.patch_size)
        for f in ref.frames:
            plist = ref.patches[f.frame_id]
            m = ref.patch_size ** 2
            grids = np.stack([p.grid for p in plist]) if plist else np.zeros((0, m, 2))
            g.add_frame_arrays(f.pose.q, f.pose.t, f.timestamp, grids,
                               np.array([p.inverse_depth for p in plist]),
                               np.array([-1 if p.landmark_id is None else p.landmark_id
                                         for p in plist], dtype=np.int64), f.is_keyframe)
            g._feat.view[f.frame_id] = f.has_dense_features
        e = ref.edges
        if e:
            g.add_edge_arrays(np.array([x.src_frame for x in e]), np.array([x.src_patch for x in e]),
                              np.array([x.dst_frame for x in e]), np.stack([x.target for x in e]),
                              np.stack([x.confidence for x in e]),
                              np.array([_KIND_CODE[x.kind] for x in e], dtype=np.uint8))
        return g

    # -- device mirror ------------------------------------------------------------

    def device(self) -> dict:
        """Device mirror (torch CUDA tensors), re-uploading only what changed."""
        import torch
        mir = self._mirror
        dev = "cuda"
        if mir is None:
            mir = self._mirror = {"pose_ver": -1, "patch_ver": -1, "n_edges": 0}
        if mir["pose_ver"] != self._pose_ver or mir["q"].shape[0] != self.n_frames:
            mir["q"] = torch.as_tensor(np.ascontiguousarray(self._q.view), device=dev)
            mir["t"] = torch.as_tensor(np.ascontiguousarray(self._t.view), device=dev)
            mir["pose_ver"] = self._pose_ver
        if mir["patch_ver"] != self._patch_ver:
            mir["patch_grid"] = torch.as_tensor(np.ascontiguousarray(self._grid.view), device=dev)
            mir["patch_depth"] = torch.as_tensor(np.ascontiguousarray(self._depth.view), device=dev)
            mir["patch_ver"] = self._patch_ver
        ne = self.n_edges
        if mir["n_edges"] != ne or self._edge_clean < ne:
            lo = min(self._edge_clean, mir["n_edges"])
            off = np.asarray(self._poff, dtype=np.int64)
            new = {
                "edge_src": self._src.view[lo:].astype(np.int32),
                "edge_dst": self._dst.view[lo:].astype(np.int32),
                "edge_gpatch": (off[self._src.view[lo:]] + self._pat.view[lo:]).astype(np.int32),
                "edge_target": np.ascontiguousarray(self._tgt.view[lo:]),
                "edge_conf": np.ascontiguousarray(self._conf.view[lo:]),
            }
            for k, v in new.items():
                tv = torch.as_tensor(v, device=dev)
                if lo == 0 or k not in mir:
                    mir[k] = tv
                else:
                    mir[k] = torch.cat([mir[k][:lo], tv])
            mir["n_edges"] = ne
            self._edge_clean = ne
        return mir

    def dpv_view(self):
        """The device mirror as the C-ABI's dpv_graph view (syncs it first)."""
        from . import _lib
        mir = self.device()
        g = _lib.DpvGraph()
        g.n_frames = self.n_frames
        g.cells = self.patch_size ** 2
        g.n_patches = self.n_patches
        g.n_edges = self.n_edges
        g.patch_grid = mir["patch_grid"].data_ptr()
        g.edge_src = mir["edge_src"].data_ptr() if g.n_edges else 0
        g.edge_gpatch = mir["edge_gpatch"].data_ptr() if g.n_edges else 0
        g.edge_dst = mir["edge_dst"].data_ptr() if g.n_edges else 0
        g.edge_target = mir["edge_target"].data_ptr() if g.n_edges else 0
        g.edge_conf = mir["edge_conf"].data_ptr() if g.n_edges else 0
        for i, v in enumerate(self.intrinsics.as_array()):
            g.intr[i] = float(v)
        return g

    def _mirror_poses_written(self, q_dev, t_dev, rows, depth_rows_dev=None):
        """Keep the device mirror current after a device-side write-back."""
        if self._mirror is not None and self._mirror.get("pose_ver") == self._pose_ver - 1:
            self._mirror["q"] = q_dev
            self._mirror["t"] = t_dev
            self._mirror["pose_ver"] = self._pose_ver
