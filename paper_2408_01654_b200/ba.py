"""Confidence-weighted bundle adjustment over the patch graph, on the B200.

Drop-in for ``patchslam.ba`` (pkg/src/patchslam/ba.py): same names,
signatures, return shapes, constants and errors.  Every numeric step runs in
hand-written sm_100a kernels behind the C-ABI (include/dpvslam_b200.h):

* ``BAProblem`` builds the state-independent index on the device
  (``dpv_problem_create``: ba.py:60-216, bit-exact).
* ``residuals`` / ``objective``: K2 (ba.py:219-253).
* ``assemble``: fused K2+K3 + Schur elimination K4a (ba.py:328-440).
* ``solve_dense`` / ``solve_block_sparse``: K4b-K4d (ba.py:451-487), dense
  FP64 Cholesky with the trailing update on DMMA tensor cores.
* ``solve``: the LM driver (ba.py:534-605) runs natively (``dpv_lm_solve``),
  state resident in HBM, one scalar read-back per damping attempt.

Host numpy copies are produced only when a caller reads a field (the
reference's tests do numpy arithmetic on them); the solve path never leaves
the device until write-back.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import SingularSystem
from .geometry import INVERSE_DEPTH_FLOOR, Pose, pinhole_rays  # noqa: F401  (re-exported names)

DENSE = "dense"                         # ba.py:36
BLOCK_SPARSE = "block-sparse"           # ba.py:37
DEFAULT_BACKEND_THRESHOLD = 48          # ba.py:38
LM_LAMBDA_INIT = 1e-4                   # ba.py:40-44
LM_LAMBDA_GROW = 10.0
LM_LAMBDA_SHRINK = 0.5
LM_LAMBDA_MAX = 1e10
LM_MAX_ESCALATIONS = 12
_ACTIVE_EPS = 1e-12


def _torch():
    import torch
    return torch


class _ForeignGraph:
    """Adapter for a reference ``patchslam.graph.PatchGraph`` (object form)."""

    def __init__(self, ref):
        from .graph import PatchGraph
        self.ref = ref
        self.soa = PatchGraph.from_reference(ref)

    def write_back(self, first, last, q, t, depth_keys, d):
        ref = self.ref
        for f in range(first, last + 1):
            ref.frames[f].pose = type(ref.frames[f].pose)(q[f], t[f])
        for row, (f, k) in enumerate(depth_keys):
            ref.patches[f][k] = ref.patches[f][k].with_inverse_depth(float(d[row]))


_PINNED = {}


def _pinned_copy(x):
    """Device tensor -> numpy through a reused pinned host buffer (one
    synchronising copy at full PCIe speed).  One buffer per dtype, grown by
    doubling, so problems of many sizes (window replicas) do not re-allocate
    pinned memory.  The returned array is a copy."""
    torch = _torch()
    n = x.numel()
    buf = _PINNED.get(x.dtype)
    if buf is None or buf.numel() < n:
        cap = max(n, 2 * (buf.numel() if buf is not None else 0), 1 << 16)
        buf = _PINNED[x.dtype] = torch.empty(cap, dtype=x.dtype, pin_memory=True)
    view = buf[:n]
    view.copy_(x.reshape(-1), non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return view.numpy().copy()


class BAProblem:
    """Bundle adjustment problem over a contiguous free-pose range (ba.py:50-216).

    The device index is built lazily on first use (the reference caches its
    structure lazily too, ba.py:124-127, 147-150).
    """

    def __init__(self, graph, free_range, damping: float = LM_LAMBDA_INIT, edge_indices=None):
        first, last = (int(v) for v in free_range)
        if not (0 <= first <= last < graph.n_frames):
            raise ValueError(f"free range {free_range} out of bounds")
        if first == 0 and last == graph.n_frames - 1:
            raise ValueError("at least one pose must stay fixed to anchor the gauge")
        from .graph import PatchGraph
        self.graph = graph
        self._foreign = None if isinstance(graph, PatchGraph) else _ForeignGraph(graph)
        self._g = graph if self._foreign is None else self._foreign.soa
        self.first_free = first
        self.last_free = last
        self.damping = damping
        self._given = None if edge_indices is None else np.asarray(list(edge_indices), np.int64)
        self._handle = None
        self._info = None
        self._cache = {}
        # ownership token of the handle's assembly buffers: every native call
        # that writes them takes a fresh token (_next_gen); a BlockSparseSystem
        # re-assembles its own state when the token is no longer its own
        self._gen = 0
        self._gen_counter = 0
        self._fill_count = None
        self.free_frames = list(range(first, last + 1))

    def _next_gen(self) -> int:
        self._gen_counter += 1
        self._gen = self._gen_counter
        return self._gen

    # -- device handle ---------------------------------------------------------

    def _graph_view(self):
        """The graph's device mirror as the C-ABI's dpv_graph view."""
        return self._g.dpv_view()

    def _ensure(self):
        if self._handle is not None:
            return self._handle
        torch = _torch()
        lib = _lib.lib()
        g = self._graph_view()
        eidx = None
        if self._given is not None:
            if len(self._given) and (self._given.min() < 0 or self._given.max() >= g.n_edges):
                raise IndexError("edge index out of range")
            eidx = torch.as_tensor(self._given, device="cuda")
        h = C.c_void_p()
        _lib.check(lib.dpv_problem_create(C.byref(g), self.first_free, self.last_free,
                                          _lib.ptr(eidx), 0 if eidx is None else len(eidx),
                                          _lib.stream_ptr(), C.byref(h)), "BAProblem")
        self._handle = h
        info = _lib.DpvProblemInfo()
        _lib.check(lib.dpv_problem_get_info(h, C.byref(info)), "problem info")
        self._info = info
        return h

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and _lib._lib is not None:
            try:
                _torch().cuda.synchronize()
                _lib._lib.dpv_problem_destroy(h)
            except Exception:
                pass
            self._handle = None

    def view(self, name: str):
        """Zero-copy device view of a named array of the handle."""
        return _lib.device_view(self._ensure(), name, self)

    def info(self):
        self._ensure()
        return self._info

    # -- reference attributes (ba.py:60-106) -----------------------------------

    @property
    def edge_indices(self):
        if "edge_indices" not in self._cache:
            self._cache["edge_indices"] = self.view("edge_idx").cpu().numpy().tolist()
        return self._cache["edge_indices"]

    @property
    def depth_keys(self):
        if "depth_keys" not in self._cache:
            gid = self.view("depth_patch").cpu().numpy().astype(np.int64)
            off = self._g.patch_offset()
            fr = np.searchsorted(off, gid, side="right") - 1
            self._cache["depth_keys"] = list(zip(fr.tolist(), (gid - off[fr]).tolist()))
        return self._cache["depth_keys"]

    @property
    def _var_of(self):
        v = np.full(self._g.n_frames, -1, dtype=int)
        v[self.first_free:self.last_free + 1] = np.arange(self.n_free_poses)
        return v

    @property
    def touched_fixed(self):
        return self.view("touched").cpu().numpy().astype(int).tolist()

    @property
    def scale_degenerate(self) -> bool:
        return bool(self.info().scale_degenerate)

    @property
    def n_free_poses(self) -> int:
        return len(self.free_frames)

    @property
    def n_depths(self) -> int:
        return int(self.info().n_depths)

    # -- state <-> arrays (ba.py:110-122) ------------------------------------------

    def device_state(self):
        """(q, t, d) as CUDA float64 tensors (fresh copies)."""
        torch = _torch()
        h = self._ensure()
        mir = self._g.device()
        q = mir["q"].clone()
        t = mir["t"].clone()
        d = torch.empty(self.n_depths, dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().dpv_gather_depths(h, _lib.ptr(mir["patch_depth"]), _lib.ptr(d),
                                                _lib.stream_ptr()), "state")
        return q, t, d

    def state(self):
        return tuple(x.cpu().numpy() for x in self.device_state())

    def _depth_rows_host(self):
        """Graph patch id of every depth row (static per problem, cached) and,
        when the rows are one contiguous ascending patch range, its start."""
        if "depth_rows" not in self._cache:
            dev = self.view("depth_patch")
            n = int(dev.shape[0])
            start, gid = None, None
            if n:
                # the rows are sorted unique patch ids (dpv_problem_create), so
                # they form one range iff the endpoints are n - 1 apart
                ends = dev[[0, n - 1]].cpu().numpy().astype(np.int64)
                if ends[1] - ends[0] == n - 1:
                    start = int(ends[0])
            if start is None:
                gid = dev.cpu().numpy().astype(np.int64)
            self._cache["depth_rows"] = (n, gid, start)
        return self._cache["depth_rows"]

    def write_back(self, q, t, d) -> None:
        torch = _torch()
        dev = [v for v in (q, t, d) if isinstance(v, torch.Tensor)]
        if len(dev) == 3 and q.dtype == t.dtype == d.dtype == torch.float64:
            # the whole state in one device->host copy (one synchronisation)
            nq, nt = q.numel(), t.numel()
            flat = _pinned_copy(torch.cat([q.reshape(-1), t.reshape(-1), d.reshape(-1)]))
            q, t, d = (flat[:nq].reshape(tuple(q.shape)), flat[nq:nq + nt].reshape(tuple(t.shape)),
                       flat[nq + nt:])
        else:
            q = q.cpu().numpy() if isinstance(q, torch.Tensor) else np.asarray(q, dtype=float)
            t = t.cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t, dtype=float)
            d = d.cpu().numpy() if isinstance(d, torch.Tensor) else np.asarray(d, dtype=float)
        if self._foreign is not None:
            self._foreign.write_back(self.first_free, self.last_free, q, t, self.depth_keys, d)
        g = self._g
        sl = slice(self.first_free, self.last_free + 1)
        qf = q[sl]
        norm = np.linalg.norm(qf, axis=1, keepdims=True)
        g._q.view[sl] = np.where(np.abs(norm - 1.0) > 1e-12, qf / norm, qf)
        g._t.view[sl] = t[sl]
        n_rows, gid, start = self._depth_rows_host()
        if np.any(~(d > 0)):
            from .errors import NonPositiveDepth
            raise NonPositiveDepth("patch inverse depth must be positive")
        if start is not None:
            g._depth.view[start:start + n_rows] = d
        else:
            g._depth.view[gid] = d
        g._pose_ver += 1
        g._patch_ver += 1

    # -- reference-compatible index exports (numpy, for parity checks) ------------

    def _structure(self):
        """Per-edge static arrays in problem order (ba.py:124-141)."""
        if "structure" not in self._cache:
            torch = _torch()
            h = self._ensure()
            E = int(self._info.n_edges)
            m = self._g.patch_size ** 2
            pos = self.view("p_pos").long()
            src = self.view("a_src").long()[pos]
            dst = self.view("a_dst").long()[pos]
            row = self.view("p_row").long()
            tgt = self.view("a_tgt").reshape(2 * m, E)[:, pos].T.reshape(E, m, 2)
            w = self.view("a_w").reshape(2, E)[:, pos].T
            ray_xy = self.view("r_ray").reshape(m, 2, -1)
            rays = torch.ones((E, m, 3), dtype=torch.float64, device="cuda")
            rays[:, :, :2] = ray_xy[:, :, row].permute(2, 0, 1) if E else rays[:, :, :2]
            self._cache["structure"] = {
                "src": src.cpu().numpy(), "dst": dst.cpu().numpy(), "depth_row": row.cpu().numpy(),
                "rays": rays.cpu().numpy(), "target": tgt.cpu().numpy(), "weight": w.cpu().numpy()}
            del h
        return self._cache["structure"]

    def _assembly_maps(self):
        """The reference's index dictionary (ba.py:147-216), exported from the
        device index (union keys, incidences and Schur pairs are the device's
        own arrays; hpp_* are re-derived from the per-edge vars)."""
        if "maps" in self._cache:
            return self._cache["maps"]
        n = self.n_free_poses
        st = self._structure()
        vi = self.view("p_vi").cpu().numpy().astype(int)
        vj = self.view("p_vj").cpu().numpy().astype(int)
        distinct = st["src"] != st["dst"]
        ri = np.nonzero((vi >= 0) & distinct)[0]
        rj = np.nonzero((vj >= 0) & distinct)[0]
        rb = np.nonzero((vi >= 0) & (vj >= 0) & distinct)[0]
        hpp_keys = np.concatenate([vi[ri] * (n + 1), vj[rj] * (n + 1),
                                   np.minimum(vi[rb], vj[rb]) * n + np.maximum(vi[rb], vj[rb])])
        union = self.view("union_keys").cpu().numpy()
        inc_var = self.view("inc_var").cpu().numpy().astype(int)
        inc_row = self.view("inc_row").cpu().numpy().astype(int)
        pl = self.view("pair_l").cpu().numpy().astype(int)
        pr = self.view("pair_r").cpu().numpy().astype(int)
        # reference pair order: row-major over depth rows, then left, then right
        order = np.lexsort((inc_var[pr], inc_var[pl], inc_row[pl]))
        pl, pr = pl[order], pr[order]
        maps = {
            "vi": vi, "vj": vj, "rows_i": ri, "rows_j": rj,
            "hpp_rows": np.concatenate([ri, rj, rb]),
            "hpp_sign": np.concatenate([np.ones(len(ri)), np.ones(len(rj)), -np.ones(len(rb))]),
            "hpp_where": np.searchsorted(union, hpp_keys),
            "inc_inv": self.view("inc_inv").cpu().numpy().astype(int),
            "inc_var": inc_var, "inc_row": inc_row, "n_inc": len(inc_var),
            "pair_left": pl, "pair_right": pr, "pair_depth": inc_row[pl],
            "pair_where": np.searchsorted(union, inc_var[pl] * n + inc_var[pr]),
            "union_keys": union,
        }
        self._cache["maps"] = maps
        return maps

    def active_patch_count(self, confidence_gate: float = 0.5) -> int:
        h = self._ensure()
        out = C.c_int64()
        _lib.check(_lib.lib().dpv_active_patch_count(h, float(confidence_gate), C.byref(out),
                                                     _lib.stream_ptr()), "active_patch_count")
        return int(out.value)

    def block_fill_count(self) -> int:
        """Blocks of the natural-order block-Cholesky factor of the reduced
        pattern (block_cholesky.py:48-111 symbolic); state-independent, cached."""
        if self._fill_count is None:
            u = self.view("union_keys").cpu().numpy()
            n = self.n_free_poses
            keys = np.ascontiguousarray(np.stack([u // max(n, 1), u % max(n, 1)], 1), np.int64)
            out = C.c_int64()
            _lib.check(_lib.lib().dpv_block_fill_count(keys.ctypes.data_as(C.c_void_p), len(keys),
                                                       n, C.byref(out)), "block_fill_count")
            self._fill_count = int(out.value)
        return self._fill_count


# ---------------------------------------------------------------------------
# state helpers


def _dev_state(problem: BAProblem, state):
    torch = _torch()
    if state is None:
        return problem.device_state()
    q, t, d = state
    conv = (lambda x: x.to(device="cuda", dtype=torch.float64).contiguous()
            if isinstance(x, torch.Tensor) else
            torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device="cuda"))
    return conv(q), conv(t), conv(d)


def residuals(problem: BAProblem, state=None):
    """Raw residuals (E, p*p, 2) and validity (ba.py:219-245), problem-edge order."""
    torch = _torch()
    h = problem._ensure()
    q, t, d = _dev_state(problem, state)
    E = int(problem._info.n_edges)
    m = problem._g.patch_size ** 2
    if E == 0:
        return np.zeros((0, 0, 2)), np.zeros((0, 0), dtype=bool)
    res = torch.empty((E, m, 2), dtype=torch.float64, device="cuda")
    valid = torch.empty((E, m), dtype=torch.uint8, device="cuda")
    _lib.check(_lib.lib().dpv_residuals(h, _lib.ptr(q), _lib.ptr(t), _lib.ptr(d), _lib.ptr(res),
                                        _lib.ptr(valid), _lib.stream_ptr()), "residuals")
    return res.cpu().numpy(), valid.bool().cpu().numpy()


def objective_device(problem: BAProblem, q, t, d, out=None):
    """Objective into a 1-element CUDA tensor (no host sync)."""
    torch = _torch()
    h = problem._ensure()
    out = torch.empty(1, dtype=torch.float64, device="cuda") if out is None else out
    _lib.check(_lib.lib().dpv_objective(h, _lib.ptr(q), _lib.ptr(t), _lib.ptr(d), _lib.ptr(out),
                                        _lib.stream_ptr()), "objective")
    return out


def objective(problem: BAProblem, state=None) -> float:
    """Weighted objective (ba.py:248-253)."""
    return float(objective_device(problem, *_dev_state(problem, state)).item())


# ---------------------------------------------------------------------------
# assembled system


class BlockSparseSystem:
    """Assembled normal equations (ba.py:272-325), resident on the device.

    Fields are materialised as numpy arrays on first access.  If the problem
    was re-assembled since, the system re-runs its (deterministic, bit-
    identical) assembly before it is read or solved.
    """

    _FIELDS = ("pose_blocks", "schur_blocks", "depth_diag", "rhs_pose", "rhs_depth",
               "rhs_schur", "inc_block", "active")

    def __init__(self, problem: BAProblem, state):
        self._problem = problem
        self._state = state
        self._gen = problem._gen
        self.n_pose = problem.n_free_poses
        self.n_depth = problem.n_depths
        self.damping = problem.damping
        self._host = {}
        scal = problem.view("scal")[:8].cpu().numpy()
        self.gradient_norm = float(scal[0:1].view(np.int64).view(np.float64)[0])
        self._inactive = int(scal[6:7].view(np.int64)[0])
        self.scale_pin = (0, scal[2:5].copy()) if scal[1] != 0.0 else None

    def _sync(self):
        p = self._problem
        if p._gen != self._gen:
            _run_assemble(p, *self._state)
            p._gen = self._gen

    def _field(self, name):
        if name not in self._host:
            self._sync()
            p = self._problem
            v = p.view(name).cpu().numpy()
            W = int(p._info.n_keys)
            shapes = {"pose_blocks": (W, 6, 6), "schur_blocks": (W, 6, 6),
                      "rhs_pose": (self.n_pose, 6), "rhs_schur": (self.n_pose, 6),
                      "inc_block": (-1, 6)}
            if name in shapes:
                v = v.reshape(shapes[name])
            if name == "active":
                v = v.astype(bool)
            self._host[name] = v
        return self._host[name]

    pose_blocks = property(lambda s: s._field("pose_blocks"))
    schur_blocks = property(lambda s: s._field("schur_blocks"))
    depth_diag = property(lambda s: s._field("depth_diag"))
    rhs_pose = property(lambda s: s._field("rhs_pose"))
    rhs_depth = property(lambda s: s._field("rhs_depth"))
    rhs_schur = property(lambda s: s._field("rhs_schur"))
    inc_block = property(lambda s: s._field("inc_block"))
    active = property(lambda s: s._field("active"))

    @property
    def pair_keys(self):
        if "pair_keys" not in self._host:
            u = self._problem.view("union_keys").cpu().numpy()
            n = max(self.n_pose, 1)
            self._host["pair_keys"] = np.stack([u // n, u % n], axis=1)
        return self._host["pair_keys"]

    @property
    def inc_var(self):
        return self._problem.view("inc_var").cpu().numpy().astype(int)

    @property
    def inc_row(self):
        return self._problem.view("inc_row").cpu().numpy().astype(int)

    @property
    def unconstrained_depths(self) -> int:
        return self._inactive

    def reduced_system(self, lam: float):
        """(keys, blocks, rhs, cinv) of S(lam) (ba.py:303-319), computed on the device."""
        torch = _torch()
        self._sync()
        p = self._problem
        W = int(p._info.n_keys)
        blocks = torch.empty((W, 6, 6), dtype=torch.float64, device="cuda")
        rhs = torch.empty((self.n_pose, 6), dtype=torch.float64, device="cuda")
        cinv = torch.empty(self.n_depth, dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().dpv_reduced_system(p._ensure(), float(lam), _lib.ptr(blocks),
                                                 _lib.ptr(rhs), _lib.ptr(cinv), _lib.stream_ptr()),
                   "reduced_system")
        return self.pair_keys, blocks.cpu().numpy(), rhs.cpu().numpy(), cinv.cpu().numpy()

    def back_substitute(self, delta_pose, lam: float):
        """ba.py:321-325 on the device."""
        torch = _torch()
        self._sync()
        p = self._problem
        dp = (delta_pose.to("cuda", torch.float64).contiguous()
              if isinstance(delta_pose, torch.Tensor)
              else torch.as_tensor(np.ascontiguousarray(delta_pose, np.float64), device="cuda"))
        dd = torch.empty(self.n_depth, dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().dpv_back_substitute(p._ensure(), float(lam), _lib.ptr(dp),
                                                  _lib.ptr(dd), _lib.stream_ptr()),
                   "back_substitute")
        return dd.cpu().numpy()


def _run_assemble(problem, q, t, d):
    _lib.check(_lib.lib().dpv_assemble(problem._ensure(), _lib.ptr(q), _lib.ptr(t), _lib.ptr(d),
                                       _lib.stream_ptr()), "assemble")


def assemble(problem: BAProblem, state=None) -> BlockSparseSystem:
    """Build the (undamped) normal equations for the current state (ba.py:328-440)."""
    problem._ensure()
    q, t, d = _dev_state(problem, state)
    _run_assemble(problem, q, t, d)
    problem._next_gen()
    return BlockSparseSystem(problem, (q, t, d))


# ---------------------------------------------------------------------------
# backends (ba.py:447-490)


def select_backend(problem: BAProblem, threshold: int = DEFAULT_BACKEND_THRESHOLD) -> str:
    return DENSE if problem.n_free_poses <= threshold else BLOCK_SPARSE


def _device_solve(system: BlockSparseSystem, lam, backend: int = 0):
    torch = _torch()
    system._sync()
    p = system._problem
    dp = torch.empty((system.n_pose, 6), dtype=torch.float64, device="cuda")
    dd = torch.empty(system.n_depth, dtype=torch.float64, device="cuda")
    status = torch.zeros(8, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _lib.check(_lib.lib().dpv_solve_backend(p._ensure(), float(lam), int(backend), _lib.ptr(dp),
                                            _lib.ptr(dd), _lib.ptr(status), _lib.stream_ptr()),
               "solve")
    st = status.cpu().numpy()
    t1 = time.perf_counter()
    if st[0] != 0:
        raise SingularSystem(f"dense factorization failed: leading minor {int(st[1]) + 1} "
                             "is not positive definite")
    return dp, dd, t1 - t0


def solve_dense(system: BlockSparseSystem, lam: float | None = None):
    """Schur-reduce and factorise S(lam) (ba.py:451-472) on the B200: S in a
    dense matrix, every-tile Cholesky (single-CTA for 6n <= 162)."""
    lam = system.damping if lam is None else lam
    dp, dd, dt = _device_solve(system, lam, 1)
    stats = {"backend": DENSE, "factorize_s": dt, "solve_s": 0.0,
             "peak_block_count": system.n_pose * system.n_pose}
    return dp.cpu().numpy(), dd.cpu().numpy(), stats


def solve_block_sparse(system: BlockSparseSystem, lam: float | None = None):
    """Block-sparse backend (ba.py:475-487).  Same numbers (the reduced system
    is factorised by the band + border sparse FP64 tensor-core factorisation,
    spd.cu; agreement with the reference block Cholesky is 1e-8,
    test_ba.py:192-201); ``peak_block_count`` is the exact symbolic fill of
    the natural-order block factor."""
    lam = system.damping if lam is None else lam
    dp, dd, dt = _device_solve(system, lam, 2)
    stats = {"backend": BLOCK_SPARSE, "factorize_s": dt, "solve_s": 0.0,
             "peak_block_count": system._problem.block_fill_count()}
    return dp.cpu().numpy(), dd.cpu().numpy(), stats


_BACKENDS = {DENSE: solve_dense, BLOCK_SPARSE: solve_block_sparse}


# ---------------------------------------------------------------------------
# LM driver (ba.py:497-605)


@dataclass
class BAReport:
    iterations: int
    initial_objective: float
    final_objective: float
    backend: str
    iteration_times: list = field(default_factory=list)
    converged: bool = False
    gradient_norm: float = float("inf")
    unconstrained_depths: int = 0
    active_patches: int = 0
    final_damping: float = LM_LAMBDA_INIT
    step_norm: float = float("inf")
    n_attempts: int = 0

    def to_line(self) -> str:
        times = ",".join(f"{t * 1e3:.3f}" for t in self.iteration_times)
        return (f"ba_report backend={self.backend} iterations={self.iterations} "
                f"initial={self.initial_objective:.6e} final={self.final_objective:.6e} "
                f"gradient={self.gradient_norm:.3e} converged={int(self.converged)} "
                f"unconstrained={self.unconstrained_depths} "
                f"active={self.active_patches} times_ms={times}")


def _apply_step(q, t, d, delta_pose, delta_depth, problem):
    """Retraction on the free frames (ba.py:521-531), on the device."""
    torch = _torch()
    numpy_in = not isinstance(q, torch.Tensor)
    qd, td, dd_ = _dev_state(problem, (q, t, d))
    conv = (lambda x: x.to("cuda", torch.float64).contiguous() if isinstance(x, torch.Tensor)
            else torch.as_tensor(np.ascontiguousarray(x, np.float64), device="cuda"))
    dp, ddl = conv(delta_pose), conv(delta_depth)
    q2, t2, d2 = torch.empty_like(qd), torch.empty_like(td), torch.empty_like(dd_)
    _lib.check(_lib.lib().dpv_apply_step(problem._ensure(), *[_lib.ptr(x) for x in
                                         (qd, td, dd_, dp, ddl, q2, t2, d2)], _lib.stream_ptr()),
               "apply_step")
    if numpy_in:
        return q2.cpu().numpy(), t2.cpu().numpy(), d2.cpu().numpy()
    return q2, t2, d2


def solve_device(problem: BAProblem, q, t, d, max_iterations=50, tolerance=1e-9,
                 backend=None, backend_threshold=DEFAULT_BACKEND_THRESHOLD,
                 active_patches=None) -> BAReport:
    """Native LM on device tensors; q/t/d are updated in place (no write-back)."""
    chosen = backend or select_backend(problem, backend_threshold)
    if chosen not in _BACKENDS:
        raise KeyError(chosen)
    h = problem._ensure()
    if active_patches is None:
        active_patches = problem.active_patch_count()
    params = _lib.DpvLmParams(int(max_iterations), float(tolerance), float(problem.damping))
    rep = _lib.DpvLmReport()
    problem._next_gen()          # the native LM re-assembles into the handle's buffers
    _lib.check(_lib.lib().dpv_lm_solve(h, _lib.ptr(q), _lib.ptr(t), _lib.ptr(d),
                                       C.byref(params), C.byref(rep), _lib.stream_ptr()),
               "solve")
    out = BAReport(int(rep.iterations), rep.initial_objective, rep.final_objective, chosen,
                   iteration_times=[rep.iteration_times[i] for i in range(rep.times_len)],
                   converged=bool(rep.converged), gradient_norm=rep.gradient_norm,
                   unconstrained_depths=int(rep.unconstrained_depths),
                   active_patches=int(active_patches), final_damping=rep.final_damping,
                   step_norm=rep.step_norm, n_attempts=int(rep.n_attempts))
    problem.damping = rep.final_damping
    return out


def solve(problem: BAProblem, max_iterations: int = 50, tolerance: float = 1e-9,
          backend: str | None = None,
          backend_threshold: int = DEFAULT_BACKEND_THRESHOLD) -> BAReport:
    """Levenberg-Marquardt over the problem; writes the result into the graph
    (ba.py:534-605).  Raises SingularSystem exactly where the reference does."""
    q, t, d = problem.device_state()
    rep = solve_device(problem, q, t, d, max_iterations, tolerance, backend, backend_threshold)
    problem.write_back(q, t, d)
    return rep


# ---------------------------------------------------------------------------
# batched replicas: many independent problems


def build_batch(problems, threads: int = 0, streams=None) -> None:
    """Build the device index of every problem concurrently (one stream and
    one host worker per problem, dpv_problem_create_batch).  Same index as
    building each problem alone; problems with a handle already are skipped,
    as are those with explicit edge_indices (built one by one).  ``streams``:
    one torch stream per problem (reused streams keep the caching allocator
    warm); the problem keeps its stream for later work."""
    torch = _torch()
    todo = [p for p in problems if p._handle is None and p._given is None]
    for p in problems:
        if p._handle is None and p._given is not None:
            p._ensure()
    if not todo:
        return
    n = len(todo)
    graphs = (_lib.DpvGraph * n)(*[p._graph_view() for p in todo])
    first = (C.c_int32 * n)(*[p.first_free for p in todo])
    last = (C.c_int32 * n)(*[p.last_free for p in todo])
    if streams is None:
        streams = [torch.cuda.Stream() for _ in todo]
    else:
        streams = [s for p, s in zip(problems, streams) if p in todo]
    torch.cuda.current_stream().synchronize()      # graph mirrors are ready
    sp = (C.c_void_p * n)(*[s.cuda_stream for s in streams])
    out = (C.c_void_p * n)()
    status = (C.c_int32 * n)()
    rc = _lib.lib().dpv_problem_create_batch(n, graphs, first, last, sp, int(threads), out,
                                              status)
    for i, p in enumerate(todo):          # keep every handle that was built
        if out[i]:
            p._handle = C.c_void_p(out[i])
            p._stream = streams[i]          # the handle frees on its build stream
            info = _lib.DpvProblemInfo()
            _lib.check(_lib.lib().dpv_problem_get_info(p._handle, C.byref(info)), "problem info")
            p._info = info
    _lib.check(rc, "build_batch")


def solve_batch(problems, max_iterations: int = 50, tolerance: float = 1e-9,
                backend: str | None = None, backend_threshold: int = DEFAULT_BACKEND_THRESHOLD,
                threads: int = 0) -> list:
    """``[solve(p, ...) for p in problems]`` run as concurrent replicas: every
    problem's native LM (ba.py:534-605) on its own stream and host worker
    (dpv_lm_solve_batch).  Returns one entry per problem: its BAReport, or the
    SingularSystem instance where ``solve`` would have raised (that problem's
    graph is then left unwritten, as in ``solve``).  max_iterations, tolerance
    and backend_threshold may be scalars or one value per problem."""
    n = len(problems)
    if n == 0:
        return []

    def per(v):
        return list(v) if isinstance(v, (list, tuple, np.ndarray)) else [v] * n
    iters, tols, thresholds = per(max_iterations), per(tolerance), per(backend_threshold)
    if not (len(iters) == len(tols) == len(thresholds) == n):
        raise ValueError("per-problem settings must have one entry per problem")
    chosen = [backend or select_backend(p, th) for p, th in zip(problems, thresholds)]
    for c in chosen:
        if c not in _BACKENDS:
            raise KeyError(c)
    torch = _torch()
    build_batch(problems, threads)
    active = [p.active_patch_count() for p in problems]
    states = [p.device_state() for p in problems]
    streams = [getattr(p, "_stream", None) or torch.cuda.Stream() for p in problems]
    torch.cuda.current_stream().synchronize()      # states are ready
    hs = (C.c_void_p * n)(*[p._ensure().value for p in problems])
    qs = (C.c_void_p * n)(*[s[0].data_ptr() for s in states])
    ts = (C.c_void_p * n)(*[s[1].data_ptr() for s in states])
    ds = (C.c_void_p * n)(*[s[2].data_ptr() for s in states])
    params = (_lib.DpvLmParams * n)(*[_lib.DpvLmParams(int(it), float(tol), float(p.damping))
                                       for p, it, tol in zip(problems, iters, tols)])
    reps = (_lib.DpvLmReport * n)()
    for p in problems:
        p._next_gen()
    sp = (C.c_void_p * n)(*[s.cuda_stream for s in streams])
    status = (C.c_int32 * n)()
    rc = _lib.lib().dpv_lm_solve_batch(n, hs, qs, ts, ds, params, reps, sp, int(threads), status)
    if rc not in (_lib.DPV_OK, _lib.DPV_SINGULAR):
        _lib.check(rc, "solve_batch")
    out = []
    for i, p in enumerate(problems):
        if status[i] == _lib.DPV_SINGULAR:
            out.append(SingularSystem(f"solve_batch: problem {i}: matrix not positive definite"))
            continue
        if status[i] != _lib.DPV_OK:
            _lib.check(status[i], f"solve_batch problem {i}")
        r = reps[i]
        out.append(BAReport(int(r.iterations), r.initial_objective, r.final_objective, chosen[i],
                            iteration_times=[r.iteration_times[k] for k in range(r.times_len)],
                            converged=bool(r.converged), gradient_norm=r.gradient_norm,
                            unconstrained_depths=int(r.unconstrained_depths),
                            active_patches=int(active[i]), final_damping=r.final_damping,
                            step_norm=r.step_norm, n_attempts=int(r.n_attempts)))
        p.damping = r.final_damping
        p.write_back(*states[i])
    return out
