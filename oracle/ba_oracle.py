"""Float64 numpy restatement of the reference bundle adjustment on SoA graphs.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates
/root/reference/pkg/src/patchslam/ba.py (problem construction, residuals,
objective, assembly with Schur elimination of inverse depths, damped reduced
system, dense and block-sparse solves, retraction, LM driver) and
block_cholesky.py, operating on the structure-of-arrays graph dictionary the
B200 package uses (keys ``frame_q, frame_t, patch_offset, patch_grid,
patch_depth, edge_src, edge_patch, edge_dst, edge_target, edge_conf, intr``).

Index arrays are meant to be bit-identical to the reference's; float results
agree to rounding (summation order of numpy matmul/einsum may differ).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

from .geometry_oracle import (INVERSE_DEPTH_FLOOR, exp_rotation, hamilton, normalize,
                              quat_to_rot, rays_from_grid, reproject, rotate)

DENSE = "dense"                 # ba.py:36
BLOCK_SPARSE = "block-sparse"   # ba.py:37
THRESHOLD = 48                  # ba.py:38
LAMBDA_INIT = 1e-4              # ba.py:40-44
LAMBDA_GROW = 10.0
LAMBDA_SHRINK = 0.5
LAMBDA_MAX = 1e10
MAX_ESCALATIONS = 12
CHUNK = 32768                   # ba.py:46
ACTIVE_EPS = 1e-12              # ba.py:47


class OracleSingular(Exception):
    """Mirror of patchslam.errors.SingularSystem (errors.py:28-29)."""


# ---------------------------------------------------------------------------
# problem construction (ba.py:60-216)


class OracleProblem:
    """ba.BAProblem restated on a SoA graph (ba.py:60-98)."""

    def __init__(self, g: dict, free_range, damping=LAMBDA_INIT, edge_indices=None):
        n_frames = len(g["frame_q"])
        first, last = (int(v) for v in free_range)
        if not (0 <= first <= last < n_frames):
            raise ValueError(f"free range {free_range} out of bounds")
        if first == 0 and last == n_frames - 1:
            raise ValueError("at least one pose must stay fixed to anchor the gauge")
        self.g = g
        self.first_free, self.last_free = first, last
        self.damping = damping
        src_all = np.asarray(g["edge_src"], dtype=np.int64)
        dst_all = np.asarray(g["edge_dst"], dtype=np.int64)
        if edge_indices is None:
            inside = (((src_all >= first) & (src_all <= last))
                      | ((dst_all >= first) & (dst_all <= last)))
            edge_indices = np.nonzero(inside)[0]
        self.edge_indices = np.asarray(edge_indices, dtype=np.int64).reshape(-1)
        src = src_all[self.edge_indices]
        dst = dst_all[self.edge_indices]
        gpatch = (np.asarray(g["patch_offset"], dtype=np.int64)[src]
                  + np.asarray(g["edge_patch"], dtype=np.int64)[self.edge_indices])
        # sorted {(src_frame, src_patch)}: global patch ids are monotone in that pair
        self.depth_patch = np.unique(gpatch)
        self.edge_row = np.searchsorted(self.depth_patch, gpatch)
        self.free_frames = np.arange(first, last + 1)
        self.var_of = np.full(n_frames, -1, dtype=np.int64)
        self.var_of[first:last + 1] = np.arange(last - first + 1)
        ends = np.concatenate([src, dst])
        self.touched_fixed = np.unique(ends[self.var_of[ends] < 0])
        self.scale_degenerate = len(self.touched_fixed) <= 1
        self._src, self._dst = src, dst
        self._static = None
        self._maps = None

    @property
    def n_free(self) -> int:
        return len(self.free_frames)

    @property
    def n_depth(self) -> int:
        return len(self.depth_patch)

    def depth_keys(self) -> np.ndarray:
        off = np.asarray(self.g["patch_offset"], dtype=np.int64)
        frame = np.searchsorted(off, self.depth_patch, side="right") - 1
        return np.stack([frame, self.depth_patch - off[frame]], axis=1)

    def state(self):
        """ba.py:110-115."""
        return (np.array(self.g["frame_q"], dtype=float), np.array(self.g["frame_t"], dtype=float),
                np.array(self.g["patch_depth"], dtype=float)[self.depth_patch])

    def write_back(self, q, t, d) -> None:
        """ba.py:117-122 (Pose renormalises only on drift > 1e-12, geometry.py:174-180)."""
        sl = slice(self.first_free, self.last_free + 1)
        qf = np.array(q[sl], dtype=float)
        norm = np.linalg.norm(qf, axis=1, keepdims=True)
        qf = np.where(np.abs(norm - 1.0) > 1e-12, qf / norm, qf)
        self.g["frame_q"][sl] = qf
        self.g["frame_t"][sl] = t[sl]
        self.g["patch_depth"][self.depth_patch] = d

    def structure(self):
        """Per-edge static arrays.  ba.py:124-141."""
        if self._static is None:
            g = self.g
            gpatch = self.depth_patch[self.edge_row]
            self._static = {
                "src": self._src, "dst": self._dst, "depth_row": self.edge_row,
                "rays": rays_from_grid(np.asarray(g["patch_grid"])[gpatch], g["intr"]),
                "target": np.asarray(g["edge_target"], dtype=float)[self.edge_indices],
                "weight": np.asarray(g["edge_conf"], dtype=float)[self.edge_indices],
            }
        return self._static

    def active_patch_count(self, gate=0.5) -> int:
        """graph.py:232-241 via ba.py:143-145."""
        conf = np.asarray(self.g["edge_conf"])[self.edge_indices]
        hit = conf.max(axis=1, initial=-np.inf) > gate if len(conf) else np.zeros(0, bool)
        return int(len(np.unique(self.edge_row[hit])))

    def maps(self):
        """State-independent normal-equation index.  ba.py:147-216."""
        if self._maps is not None:
            return self._maps
        st = self.structure()
        nf, nd = self.n_free, self.n_depth
        vi = self.var_of[st["src"]]
        vj = self.var_of[st["dst"]]
        distinct = st["src"] != st["dst"]
        ri = np.nonzero((vi >= 0) & distinct)[0]
        rj = np.nonzero((vj >= 0) & distinct)[0]
        rb = np.nonzero((vi >= 0) & (vj >= 0) & distinct)[0]
        lo = np.minimum(vi[rb], vj[rb])
        hi = np.maximum(vi[rb], vj[rb])
        hpp_keys = np.concatenate([vi[ri] * (nf + 1), vj[rj] * (nf + 1), lo * nf + hi])
        hpp_sign = np.concatenate([np.ones(len(ri)), np.ones(len(rj)), -np.ones(len(rb))])
        hpp_rows = np.concatenate([ri, rj, rb])
        row = st["depth_row"]
        inc_keys = np.concatenate([vi[ri] * nd + row[ri], vj[rj] * nd + row[rj]]).astype(np.int64)
        uniq, inc_inv = np.unique(inc_keys, return_inverse=True)
        inc_var = uniq // max(nd, 1)
        inc_row = uniq % max(nd, 1)
        # incidence pairs per depth row: all (l, r) with var[l] <= var[r]
        order = np.argsort(inc_row, kind="stable")
        s_var = inc_var[order]
        cnt = np.bincount(inc_row[order], minlength=nd) if len(order) else np.zeros(nd, np.int64)
        start = np.concatenate([[0], np.cumsum(cnt)[:-1]]).astype(np.int64)
        npair = cnt * cnt
        tot = int(npair.sum())
        seg = np.repeat(np.arange(nd), npair)
        local = np.arange(tot) - np.repeat(np.concatenate([[0], np.cumsum(npair)[:-1]]), npair)
        m = np.maximum(cnt[seg], 1)
        left = start[seg] + local // m
        right = start[seg] + local % m
        keep = s_var[left] <= s_var[right]
        left, right = left[keep], right[keep]
        schur_keys = s_var[left] * nf + s_var[right]
        union = np.unique(np.concatenate([hpp_keys, schur_keys, np.arange(nf) * (nf + 1)]))
        self._maps = {
            "vi": vi, "vj": vj, "rows_i": ri, "rows_j": rj,
            "hpp_rows": hpp_rows, "hpp_sign": hpp_sign,
            "hpp_where": np.searchsorted(union, hpp_keys),
            "inc_inv": inc_inv, "inc_var": inc_var, "inc_row": inc_row, "n_inc": len(uniq),
            "pair_left": order[left], "pair_right": order[right],
            "pair_depth": inc_row[order[left]],
            "pair_where": np.searchsorted(union, schur_keys),
            "union_keys": union,
        }
        return self._maps


# ---------------------------------------------------------------------------
# residuals / objective (ba.py:219-253)


def _gather(problem, state, lo, hi):
    st = problem.structure()
    q, t, d = state
    rot = quat_to_rot(q)
    s, j = st["src"][lo:hi], st["dst"][lo:hi]
    return st["rays"][lo:hi], d[st["depth_row"][lo:hi]], rot[s], t[s], rot[j], t[j]


def residuals(problem, state=None):
    st = problem.structure()
    state = problem.state() if state is None else state
    e = len(problem.edge_indices)
    res = np.empty((e, st["target"].shape[1] if e else 0, 2))
    valid = np.empty(res.shape[:2], dtype=bool)
    for lo in range(0, e, CHUNK):
        hi = min(lo + CHUNK, e)
        pix, ok = reproject(*_gather(problem, state, lo, hi), problem.g["intr"])
        res[lo:hi] = pix - st["target"][lo:hi]
        valid[lo:hi] = ok
    return res, valid


def objective(problem, state=None) -> float:
    res, valid = residuals(problem, state)
    w = problem.structure()["weight"][:, None, :] * valid[..., None]
    return float(np.sum(w * res * res))


# ---------------------------------------------------------------------------
# assembly (ba.py:260-440)


def scatter_sum(idx, values, size):
    """np.bincount scatter (ba.py:260-269)."""
    values = np.asarray(values, dtype=float)
    flat = values.reshape(len(values), -1)
    k = flat.shape[1]
    comp = (np.asarray(idx, dtype=np.int64)[:, None] * k + np.arange(k)).ravel()
    return np.bincount(comp, weights=flat.ravel(), minlength=size * k).reshape(
        (size,) + values.shape[1:])


@dataclass
class OracleSystem:
    """ba.BlockSparseSystem restated (ba.py:272-325)."""
    n_pose: int
    n_depth: int
    pair_keys: np.ndarray
    pose_blocks: np.ndarray
    schur_blocks: np.ndarray
    depth_diag: np.ndarray
    rhs_pose: np.ndarray
    rhs_depth: np.ndarray
    rhs_schur: np.ndarray
    inc_var: np.ndarray
    inc_row: np.ndarray
    inc_block: np.ndarray
    active: np.ndarray
    damping: float = LAMBDA_INIT
    scale_pin: tuple | None = None
    gradient_norm: float = 0.0

    @property
    def unconstrained_depths(self) -> int:
        return int((~self.active).sum())

    def cinv(self, lam):
        return np.where(self.active, 1.0 / (self.depth_diag * (1.0 + lam) + ~self.active), 0.0)

    def reduced_system(self, lam):
        """S = H - E C^-1 E^T / (1+lam) with multiplicative diagonal damping and scale pin."""
        blocks = self.pose_blocks - self.schur_blocks / (1.0 + lam)
        diag = self.pair_keys[:, 0] == self.pair_keys[:, 1]
        di = np.arange(6)
        dsel = np.nonzero(diag)[0]
        blocks[dsel[:, None], di[None, :], di[None, :]] += \
            lam * self.pose_blocks[dsel[:, None], di[None, :], di[None, :]]
        if self.scale_pin is not None:
            var, u = self.scale_pin
            hit = np.nonzero(diag & (self.pair_keys[:, 0] == var))[0]
            if len(hit):
                b = blocks[hit[0]]
                mu = 1e6 * max(1.0, float(np.abs(np.diagonal(b)).max()))
                b[:3, :3] += mu * np.outer(u, u)
        rhs = self.rhs_pose - self.rhs_schur / (1.0 + lam)
        return self.pair_keys, blocks, rhs, self.cinv(lam)

    def back_substitute(self, dp, lam):
        coupled = (self.inc_block * dp[self.inc_var]).sum(-1)
        return self.cinv(lam) * (self.rhs_depth - scatter_sum(self.inc_row, coupled, self.n_depth))


def edge_terms(problem, state, lo, hi):
    """Per-edge whitened Gram terms (ba.py:349-366)."""
    st = problem.structure()
    pix, ok, jp, jd = reproject(*_gather(problem, state, lo, hi), problem.g["intr"],
                                jacobians=True)
    res = pix - st["target"][lo:hi]
    sw = np.sqrt(st["weight"][lo:hi][:, None, :] * ok[..., None])
    ne, m = ok.shape
    jw = (jp * sw[..., None]).reshape(ne, 2 * m, 6)
    rw = (res * sw).reshape(ne, 2 * m)
    jdw = (jd * sw).reshape(ne, 2 * m)
    hpp = np.einsum("eri,erj->eij", jw, jw)
    e_pd = np.einsum("eri,er->ei", jw, jdw)
    c_dd = np.einsum("er,er->e", jdw, jdw)
    g_p = np.einsum("eri,er->ei", jw, rw)
    g_d = np.einsum("er,er->e", jdw, rw)
    return hpp, e_pd, c_dd, g_p, g_d


def assemble(problem, state=None) -> OracleSystem:
    """ba.py:328-440."""
    st = problem.structure()
    state = problem.state() if state is None else state
    q, t, d = state
    nf, nd = problem.n_free, problem.n_depth
    e = len(problem.edge_indices)
    hpp = np.zeros((e, 6, 6))
    e_pd = np.zeros((e, 6))
    c_dd = np.zeros(e)
    g_p = np.zeros((e, 6))
    g_d = np.zeros(e)
    for lo in range(0, e, CHUNK):
        hi = min(lo + CHUNK, e)
        hpp[lo:hi], e_pd[lo:hi], c_dd[lo:hi], g_p[lo:hi], g_d[lo:hi] = \
            edge_terms(problem, state, lo, hi)
    mp = problem.maps()
    row = st["depth_row"]
    depth_diag = scatter_sum(row, c_dd, nd)
    rhs_depth = -scatter_sum(row, g_d, nd)
    active = depth_diag > ACTIVE_EPS
    rhs_pose = np.zeros((nf, 6))
    rhs_pose += scatter_sum(mp["vi"][mp["rows_i"]], -g_p[mp["rows_i"]], nf)
    rhs_pose += scatter_sum(mp["vj"][mp["rows_j"]], g_p[mp["rows_j"]], nf)
    union = mp["union_keys"]
    w = len(union)
    pose_blocks = np.zeros((w, 6, 6))
    vals = hpp[mp["hpp_rows"]] * mp["hpp_sign"][:, None, None]
    for lo in range(0, len(vals), CHUNK * 4):
        hi = min(lo + CHUNK * 4, len(vals))
        pose_blocks += scatter_sum(mp["hpp_where"][lo:hi], vals[lo:hi], w)
    if mp["n_inc"]:
        inc_vals = np.concatenate([e_pd[mp["rows_i"]], -e_pd[mp["rows_j"]]])
        inc_block = scatter_sum(mp["inc_inv"], inc_vals, mp["n_inc"])
    else:
        inc_block = np.zeros((0, 6))
    cinv0 = np.where(active, 1.0 / (depth_diag + ~active), 0.0)
    schur_blocks = np.zeros((w, 6, 6))
    left, right, gi = mp["pair_left"], mp["pair_right"], mp["pair_depth"]
    for lo in range(0, len(left), CHUNK * 4):
        hi = min(lo + CHUNK * 4, len(left))
        contrib = (inc_block[left[lo:hi]] * cinv0[gi[lo:hi], None])[:, :, None] \
            * inc_block[right[lo:hi]][:, None, :]
        schur_blocks += scatter_sum(mp["pair_where"][lo:hi], contrib, w)
    inc_var, inc_row = mp["inc_var"], mp["inc_row"]
    if len(inc_var):
        rhs_schur = scatter_sum(inc_var, inc_block * (cinv0[inc_row] * rhs_depth[inc_row])[:, None], nf)
    else:
        rhs_schur = np.zeros((nf, 6))
    pin = None
    if problem.scale_degenerate and nf > 0:
        ref = t[problem.touched_fixed[0]] if len(problem.touched_fixed) else np.zeros(3)
        u = t[problem.first_free] - ref
        nrm = np.linalg.norm(u)
        if nrm > 1e-9:
            pin = (0, u / nrm)
    grad = float(max(np.abs(rhs_pose).max(initial=0.0),
                     np.abs(rhs_depth[active]).max(initial=0.0)))
    return OracleSystem(nf, nd, np.stack([union // max(nf, 1), union % max(nf, 1)], axis=1),
                        pose_blocks, schur_blocks, depth_diag, rhs_pose, rhs_depth, rhs_schur,
                        inc_var, inc_row, inc_block, active, problem.damping, pin, grad)


# ---------------------------------------------------------------------------
# solvers (ba.py:447-490; block_cholesky.py:21-111)


def select_backend(problem, threshold=THRESHOLD):
    return DENSE if problem.n_free <= threshold else BLOCK_SPARSE


def solve_dense(system: OracleSystem, lam=None):
    """ba.py:451-472 (LAPACK potrf/potrs through scipy)."""
    lam = system.damping if lam is None else lam
    keys, blocks, rhs, _ = system.reduced_system(lam)
    n = system.n_pose
    t0 = time.perf_counter()
    full = np.zeros((6 * n, 6 * n))
    for (a, b), blk in zip(keys, blocks):
        full[6 * a:6 * a + 6, 6 * b:6 * b + 6] = blk
        if a != b:
            full[6 * b:6 * b + 6, 6 * a:6 * a + 6] = blk.T
    try:
        cho = scipy.linalg.cho_factor(full, check_finite=False)
    except (scipy.linalg.LinAlgError, ValueError) as exc:
        raise OracleSingular(f"dense factorization failed: {exc}") from exc
    t1 = time.perf_counter()
    dp = scipy.linalg.cho_solve(cho, rhs.ravel(), check_finite=False).reshape(n, 6)
    dd = system.back_substitute(dp, lam)
    t2 = time.perf_counter()
    return dp, dd, {"backend": DENSE, "factorize_s": t1 - t0, "solve_s": t2 - t1,
                    "peak_block_count": n * n}


@dataclass
class OracleFactor:
    n: int
    diag_inv: np.ndarray
    lower: dict = field(default_factory=dict)     # (i, j) i > j -> L_ij
    block_count: int = 0

    def solve(self, rhs):
        """Forward then backward block substitution (block_cholesky.py:31-45)."""
        by_row: dict[int, list] = {}
        by_col: dict[int, list] = {}
        for (i, j), blk in self.lower.items():
            by_row.setdefault(i, []).append((j, blk))
            by_col.setdefault(j, []).append((i, blk))
        y = np.empty_like(rhs)
        for j in range(self.n):
            acc = rhs[j].copy()
            for c, blk in sorted(by_row.get(j, []), key=lambda r: r[0]):
                acc -= blk @ y[c]
            y[j] = self.diag_inv[j] @ acc
        x = np.empty_like(y)
        for j in range(self.n - 1, -1, -1):
            acc = y[j].copy()
            for r, blk in sorted(by_col.get(j, []), key=lambda r: r[0]):
                acc -= blk.T @ x[r]
            x[j] = self.diag_inv[j].T @ acc
        return x


def block_cholesky(keys, blocks, n) -> OracleFactor:
    """Right-looking 6x6-block Cholesky, natural order, dynamic fill
    (block_cholesky.py:48-111).  Missing / non-PD diagonal -> OracleSingular."""
    work = {}
    below = [set() for _ in range(n)]
    for (a, b), blk in zip(np.asarray(keys).tolist(), blocks):
        if a == b:
            work[(a, a)] = np.array(blk, dtype=float)
        else:
            work[(b, a)] = np.array(blk, dtype=float).T.copy()
            below[a].add(b)
    diag_inv = np.empty((n, 6, 6))
    fac = OracleFactor(n, diag_inv)
    count = n
    for j in range(n):
        if (j, j) not in work:
            raise OracleSingular(f"missing diagonal block {j}")
        d = work.pop((j, j))
        try:
            ljj = np.linalg.cholesky(d)
        except np.linalg.LinAlgError as exc:
            raise OracleSingular(f"diagonal block {j} is not positive definite") from exc
        inv = np.linalg.inv(ljj)
        diag_inv[j] = inv
        rows = sorted(below[j])
        if not rows:
            continue
        col = [work.pop((i, j)) @ inv.T for i in rows]
        count += len(rows)
        for i, blk in zip(rows, col):
            fac.lower[(i, j)] = blk
        for p, i in enumerate(rows):
            for qq in range(p + 1):
                k = rows[qq]
                upd = col[p] @ col[qq].T
                if (i, k) in work:
                    work[(i, k)] -= upd
                else:
                    work[(i, k)] = -upd
                    if i != k:
                        below[k].add(i)
    fac.block_count = count
    return fac


def solve_block_sparse(system: OracleSystem, lam=None):
    """ba.py:475-487."""
    lam = system.damping if lam is None else lam
    keys, blocks, rhs, _ = system.reduced_system(lam)
    t0 = time.perf_counter()
    fac = block_cholesky(keys, blocks, system.n_pose)
    t1 = time.perf_counter()
    dp = fac.solve(rhs)
    dd = system.back_substitute(dp, lam)
    t2 = time.perf_counter()
    return dp, dd, {"backend": BLOCK_SPARSE, "factorize_s": t1 - t0, "solve_s": t2 - t1,
                    "peak_block_count": fac.block_count}


BACKENDS = {DENSE: solve_dense, BLOCK_SPARSE: solve_block_sparse}


# ---------------------------------------------------------------------------
# retraction + LM (ba.py:497-605)


@dataclass
class OracleReport:
    iterations: int
    initial_objective: float
    final_objective: float
    backend: str
    iteration_times: list = field(default_factory=list)
    converged: bool = False
    gradient_norm: float = float("inf")
    unconstrained_depths: int = 0
    active_patches: int = 0
    final_damping: float = LAMBDA_INIT
    step_norm: float = float("inf")


def apply_step(q, t, d, dp, dd, problem):
    """Left-multiplicative retraction, first-order translation (ba.py:521-531)."""
    q2, t2, d2 = q.copy(), t.copy(), d.copy()
    fr = problem.free_frames
    dq = exp_rotation(dp[:, 3:])
    q2[fr] = normalize(hamilton(dq, q[fr]))
    t2[fr] = rotate(dq, t[fr]) + dp[:, :3]
    d2 += dd
    np.maximum(d2, INVERSE_DEPTH_FLOOR, out=d2)
    return q2, t2, d2


def lm_solve(problem, max_iterations=50, tolerance=1e-9, backend=None, threshold=THRESHOLD):
    """ba.solve restated (ba.py:534-605); writes the result back into problem.g."""
    chosen = backend or select_backend(problem, threshold)
    solver = BACKENDS[chosen]
    q, t, d = problem.state()
    obj = objective(problem, (q, t, d))
    rep = OracleReport(0, obj, obj, chosen, active_patches=problem.active_patch_count())
    lam = problem.damping
    for _ in range(max_iterations):
        tic = time.perf_counter()
        system = assemble(problem, (q, t, d))
        rep.gradient_norm = system.gradient_norm
        rep.unconstrained_depths = system.unconstrained_depths
        accepted = False
        solved = False
        singular = None
        for _ in range(MAX_ESCALATIONS + 1):
            try:
                dp, dd, _ = solver(system, lam)
            except OracleSingular as exc:
                singular = exc
                lam *= LAMBDA_GROW
                if lam > LAMBDA_MAX:
                    raise
                continue
            solved = True
            cand = apply_step(q, t, d, dp, dd, problem)
            cobj = objective(problem, cand)
            if cobj <= obj * (1 + 1e-12) + 1e-300:
                q, t, d = cand
                obj = min(cobj, obj)
                rep.step_norm = float(np.sqrt((dp ** 2).sum() + (dd ** 2).sum()))
                lam = max(lam * LAMBDA_SHRINK, 1e-12)
                accepted = True
                break
            lam *= LAMBDA_GROW
            if lam > LAMBDA_MAX:
                break
        rep.iteration_times.append(time.perf_counter() - tic)
        if not accepted:
            if singular is not None and not solved:
                raise singular
            break
        rep.iterations += 1
        rep.final_objective = obj
        if system.gradient_norm < tolerance:
            rep.converged = True
            break
    else:
        rep.converged = rep.gradient_norm < tolerance
    if rep.gradient_norm < tolerance:
        rep.converged = True
    rep.final_damping = lam
    problem.damping = lam
    problem.write_back(q, t, d)
    return rep
