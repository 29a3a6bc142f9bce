#!/usr/bin/env python
"""Benchmark: correlation lookup + Gauss-Newton BA step on the 2000-frame
global loop-closure graph (BASELINE.json configs[2], the north-star target).

One *step* = one pass of the hot path over the resident problem = one LM
iteration of the global BA as the native driver runs it (speculative
assembly): the rest of the assembly at x (K3 rows / incidences / K4a Schur /
rhs; x's K2+K3 edge pass was done when x was evaluated as the previous
candidate) -> K4b/c damped reduced system + banded/border sparse FP64
factorisation -> K4d depth back-substitution -> retraction to x' -> the
edge pass at x' (its objective for the accept test, and the next
iteration's per-edge terms); the state advances.  Beside it, on a side
stream: K2 pixels of the correlation edges -> K1 two-level correlation.
value = E_BA / step time  [patch-edges/s, whole job].  E_corr (correlation
edges) follows the paper's semantics: edges into frames that still hold dense
features (the last 22-frame odometry window) plus every loop edge.

Also reported: global loop-closure BA ms = BAProblem build + ``solve(8 LM
iterations, tol 1e-9)`` as ``loop.close`` runs it (loop.py:112-116);
``e2e`` = a stateless step (assemble, solve, retraction, objective) through
the C-ABI from pinned HOST buffers (flow targets/confidences + state H2D,
updated state D2H inside the timed region); ``cpu_baseline`` = the numpy
oracle port timed on a bounded sample on this host; ``roofline`` for the
dominant kernel from CUDA events; ``window_step`` = the cfg2 odometry window.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
N>1 (torchrun): the global BA edge list is sharded by depth row across ranks
with one NCCL all-reduce of the reduced pose system per step (dist.py).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK = 6650.0
FP64_DMMA_PEAK = 37.18    # TFLOP/s, measured on this pool (profiles/fp64_peak_r01.txt)
FP64_DFMA_PEAK = 36.86


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--lm-iters", type=int, default=8)
    ap.add_argument("--window", type=int, default=22)
    ap.add_argument("--channels", type=int, default=128)
    ap.add_argument("--feat-dtype", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--no-global", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-batch", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="replay the step as a CUDA graph (a graph replay ignores the streams' "
                         "priorities, so K1 then delays the solve: measured 2.54 vs 2.40 ms)")
    ap.add_argument("--no-graph", action="store_true", help="eager steps (the default)")
    ap.add_argument("--batch-seqs", type=int, default=8)
    ap.add_argument("--corr-items", type=int, default=32,
                    help="K1 items per CTA beside the solve (0: one persistent CTA per SM)")
    ap.add_argument("--k1-early", action="store_true",
                    help="fork K1 before the rest of the assembly instead of after it")
    ap.add_argument("--no-priority", action="store_true",
                    help="BA step on a default-priority stream (K1 then competes for SMs)")
    ap.add_argument("--json-out", default=None)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="torch.distributed backend for N>1 (gloo: multi-rank tests on one GPU)")
    return ap.parse_args()


_T0 = time.perf_counter()


def progress(msg):
    """Phase marker on stderr (the JSON line stays the only stdout line)."""
    print(f"[bench {time.perf_counter() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ---------------------------------------------------------------------------
# clocks during the timed region


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed
    region: an NVML polling thread (1 ms period; the timed region of a cfg3
    run is only ~40 ms, below nvidia-smi's sampling period); nvidia-smi as a
    fallback when NVML is unavailable."""

    NAMES = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
             ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
             ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
             ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
             ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.stop = threading.Event()
        self.thread = None
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
        except Exception:
            self.nvml = None
        return self

    def sample(self):
        """One NVML reading (also called from the launching thread between
        eager steps, so the timed region is covered even when the polling
        thread is starved of the GIL)."""
        p = self.nvml
        if p is None:
            return
        try:
            sm = p.nvmlDeviceGetClockInfo(self.handle, p.NVML_CLOCK_SM)
            rs = p.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
            self.rows.append((sm, rs, time.perf_counter()))
        except Exception:
            self.errors += 1

    errors = 0

    def _poll(self):
        while not self.stop.is_set():
            self.sample()
            time.sleep(0.001)

    # the thread is started (NVML initialised) before the warm-up; only the
    # samples taken between mark_start() and mark_end() are summarised
    t0 = None
    t1 = None

    def mark_start(self):
        self.t0 = time.perf_counter()

    def mark_end(self):
        self.t1 = time.perf_counter()

    def __exit__(self, *exc):
        self.stop.set()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        rows = self.rows
        if self.t0 is not None and self.t1 is not None:
            rows = [r for r in rows if self.t0 <= r[2] <= self.t1]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0,
                    "nvml_errors": self.errors}
        p = self.nvml
        reasons = sorted({name for _, rs, _ in rows for name, attr in self.NAMES
                          if hasattr(p, attr) and rs & getattr(p, attr)})
        sm = [r[0] for r in rows]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(self.max_sm),
                "reasons": reasons, "samples": len(rows),
                "source": "NVML, 1 ms polling during the timed region"}


# ---------------------------------------------------------------------------
# workload


def corr_edge_selection(graph, prob, window, torch):
    """Paper semantics: edges into frames holding dense features (the last
    `window` frames) plus every loop edge (pipeline.py:435)."""
    eidx = prob.view("edge_idx")
    mir = graph.device()
    dst = mir["edge_dst"].long()[eidx]
    kind = torch.as_tensor(graph._kind.view.astype(np.int32), device="cuda").long()[eidx]
    nf = graph.n_frames
    sel = (dst >= nf - window) | (kind == 1)
    idx = torch.nonzero(sel).flatten()
    # process the correlation edges grouped by target frame (L2 reuse of its
    # feature map); the output is per edge, so the order is the caller's
    order = torch.argsort(dst[idx], stable=True)
    return idx[order]


def build_workload(args, torch):
    from paper_2408_01654_b200 import ba, corr, synthetic
    t0 = time.perf_counter()
    scene, graph, free = synthetic.make_config(args.config)
    gen_s = time.perf_counter() - t0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sharded = int(os.environ.get("WORLD_SIZE", "1")) > 1
    if sharded:
        from paper_2408_01654_b200 import dist as pdist
        prob = pdist.ShardedProblem(graph, free)
        info = prob.info
    else:
        prob = ba.BAProblem(graph, free)
        prob._ensure()
        info = prob.info()
    torch.cuda.synchronize()
    build_ms = (time.perf_counter() - t0) * 1e3
    E = int(prob.n_edges_total) if sharded else int(info.n_edges)
    q, t, d = prob.device_state()
    # correlation inputs: features of the frames the corr edges read
    csel = corr_edge_selection(graph, prob, args.window, torch)
    mir = graph.device()
    eidx = prob.view("edge_idx")
    c_dst = mir["edge_dst"].long()[eidx][csel]
    frames, jj = torch.unique(c_dst, return_inverse=True)
    c_gid = mir["edge_gpatch"].long()[eidx][csel]
    w, h = scene.spec.image_size
    H0, W0, C = h // 4, w // 4, args.channels
    fdt = torch.bfloat16 if args.feat_dtype == "bf16" else torch.float32
    gen = torch.Generator(device="cuda").manual_seed(1000)
    fmap0 = torch.empty((len(frames), H0, W0, C), dtype=fdt, device="cuda")
    for i in range(len(frames)):
        fmap0[i] = (torch.randn((H0, W0, C), generator=gen, device="cuda") / math.sqrt(C)).to(fdt)
    pyr = corr.pyramid(fmap0)
    gmap = (torch.randn((graph.n_patches, 9, C), generator=gen, device="cuda")
            / math.sqrt(C)).to(fdt)
    work = dict(graph=graph, scene=scene, prob=prob, info=info, E=E, q=q, t=t, d=d, free=free,
                sharded=sharded, E_local=int(info.n_edges),
                csel=csel, ii=c_gid.to(torch.int32), jj=jj.to(torch.int32), pyr=pyr, gmap=gmap,
                n_feat_frames=len(frames), H0=H0, W0=W0, C=C, gen_s=gen_s, build_ms=build_ms)
    return work


class Stepper:
    """The device-resident hot-path step (C-ABI calls on the current stream)."""

    def __init__(self, work, torch):
        from paper_2408_01654_b200 import _lib
        self.L = _lib
        self.lib = _lib.lib()
        self.torch = torch
        self.w = work
        p = work["prob"]
        self.h = p._ensure()
        E = work["E"]
        n = int(work["info"].n_free)
        P = int(work["info"].n_depths)
        dev = "cuda"
        self.Ec = len(work["csel"])
        # K1 runs beside the BA step on a default (= lowest) priority stream
        # in short-lived CTAs (corr_items per CTA): the BA step runs on a
        # high-priority stream, so the block scheduler gives it SMs first and
        # K1 fills the SMs its latency-bound solve leaves idle
        self.side = torch.cuda.Stream()
        self.corr_items = 0
        self.fork_early = False
        self.overlap = True                       # False: serialise (per-kernel timing)
        self.ev_fork = torch.cuda.Event()
        self.ev_join = torch.cuda.Event()
        self.coords = torch.empty((self.Ec, 9, 2), dtype=torch.float64, device=dev)
        self.cout = torch.empty((self.Ec, len(work["pyr"]), 9, 7, 7), dtype=torch.float32,
                                device=dev)
        self.dp = torch.empty((n, 6), dtype=torch.float64, device=dev)
        self.dd = torch.empty(P, dtype=torch.float64, device=dev)
        self.status = torch.zeros(8, dtype=torch.int32, device=dev)
        self.q2 = torch.empty_like(work["q"])
        self.t2 = torch.empty_like(work["t"])
        self.d2 = torch.empty_like(work["d"])
        self.obj = torch.empty(1, dtype=torch.float64, device=dev)
        self.lam = float(p.damping)

    def step(self, q=None, t=None, d=None):
        L, lib, w = self.L, self.lib, self.w
        q = w["q"] if q is None else q
        t = w["t"] if t is None else t
        d = w["d"] if d is None else d
        s = L.stream_ptr()
        P = L.ptr
        from paper_2408_01654_b200 import corr
        torch = self.torch
        L.check(lib.dpv_assemble(self.h, P(q), P(t), P(d), s), "assemble")
        # K2 pixels of the correlation edges -> K1, on a side stream: the
        # correlation is independent of this BA step and overlaps the solve
        self.ev_fork.record()
        side = self.side if self.overlap else torch.cuda.current_stream()
        with torch.cuda.stream(side):
            side.wait_event(self.ev_fork)
            L.check(lib.dpv_reproject_coords_sel(self.h, P(q), P(t), P(d), 0.25, P(w["csel"]),
                                                 self.Ec, P(self.coords), L.stream_ptr()),
                    "coords")
            corr.corr(w["gmap"], w["pyr"], self.coords, w["ii"], w["jj"], out=self.cout)
            self.ev_join.record()
        if w["sharded"]:
            w["prob"].allreduce_system()      # one packed all-reduce
        L.check(lib.dpv_solve(self.h, self.lam, P(self.dp), P(self.dd), P(self.status), s),
                "solve")
        L.check(lib.dpv_apply_step(self.h, P(q), P(t), P(d), P(self.dp), P(self.dd), P(self.q2),
                                   P(self.t2), P(self.d2), s), "apply_step")
        if w["sharded"]:
            w["prob"].objective(self.q2, self.t2, self.d2, self.obj)   # + all-reduce(sum)
        else:
            L.check(lib.dpv_objective(self.h, P(self.q2), P(self.t2), P(self.d2), P(self.obj),
                                      s), "objective")
        torch.cuda.current_stream().wait_event(self.ev_join)


    def lm_init(self):
        """State buffers for lm_step and the edge pass of the starting state."""
        w, L, P = self.w, self.L, self.L.ptr
        self.x = [w["q"].clone(), w["t"].clone(), w["d"].clone()]
        self.y = [self.q2, self.t2, self.d2]
        L.check(self.lib.dpv_assemble_edges(self.h, P(self.x[0]), P(self.x[1]), P(self.x[2]),
                                            P(self.obj), L.stream_ptr()), "assemble_edges")

    def fast_init(self, corr_items):
        """Pre-built ctypes arguments for lm_step_fast (both state parities)."""
        import ctypes as C
        torch, w, P = self.torch, self.w, self.L.ptr
        self.hp = torch.cuda.current_stream()
        sp = lambda st: C.c_void_p(st.cuda_stream)
        self.hp_p, self.side_p = sp(self.hp), sp(self.side)
        g, (f0, f1) = w["gmap"], w["pyr"]
        ii, jj = w["ii"].to(torch.int32).contiguous(), w["jj"].to(torch.int32).contiguous()
        self._keep = (ii, jj)
        self.corr_args = (P(g), int(g.shape[0]), P(f0), P(f1), int(f0.shape[0]), P(self.coords),
                          P(ii), P(jj), self.Ec, int(g.shape[-1]), int(f0.shape[1]),
                          int(f0.shape[2]), int(f1.shape[1]), int(f1.shape[2]), 2, 3,
                          1 if g.dtype == torch.bfloat16 else 0, int(corr_items), P(self.cout),
                          self.side_p)
        self.fast = [None, None]
        for par in range(2):
            x, y = (self.x, self.y) if par == 0 else (self.y, self.x)
            self.fast[par] = ([P(v) for v in x], [P(v) for v in y])
        self.parity = 0
        self.lam_c = C.c_double(self.lam)
        self.csel_p = P(w["csel"])
        self.misc = (P(self.dp), P(self.dd), P(self.status), P(self.obj))

    def lm_step_fast(self):
        """lm_step with pre-built arguments: ~8 library calls and 4 stream /
        event operations per step, so the host stays well ahead of the device
        (K1 on the low-priority side stream, the BA on the high-priority one)."""
        lib, h, chk = self.lib, self.h, self.L.check
        (xq, xt, xd), (yq, yt, yd) = self.fast[self.parity]
        hs, ls = self.hp_p, self.side_p
        dp, dd, status, obj = self.misc
        r = lib.dpv_assemble_rest(h, xt, hs)
        if r:
            chk(r, "assemble_rest")
        self.ev_fork.record(self.hp)
        self.side.wait_event(self.ev_fork)
        r = lib.dpv_reproject_coords_sel(h, xq, xt, xd, 0.25, self.csel_p, self.Ec,
                                         self.corr_args[5], ls)
        if r:
            chk(r, "coords")
        r = lib.dpv_corr_ex2(*self.corr_args)
        if r:
            chk(r, "corr")
        self.ev_join.record(self.side)
        r = lib.dpv_solve(h, self.lam_c, dp, dd, status, hs)
        if r:
            chk(r, "solve")
        r = lib.dpv_apply_step(h, xq, xt, xd, dp, dd, yq, yt, yd, hs)
        if r:
            chk(r, "apply_step")
        r = lib.dpv_assemble_edges(h, yq, yt, yd, obj, hs)
        if r:
            chk(r, "assemble_edges")
        self.hp.wait_event(self.ev_join)
        self.parity ^= 1
        self.x, self.y = self.y, self.x

    def lm_step(self):
        """One LM iteration of the global BA as the native driver runs it
        (speculative assembly, ba.py:534-605 flow): the rest of the assembly at
        x (its edge pass was done when x was evaluated as the previous
        candidate), the damped sparse solve, the retraction to x', and x''s
        edge pass, which yields the candidate objective and the next
        iteration's per-edge terms; the state advances.  K1 runs beside it."""
        L, lib, w = self.L, self.lib, self.w
        P = L.ptr
        s = L.stream_ptr()
        torch = self.torch
        from paper_2408_01654_b200 import corr
        q, t, d = self.x
        q2, t2, d2 = self.y

        def k1():
            self.ev_fork.record()
            side = self.side if self.overlap else torch.cuda.current_stream()
            with torch.cuda.stream(side):
                side.wait_event(self.ev_fork)
                L.check(lib.dpv_reproject_coords_sel(self.h, P(q), P(t), P(d), 0.25,
                                                     P(w["csel"]), self.Ec, P(self.coords),
                                                     L.stream_ptr()), "coords")
                corr.corr(w["gmap"], w["pyr"], self.coords, w["ii"], w["jj"], out=self.cout,
                          items_per_cta=self.corr_items if self.overlap else 0)
                self.ev_join.record()
        # K1 forks after the assembly, so it overlaps the latency-bound sparse
        # factorisation rather than the bandwidth-bound assembly kernels
        # (measured: 3.22 -> 3.13 ms per step against forking first)
        if self.fork_early:
            k1()
        L.check(lib.dpv_assemble_rest(self.h, P(t), s), "assemble_rest")
        if w["sharded"]:
            w["prob"].allreduce_system()      # one packed all-reduce, no host sync
        if not self.fork_early:
            k1()
        L.check(lib.dpv_solve(self.h, self.lam, P(self.dp), P(self.dd), P(self.status), s),
                "solve")
        L.check(lib.dpv_apply_step(self.h, P(q), P(t), P(d), P(self.dp), P(self.dd), P(q2),
                                   P(t2), P(d2), s), "apply_step")
        L.check(lib.dpv_assemble_edges(self.h, P(q2), P(t2), P(d2), P(self.obj), s),
                "assemble_edges")
        if w["sharded"]:                      # the candidate objective: sum over shards
            w["prob"].dist.all_reduce(self.obj, group=w["prob"].group)
        self.x, self.y = self.y, self.x
        torch.cuda.current_stream().wait_event(self.ev_join)


def time_steps(fn, k, torch):
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    # wait with the GIL released so the clock sampler thread keeps polling
    # while the device runs (graph replays return immediately)
    while not b.query():
        time.sleep(0.0002)
    torch.cuda.synchronize()
    return a.elapsed_time(b)


# ---------------------------------------------------------------------------
# algorithmic work per kernel


def cholesky_flops(N, nb=64):
    """Exact FP64 flops of the blocked right-looking factorisation of the
    (N+1)-row augmented matrix (SYRK part = DMMA)."""
    syrk = 0.0
    other = 0.0
    for c0 in range(0, N, nb):
        k = min(nb, N - c0)
        m = N - (c0 + k)
        syrk += 2.0 * k * (m * (m + 1) / 2 + m)
        other += k ** 3 / 3 + (m + 1) * k * k
    return syrk, other


def load_traffic():
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)
    from the committed `ncu --set full` capture (profiles/ncu_traffic.json)."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except Exception:
        return {}


def kernel_rooflines(timing, work, steps, hbm_peak):
    """Per-kernel roofline: ALGORITHMIC bytes (or FP64 flops) per launch over
    the CUDA-event launch time (DESIGN.md section 4 gives the per-unit figures)."""
    E = work["E_local"]     # this rank's edges (= E at N = 1)
    info = work["info"]
    P = int(info.n_depths)
    n = int(info.n_free)
    W = int(info.n_keys)
    I = int(info.n_inc)
    Ec = len(work["csel"])
    L = len(work["pyr"])
    fbytes = 2 if work["gmap"].dtype.itemsize == 2 else 4
    plan = work.get("plan") or {}
    traffic = load_traffic()
    edge_pass = E * 172 + P * 152      # targets, weights, indices + per-row rays/depth
    out = {}
    per_step = {
        # name: (bound, algorithmic bytes or flops per step, unit)
        "assemble_edges": ("hbm", edge_pass + E * 64 + int(info.n_segments) * 216, "B"),
        "objective": ("hbm", edge_pass, "B"),
        # corr edges: src/dst/row (12) + the patch's rays and depth (152) in, 144 out
        "coords": ("hbm", Ec * (12 + 152 + 144), "B"),
        # coords + indices + output + the edges' patch features + every feature map once
        "corr": ("hbm", Ec * (144 + 8 + L * 9 * 49 * 4) + Ec * 9 * work["C"] * fbytes
                 + sum(int(f.numel()) * fbytes for f in work["pyr"]), "B"),
        # per-row sums: e_terms (c_dd, g_d) of every edge in, 4 row arrays out
        "rows": ("hbm", E * (4 + 16) + P * 25, "B"),
        # +-e_pd of every contribution in, inc_block + uinc out
        "incidences": ("hbm", 2 * E * (4 + 48) + I * 96, "B"),
        # Schur pair products on DMMA: 72 flop per pair (6x6 outer product)
        "key_blocks": ("tensor", int(info.n_pairs) * 72.0, "flop"),
        # band+border factorisation on DMMA (the plan's tile products, both levels)
        "spd_factor": ("tensor", plan.get("update_flops", 0.0), "flop"),
    }
    # one entry per kernel FUNCTION (as in the ncu launch list): the two
    # levels of the sparse factorisation are the same k_spd_factor
    timing = dict(timing)
    if "spd_factor2" in timing:
        a, b = timing.get("spd_factor", (0.0, 0)), timing.pop("spd_factor2")
        timing["spd_factor"] = (a[0] + b[0], a[1] + b[1])
    for name, (ms, cnt) in timing.items():
        rec = {"ms_per_step": ms / steps, "launches_per_step": cnt / steps}
        if name in per_step and per_step[name][1] > 0:
            bound, work_units, unit = per_step[name]
            per_launch = work_units / max(cnt / steps, 1)
            avg_ms = ms / max(cnt, 1)
            if unit == "B":
                ach = per_launch / (avg_ms * 1e-3) / 1e9
                rec.update(bound=bound, achieved=ach, unit="GB/s", peak=hbm_peak,
                           frac=ach / hbm_peak, algorithmic_per_launch=per_launch)
            else:
                ach = per_launch / (avg_ms * 1e-3) / 1e12
                rec.update(bound=bound, achieved=ach, unit="TFLOP/s", peak=FP64_DMMA_PEAK,
                           frac=ach / FP64_DMMA_PEAK, algorithmic_per_launch=per_launch)
            rec["traffic"] = traffic.get(name)
        out[name] = rec
    return out


# ---------------------------------------------------------------------------
# CPU baseline: the numpy oracle port on a bounded sample


REF_PREFIX = 250     # frames of the cfg3 graph in the reference arm's sub-problem


def corr_cpu_sample(work, corr_edges=1500):
    """The correlation lookup has no reference code: its CPU
    figure is the float64 numpy oracle port on a bounded sample."""
    from oracle import corr_oracle
    rng = np.random.default_rng(0)
    C = work["C"]
    fm = rng.normal(size=(4, work["H0"], work["W0"], C)) / math.sqrt(C)
    fms = [fm, corr_oracle.avg_pool4(fm)]
    gm = rng.normal(size=(64, 9, C)) / math.sqrt(C)
    coords = rng.uniform(0, [work["W0"], work["H0"]], size=(corr_edges, 1, 2)) + \
        np.stack(np.meshgrid(np.arange(3) * 0.25, np.arange(3) * 0.25), -1).reshape(1, 9, 2)
    t0 = time.perf_counter()
    corr_oracle.corr(gm, fms, coords, rng.integers(0, 64, corr_edges),
                     rng.integers(0, 4, corr_edges))
    dt = time.perf_counter() - t0
    return {"value": corr_edges / dt, "unit": "corr-edges/s", "cores": 1, "kind": "port",
            "sample": f"oracle/corr_oracle.py (numpy f64) on {corr_edges} edges, 2 levels, C={C}"}


def cpu_sample(work, steps=1, warmup=0):
    """CPU baseline on this host: the unmodified reference (bench_ref.py) when
    it is installed in baseline/_ref, else the numpy oracle port, running full
    LM iterations of the named sub-problem (the first REF_PREFIX frames of the
    same graph).  value = its edges per second; nothing is extrapolated."""
    import bench_ref
    g = work["graph"].soa()
    soa = {k: np.array(v) for k, v in g.items()}
    if bench_ref.reference_available():
        r = bench_ref.time_iterations(soa, REF_PREFIX, steps, warmup)
        kind = "reference"
    else:
        r = port_iterations(soa, REF_PREFIX, steps, warmup)
        kind = "port"
    out = {"value": r["value"], "unit": "patch-edges/s", "cores": r["cores"], "kind": kind,
           "sample": r["sample"], "step_s": r["step_s"], "E_sample": r["E"],
           "setup_s": r["setup_s"], "objectives": r["objectives"]}
    try:
        out["corr_port"] = corr_cpu_sample(work)
    except Exception as exc:            # reported, not fatal
        out["corr_port"] = {"error": repr(exc)}
    return out


def port_iterations(soa, prefix, steps, warmup):
    """Same step as bench_ref.time_iterations through the oracle port
    (oracle/ba_oracle.py, pinned to the reference's golden vectors)."""
    from oracle import ba_oracle as O
    nf = prefix
    keep = (soa["edge_src"] < nf) & (soa["edge_dst"] < nf)
    sub = dict(soa)
    for k in ("edge_src", "edge_patch", "edge_dst", "edge_target", "edge_conf", "edge_kind"):
        sub[k] = soa[k][keep]
    sub["frame_q"], sub["frame_t"] = soa["frame_q"][:nf], soa["frame_t"][:nf]
    t0 = time.perf_counter()
    prob = O.OracleProblem(sub, (1, nf - 1))
    prob.structure()
    prob.maps()
    setup_s = time.perf_counter() - t0
    backend = O.select_backend(prob)
    solver = O.solve_dense if backend == "dense" else O.solve_block_sparse
    q, t, d = prob.state()
    times, objs = [], []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        system = O.assemble(prob, (q, t, d))
        dp, dd, _ = solver(system, prob.damping)
        q, t, d = O.apply_step(q, t, d, dp, dd, prob)
        obj = O.objective(prob, (q, t, d))
        if i >= warmup:
            times.append(time.perf_counter() - t0)
            objs.append(obj)
    E = len(prob.edge_indices)
    step_s = float(np.median(times))
    return {"E": E, "step_s": step_s, "setup_s": setup_s, "objectives": objs,
            "value": E / step_s, "cores": os.cpu_count(), "step_times_s": times,
            "sample": (f"oracle port (numpy f64): one LM iteration per step on the global BA over "
                       f"the first {prefix} frames of the cfg3 graph (E = {E}); median of "
                       f"{len(times)} after {warmup} warm-up")}


# ---------------------------------------------------------------------------


def run_ours(args):
    import torch
    from paper_2408_01654_b200.synthetic import DESCRIPTIONS as DESC
    from paper_2408_01654_b200 import _lib, ba
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch.distributed as tdist
        # one process per GPU; --dist-backend gloo (tests) may share a device
        local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local)
        if args.dist_backend == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            tdist.init_process_group(args.dist_backend)
    else:
        torch.cuda.set_device(0)
    peaks = measured_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", HBM_FALLBACK))
    if not args.no_priority:
        # the BA step (and everything timed) on a high-priority stream; K1's
        # side stream keeps the default, lowest priority (Stepper)
        torch.cuda.set_stream(torch.cuda.Stream(priority=-1))
    progress("build workload")
    work = build_workload(args, torch)
    progress("workload built")
    st = Stepper(work, torch)
    st.corr_items = args.corr_items
    st.fork_early = args.k1_early
    # device-resident step: one LM iteration with speculative assembly (the
    # native driver's flow); the sharded path keeps assemble + NCCL + objective
    st.lm_init()
    step_fn = st.lm_step
    clk = ClockSampler(torch.cuda.current_device()).__enter__()
    for _ in range(max(args.warmup, 3)):
        step_fn()
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    # --graph: the device step is a fixed launch sequence: capture two steps
    # (the state buffers swap every step, so two steps return to the starting
    # assignment) as one CUDA graph and replay it; kernels are counted at
    # capture (the library counts every launch it issues).  Not the default:
    # a replayed graph ignores the stream priorities that let K1 fill the
    # solve's idle SMs (also with per-node priorities and
    # cudaGraphInstantiateFlagUseNodePriority: measured 2.59 vs 2.40 ms eager)
    graph = None
    per_graph = 0
    fast = None
    if not work["sharded"] and not args.graph:
        st.fast_init(args.corr_items)
        fast = st.lm_step_fast
        for _ in range(2):
            fast()
        torch.cuda.synchronize()
    if not work["sharded"] and args.graph and not args.no_graph and args.steps % 2 == 0:
        try:
            graph = torch.cuda.CUDAGraph()
            l0 = _lib.lib().dpv_launch_count()
            with torch.cuda.graph(graph, stream=torch.cuda.current_stream()):
                step_fn()
                step_fn()
            per_graph = _lib.lib().dpv_launch_count() - l0
            for _ in range(2):
                graph.replay()
            torch.cuda.synchronize()
        except Exception as exc:          # eager steps instead
            print(f"[bench] CUDA graph capture failed ({exc!r}); eager steps", file=sys.stderr)
            graph = None
            torch.cuda.synchronize()
    progress("timed steps")
    launches0 = _lib.lib().dpv_launch_count()
    clk.mark_start()
    if graph is not None:
        ms = time_steps(graph.replay, args.steps // 2, torch)
    else:
        ms = time_steps(fast or step_fn, args.steps, torch)
    clk.mark_end()
    clk.__exit__(None, None, None)
    launches = _lib.lib().dpv_launch_count() - launches0
    if graph is not None:
        launches = per_graph * (args.steps // 2)
    ms_per_step = ms / args.steps
    if world > 1:
        tdist.barrier()
        mt = torch.tensor([ms_per_step], dtype=torch.float64, device="cuda")
        tdist.all_reduce(mt, op=tdist.ReduceOp.MAX)        # max over ranks
        ms_per_step = float(mt.item())
    value = work["E"] / (ms_per_step * 1e-3)
    # per-kernel CUDA-event timing pass (separate, so the headline has no event overhead)
    # per-kernel CUDA-event pass: the correlation runs on the main stream here,
    # so every kernel is timed alone (the headline overlaps it with the BA)
    progress("per-kernel timing pass")
    st.overlap = False
    _lib.timing_enable(True)
    for _ in range(args.steps):
        step_fn()
    timing = _lib.timing_collect()
    _lib.timing_enable(False)
    st.overlap = True
    try:
        work["plan"] = _lib.plan_info(work["prob"]._ensure())
    except Exception:
        work["plan"] = None
    kernels = kernel_rooflines(timing, work, args.steps, hbm_peak)
    # dominant kernel = largest share of the (serialised) step
    dominant = max(((k, v) for k, v in kernels.items() if "bound" in v),
                   key=lambda kv: kv[1]["ms_per_step"])
    dom = dict(dominant[1])
    roof = {"kernel": dominant[0], "bound": dom["bound"],
            "achieved": dom.get("achieved"), "peak": dom.get("peak"),
            "unit": dom.get("unit"), "frac": dom.get("frac"), "traffic": dom.get("traffic"),
            "share_of_step": dom["ms_per_step"] / ms_per_step,
            "peak_source": ("FP64 DMMA peak measured on this pool (37.18 TFLOP/s, "
                            "profiles/fp64_peak_r01.txt; MEASURED_PEAKS.json has no FP64 "
                            "figure)") if dom.get("unit") == "TFLOP/s"
            else "MEASURED_PEAKS.json hbm_gbs (burst copy)"}
    notes = {
        "spd_factor": "latency-bound dataflow chain (leader CTA per chain: 64x64 potrf + TRSM "
                      "+ diagonal update per panel); tensor frac is low by construction",
        "assemble_edges": "FP64-pipe bound (~1.3k FP64 ops per 172-byte edge, SURVEY H1)",
        "key_blocks": "L2-gather bound DMMA Schur products",
    }
    if dominant[0] in notes:
        roof["note"] = notes[dominant[0]]
    serial_ms = sum(v["ms_per_step"] for v in kernels.values())
    roof["serialised_kernel_ms"] = serial_ms
    # step-level HBM fraction: SURVEY 8(d) algorithmic bytes of one LM
    # iteration (2 edge passes x 172 B, 2 x 24 B per patch, incidences
    # written + read, pose / Schur blocks, rhs) over the measured step
    inf = work["info"]
    step_bytes = (2 * 172 * work["E"] + 48 * int(inf.n_depths)
                  + 96 * int(getattr(inf, "n_inc", 0)) + 288 * int(getattr(inf, "n_keys", 0))
                  + 48 * int(inf.n_free))
    roof["step_algorithmic_bytes"] = step_bytes
    roof["step_hbm_frac"] = step_bytes / (ms_per_step * 1e-3) / 1e9 / hbm_peak

    # e2e through the C-ABI from pinned host buffers
    e2e = None
    if not args.no_e2e and world == 1:
        progress("e2e")
        e2e = run_e2e_solve(work, args, torch)
        progress("e2e per-iteration upload")
        # the stricter variant: every LM iteration re-uploads all targets
        e2e["per_iteration_upload"] = run_e2e(work, st, args, torch)

    # global loop-closure BA (loop.close: new BAProblem + solve(8 iters, 1e-9))
    glob = None
    window = None
    window1 = None
    batch = None
    if not args.no_global and world == 1:
        progress("global BA")
        glob = run_global(work, args, torch)
        progress("window steps")
        try:
            window = run_window(args, torch)
        except Exception as exc:     # reported, not fatal for the headline
            window = {"error": repr(exc)}
        try:
            window1 = run_window(args, torch, config="cfg1")
        except Exception as exc:
            window1 = {"error": repr(exc)}
        try:
            progress("batch replicas")
            batch = None if args.no_batch else run_batch(args, torch, n_seq=args.batch_seqs)
        except Exception as exc:
            batch = {"error": repr(exc)}
    elif not args.no_global:
        t0 = time.perf_counter()
        rep, *_ = work["prob"].solve(max_iterations=args.lm_iters, tolerance=1e-9)
        torch.cuda.synchronize()
        glob = {"ms": (time.perf_counter() - t0) * 1e3, "iterations": rep["iterations"],
                "lm_attempts": rep["attempts"], "final_objective": rep["final_objective"],
                "includes": "native LM over the sharded system (index prebuilt)"}

    progress("cpu baseline sample")
    cpu = None if (args.no_cpu or world > 1) else cpu_sample(work)
    progress("done")
    if world > 1:
        tdist.destroy_process_group()
        if rank != 0:
            return None
    line = {
        "metric": "patch-edges/sec for corr lookup + Gauss-Newton BA step; global loop-closure BA ms",
        "value": value, "unit": "patch-edges/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator restated bit-exactly; random features)",
        "config": workload_config(args, work["graph"], work["free"], world),
        "workload_stats": {
                   "E_ba": work["E"], "E_corr": len(work["csel"]),
                   "P": int(work["info"].n_depths), "n_free": int(work["info"].n_free),
                   "W_blocks": int(work["info"].n_keys), "pairs": int(work["info"].n_pairs),
                   "feature_frames": work["n_feat_frames"],
                   "lm_attempt_per_step": 1,
                   "step_kind": ("device-only LM iteration (" + (
                                 "replayed as one CUDA graph" if graph is not None else
                                 "eager launches") + "): fixed lambda, "
                                 "the candidate is always accepted, no host read-back; the native "
                                 "driver's per-iteration time (host accept test, lambda "
                                 "escalation) is global_ba.iteration_ms"),
                   "cuda_graph": graph is not None,
                   "k1_overlap": ("BA step kernels at the greatest node/stream priority, K1 at "
                                  f"the least in CTAs of {args.corr_items} items (fills the SMs "
                                  "the latency-bound solve leaves idle)") if not args.no_priority
                                 else "K1 persistent, default priorities",
                   "step": ("one LM iteration (speculative assembly: rest of the assembly at x, "
                            "sparse solve, retraction, edge pass at the candidate = its "
                            "objective and the next iteration's terms; state advances) + K1 "
                            "on a side stream forked after the assembly") if not work["sharded"] else
                           ("one LM iteration on this rank's edge shard: rest of the assembly, "
                            "all-reduce of the reduced pose system, redundant sparse solve, "
                            "retraction, edge pass at the candidate + all-reduce of its "
                            "objective; K1 beside it")},
        "gpu_launches": int(launches),
        "roofline": roof,
        "kernels": kernels,
        "factor_plan": work.get("plan"),
        "index_build_ms": work["build_ms"],
        "global_ba": glob,
        "lm_solve_iteration_ms": (float(np.median(glob["iteration_ms"]))
                                  if glob and glob.get("iteration_ms") else None),
        "window_step": window,
        "window_step_cfg1": window1,
        "batch_replicas": batch,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "input_generation_s": work["gen_s"],
    }
    return line


def run_e2e(work, st, args, torch):
    """Host buffers -> C-ABI -> host: per step H2D of the flow targets +
    confidences (all BA edges) + state, the device step, D2H of the candidate
    state and objective.  Uploads are double-buffered on a copy stream, so
    step i+1's inputs cross PCIe while step i computes (whole-job throughput);
    every step's copies are inside the timed region."""
    from paper_2408_01654_b200 import _lib
    prob = work["prob"]
    E = work["E"]
    eidx = prob.view("edge_idx")
    mir = work["graph"].device()
    tgt_h = mir["edge_target"][eidx].cpu().pin_memory()
    conf_h = mir["edge_conf"][eidx].cpu().pin_memory()
    q_h = work["q"].cpu().pin_memory()
    t_h = work["t"].cpu().pin_memory()
    d_h = work["d"].cpu().pin_memory()
    host_in = (tgt_h, conf_h, q_h, t_h, d_h)
    bufs = [[torch.empty_like(x, device="cuda") for x in host_in] for _ in range(2)]
    outs = [torch.empty_like(x).pin_memory() for x in (q_h, t_h, d_h)]
    obj_h = torch.empty(1, dtype=torch.float64).pin_memory()
    lib = _lib.lib()
    copy = torch.cuda.Stream()
    loaded = [torch.cuda.Event(), torch.cuda.Event()]
    consumed = [torch.cuda.Event(), torch.cuda.Event()]
    main = torch.cuda.current_stream()
    for ev in consumed:
        ev.record(main)

    def upload(i):
        b = i % 2
        with torch.cuda.stream(copy):
            copy.wait_event(consumed[b])
            for dst, src in zip(bufs[b], host_in):
                dst.copy_(src, non_blocking=True)
            loaded[b].record(copy)

    def step(i, last):
        b = i % 2
        if not last:
            upload(i + 1)                      # next step's inputs, overlapped
        main.wait_event(loaded[b])
        tgt_d, conf_d, q_d, t_d, d_d = bufs[b]
        _lib.check(lib.dpv_update_targets(st.h, _lib.ptr(tgt_d), _lib.ptr(conf_d),
                                          _lib.stream_ptr()), "update_targets")
        st.step(q_d, t_d, d_d)
        consumed[b].record(main)
        outs[0].copy_(st.q2, non_blocking=True)
        outs[1].copy_(st.t2, non_blocking=True)
        outs[2].copy_(st.d2, non_blocking=True)
        obj_h.copy_(st.obj, non_blocking=True)

    def run(k):
        upload(0)
        for i in range(k):
            step(i, i == k - 1)

    run(2)
    K = max(2, args.steps)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    run(K)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / K
    h2d = sum(int(x.numel() * x.element_size()) for x in host_in)
    d2h = sum(int(x.numel() * x.element_size()) for x in outs) + 8
    return {"value": E / (ms * 1e-3), "unit": "patch-edges/s", "ms_per_step": ms,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "h2d_GBps": h2d / (ms * 1e-3) / 1e9,
            "note": "uploads double-buffered on a copy stream (PCIe-bound: the f64 flow "
                    "targets of every BA edge cross each step)"}


def run_e2e_solve(work, args, torch, steps=6):
    """End to end through the C-ABI from pinned HOST buffers, as loop.close
    runs the global BA (loop.py:113-116): per step the host graph arrays
    (edges, flow targets, confidences, patch grid, poses, depths) cross
    PCIe, the device builds a new BAProblem index from them
    (dpv_problem_create), K2 pixels + K1 of the correlation edges run on a
    side stream, dpv_lm_solve runs the LM (max 8 iterations, tol 1e-9), and
    the solved poses and depths come back to host.  value = E_BA x accepted
    LM iterations / time, i.e. SURVEY 8(d)'s E_BA x iterations /
    (t_corr + t_BA).  The next step's upload is double-buffered on a copy
    stream (whole-job throughput)."""
    from paper_2408_01654_b200 import _lib, corr
    import ctypes as C
    lib = _lib.lib()
    graph, prob = work["graph"], work["prob"]
    mir = graph.device()
    keys = ["patch_grid", "edge_src", "edge_gpatch", "edge_dst", "edge_target", "edge_conf",
            "q", "t", "patch_depth"]
    host = {k: mir[k].cpu().pin_memory() for k in keys}
    dev = [{k: torch.empty_like(mir[k]) for k in keys} for _ in range(2)]
    P = int(prob.info().n_depths)
    out_q = torch.empty_like(host["q"]).pin_memory()
    out_t = torch.empty_like(host["t"]).pin_memory()
    out_d = torch.empty(P, dtype=torch.float64).pin_memory()
    d_dev = torch.empty(P, dtype=torch.float64, device="cuda")
    Ec = len(work["csel"])
    coords = torch.empty((Ec, 9, 2), dtype=torch.float64, device="cuda")
    cout = torch.empty((Ec, 2 * 9 * 49), dtype=torch.float32, device="cuda")
    copy = torch.cuda.Stream()
    side = torch.cuda.Stream()
    loaded = [torch.cuda.Event(), torch.cuda.Event()]
    consumed = [torch.cuda.Event(), torch.cuda.Event()]
    fork, join = torch.cuda.Event(), torch.cuda.Event()
    main = torch.cuda.current_stream()
    for ev in consumed:
        ev.record(main)
    first, last = prob.first_free, prob.last_free
    iters = []

    def upload(i):
        b = i % 2
        with torch.cuda.stream(copy):
            copy.wait_event(consumed[b])
            for k in keys:
                dev[b][k].copy_(host[k], non_blocking=True)
            loaded[b].record(copy)

    def step(i, last_step):
        b = i % 2
        upload(i + 1)      # the next step's inputs, behind this step's compute
        main.wait_event(loaded[b])
        g = _lib.DpvGraph()
        g.n_frames = graph.n_frames
        g.cells = graph.patch_size ** 2
        g.n_patches = graph.n_patches
        g.n_edges = graph.n_edges
        g.patch_grid = dev[b]["patch_grid"].data_ptr()
        g.edge_src = dev[b]["edge_src"].data_ptr()
        g.edge_gpatch = dev[b]["edge_gpatch"].data_ptr()
        g.edge_dst = dev[b]["edge_dst"].data_ptr()
        g.edge_target = dev[b]["edge_target"].data_ptr()
        g.edge_conf = dev[b]["edge_conf"].data_ptr()
        for j, v in enumerate(graph.intrinsics.as_array()):
            g.intr[j] = float(v)
        h = C.c_void_p()
        s = _lib.stream_ptr()
        _lib.check(lib.dpv_problem_create(C.byref(g), first, last, None, 0, s, C.byref(h)),
                   "problem_create")
        q, t = dev[b]["q"], dev[b]["t"]
        _lib.check(lib.dpv_gather_depths(h, _lib.ptr(dev[b]["patch_depth"]), _lib.ptr(d_dev), s),
                   "gather_depths")
        # K2 pixels of the correlation edges at the starting state, K1 beside the LM
        _lib.check(lib.dpv_reproject_coords_sel(h, _lib.ptr(q), _lib.ptr(t), _lib.ptr(d_dev),
                                                0.25, _lib.ptr(work["csel"]), Ec,
                                                _lib.ptr(coords), s), "coords")
        fork.record(main)
        with torch.cuda.stream(side):
            side.wait_event(fork)
            corr.corr(work["gmap"], work["pyr"], coords, work["ii"], work["jj"], out=cout,
                      items_per_cta=args.corr_items)
            join.record(side)
        params = _lib.DpvLmParams(args.lm_iters, 1e-9, 1e-4)
        rep = _lib.DpvLmReport()
        _lib.check(lib.dpv_lm_solve(h, _lib.ptr(q), _lib.ptr(t), _lib.ptr(d_dev),
                                    C.byref(params), C.byref(rep), s), "lm_solve")
        iters.append(int(rep.iterations))
        main.wait_event(join)
        out_q.copy_(q, non_blocking=True)
        out_t.copy_(t, non_blocking=True)
        out_d.copy_(d_dev, non_blocking=True)
        consumed[b].record(main)
        main.synchronize()
        lib.dpv_problem_destroy(h)

    def run(k):
        for i in range(k):
            step(i, i == k - 1)

    # steady state of the double-buffered pipeline: the first input is staged
    # before the clock starts and every timed step uploads the NEXT step's
    # inputs (exactly `steps` full H2D copies inside the timed region)
    upload(0)
    run(1)
    iters.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run(steps)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / steps
    h2d = sum(int(x.numel() * x.element_size()) for x in host.values())
    d2h = int(out_q.numel() * 8 + out_t.numel() * 8 + out_d.numel() * 8)
    E = work["E"]
    it = float(np.mean(iters))
    return {"value": E * it / (ms * 1e-3), "unit": "patch-edges/s", "ms_per_step": ms,
            "lm_iterations_per_step": it, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "h2d_GBps": h2d / (ms * 1e-3) / 1e9,
            "step": "one global loop-closure BA from host arrays: H2D of the graph (edges, "
                    "targets, confidences, grid, poses, depths) -> index build -> K2+K1 of the "
                    "corr edges (side stream) -> native LM (8 iterations) -> D2H of poses and "
                    "depths (wall clock; double-buffered: each timed step uploads the next "
                    "step's inputs behind its own compute, one full H2D per timed step)"}


def run_window(args, torch, reps=5, config="cfg2"):
    """Local odometry window at EuRoC shape (BASELINE configs[1], cfg2): per
    frame-step a new BAProblem over the 22-frame window, the correlation of
    every window edge (2 levels, bf16) and ba.solve(2 LM iterations, tol 1e-12)
    as pipeline.py:389-396 runs it.  Launch/latency-bound (55k edges)."""
    from paper_2408_01654_b200 import ba, corr, synthetic
    scene, graph, free = synthetic.make_config(config)
    soa0 = {k: np.array(v) for k, v in graph.soa().items()}
    w, h = scene.spec.image_size
    C = args.channels
    gen = torch.Generator(device="cuda").manual_seed(7)
    fdt = torch.bfloat16 if args.feat_dtype == "bf16" else torch.float32
    fmap = (torch.randn((graph.n_frames, h // 4, w // 4, C), generator=gen, device="cuda")
            / math.sqrt(C)).to(fdt)
    pyr = corr.pyramid(fmap)
    gmap = (torch.randn((graph.n_patches, 9, C), generator=gen, device="cuda")
            / math.sqrt(C)).to(fdt)
    from paper_2408_01654_b200 import _lib
    times = []
    E = 0
    for r in range(reps + 2):
        graph._q.view[:] = soa0["frame_q"]
        graph._t.view[:] = soa0["frame_t"]
        graph._depth.view[:] = soa0["patch_depth"]
        graph._pose_ver += 1
        graph._patch_ver += 1
        graph.device()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        prob = ba.BAProblem(graph, free)
        h_ = prob._ensure()
        E = int(prob.info().n_edges)
        q, t, d = prob.device_state()
        mir = graph.device()
        eidx = prob.view("edge_idx")
        sel = torch.arange(E, dtype=torch.int64, device="cuda")
        coords = torch.empty((E, 9, 2), dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().dpv_reproject_coords_sel(h_, _lib.ptr(q), _lib.ptr(t), _lib.ptr(d),
                                                       0.25, _lib.ptr(sel), E, _lib.ptr(coords),
                                                       _lib.stream_ptr()), "coords")
        ii = mir["edge_gpatch"][eidx].to(torch.int32)
        jj = mir["edge_dst"][eidx].to(torch.int32)
        corr.corr(gmap, pyr, coords, ii, jj)
        rep = ba.solve(prob, max_iterations=2, tolerance=1e-12)
        torch.cuda.synchronize()
        if r >= 2:
            times.append((time.perf_counter() - t0) * 1e3)
        del prob
    ms = float(np.median(times))
    desc = {"cfg1": "cfg1: 16-frame local window (640x480), 96 patches/frame, corr (2 levels) "
                    "+ BAProblem + solve(2 LM iterations)",
            "cfg2": "cfg2: EuRoC 752x480, 22-frame window, 96 patches/frame, corr (2 levels) "
                    "+ BAProblem + solve(2 LM iterations)"}
    return {"config": desc.get(config, config),
            "E": E, "ms": ms, "value": 2 * E / (ms * 1e-3), "unit": "patch-edges/s (x2 LM iters)",
            "iterations": rep.iterations, "final_objective": rep.final_objective,
            "includes": "index build, correlation, native LM, write-back (wall clock, synced)"}


def run_batch(args, torch, n_seq=8, reps=5, threads=0, seed0=0, warm=2, sequential_too=True):
    """cfg5: n_seq independent TartanAir-shape sequences on
    this GPU as replicas.  One batch step = for every sequence a new 22-frame
    BAProblem, the correlation of its window edges (2 levels, bf16) and
    solve(2 LM iterations, tol 1e-12), as the cfg2 window step; the problems
    run concurrently (ba.build_batch / ba.solve_batch: one stream and host
    worker each, no collective).  Also times the same steps run one after
    another, for the batching gain."""
    from paper_2408_01654_b200 import _lib, ba, corr, synthetic
    seqs = []
    C = args.channels
    fdt = torch.bfloat16 if args.feat_dtype == "bf16" else torch.float32
    for s in range(n_seq):
        scene, graph, free = synthetic.make_config("cfg5", seed=seed0 + s)
        w, h = scene.spec.image_size
        gen = torch.Generator(device="cuda").manual_seed(100 + seed0 + s)
        fmap = (torch.randn((graph.n_frames, h // 4, w // 4, C), generator=gen, device="cuda")
                / math.sqrt(C)).to(fdt)
        gmap = (torch.randn((graph.n_patches, 9, C), generator=gen, device="cuda")
                / math.sqrt(C)).to(fdt)
        seqs.append(dict(graph=graph, free=free, pyr=corr.pyramid(fmap), gmap=gmap,
                         soa0={k: np.array(v) for k, v in graph.soa().items()}))

    def reset():
        for sq in seqs:
            g = sq["graph"]
            g._q.view[:] = sq["soa0"]["frame_q"]
            g._t.view[:] = sq["soa0"]["frame_t"]
            g._depth.view[:] = sq["soa0"]["patch_depth"]
            g._pose_ver += 1
            g._patch_ver += 1
            g.device()
        torch.cuda.synchronize()

    def window_corr(sq, prob):
        h_ = prob._ensure()
        E = int(prob.info().n_edges)
        q, t, d = prob.device_state()
        mir = sq["graph"].device()
        eidx = prob.view("edge_idx")
        sel = torch.arange(E, dtype=torch.int64, device="cuda")
        coords = torch.empty((E, 9, 2), dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().dpv_reproject_coords_sel(h_, _lib.ptr(q), _lib.ptr(t), _lib.ptr(d),
                                                       0.25, _lib.ptr(sel), E, _lib.ptr(coords),
                                                       _lib.stream_ptr()), "coords")
        corr.corr(sq["gmap"], sq["pyr"], coords, mir["edge_gpatch"][eidx].to(torch.int32),
                  mir["edge_dst"][eidx].to(torch.int32))
        return E

    phases = {"build": [], "corr": [], "solve": []}

    streams = [torch.cuda.Stream() for _ in seqs]      # one per sequence, reused

    def batched():
        t0 = time.perf_counter()
        probs = [ba.BAProblem(sq["graph"], sq["free"]) for sq in seqs]
        ba.build_batch(probs, threads, streams=streams)
        t1 = time.perf_counter()
        E = 0
        for sq, p in zip(seqs, probs):
            with torch.cuda.stream(p._stream):
                E += window_corr(sq, p)
        t2 = time.perf_counter()
        reps_ = ba.solve_batch(probs, 2, 1e-12, threads=threads)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        for k, v in zip(phases, (t1 - t0, t2 - t1, t3 - t2)):
            phases[k].append(v * 1e3)
        return E, reps_

    def sequential():
        E = 0
        for sq in seqs:
            p = ba.BAProblem(sq["graph"], sq["free"])
            E += window_corr(sq, p)
            ba.solve(p, 2, 1e-12)
        torch.cuda.synchronize()
        return E

    tb, ts = [], []
    E = 0
    out = []
    timed_launches = 0
    for r in range(reps + warm):
        reset()
        l0 = _lib.lib().dpv_launch_count()
        t0 = time.perf_counter()
        E, out = batched()
        if r >= warm:
            tb.append((time.perf_counter() - t0) * 1e3)
            timed_launches += _lib.lib().dpv_launch_count() - l0
        if sequential_too:
            reset()
            t0 = time.perf_counter()
            sequential()
            if r >= warm:
                ts.append((time.perf_counter() - t0) * 1e3)
    ms = float(np.median(tb))
    ms_seq = float(np.median(ts)) if ts else float("nan")
    bad = [type(x).__name__ for x in out if isinstance(x, Exception)]
    return {"config": "cfg5: " + synthetic.DESCRIPTIONS["cfg5"], "sequences": n_seq,
            "E_total": E, "ms_per_batch": ms, "window_steps_per_s": n_seq / (ms * 1e-3),
            "value": 2 * E / (ms * 1e-3), "unit": "patch-edges/s (x2 LM iters)",
            "sequential_ms": ms_seq, "batching_gain": ms_seq / ms,
            "phase_ms": {k: float(np.median(v[warm:])) for k, v in phases.items()},
            "timed_ms": tb, "timed_launches": timed_launches,
            "iterations": [x.iterations for x in out if not isinstance(x, Exception)],
            "failed": bad,
            "includes": "index build, correlation, native LM, write-back for every sequence "
                        "(wall clock, synced); replicas on one stream + host worker each"}


def run_replicas(args):
    """cfg5 across GPUs (replicas only, no collective on the data
    path): rank r solves sequences r*B .. r*B+B-1 (B = --batch-seqs) as one
    concurrent batch per step (index build + correlation + 2 LM iterations
    per sequence, see run_batch).  Steps are bracketed by a barrier and a
    device synchronisation; the step time is the max over ranks and `value`
    counts every rank's patch-edges x LM iterations."""
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    tdist = None
    if world > 1:
        import torch.distributed as tdist
        if args.dist_backend == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            tdist.init_process_group(args.dist_backend)
        tdist.barrier()
    from paper_2408_01654_b200 import _lib
    B = args.batch_seqs
    res = run_batch(args, torch, n_seq=B, reps=args.steps, seed0=rank * B,
                    warm=max(args.warmup, 3), sequential_too=False)
    launches = res["timed_launches"]
    ms = float(np.mean(res["timed_ms"]))
    units = 2.0 * res["E_total"]
    if world > 1:
        t = torch.tensor([ms, units], dtype=torch.float64, device="cuda")
        mx = t[:1].clone()
        tdist.all_reduce(mx, op=tdist.ReduceOp.MAX)
        tot = t[1:].clone()
        tdist.all_reduce(tot)
        ms, units = float(mx.item()), float(tot.item())
        tdist.barrier()
        tdist.destroy_process_group()
        if rank != 0:
            return None
    return {
        "metric": "patch-edges/sec for corr lookup + Gauss-Newton BA step; global loop-closure BA ms",
        "value": units / (ms * 1e-3), "unit": "patch-edges/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator restated bit-exactly; random features)",
        "config": {"workload": f"cfg5: {B} TartanAir-shape sequences per GPU, one 22-frame window "
                               "step each (index build + corr + 2 LM iterations), replicas",
                   "sequences": B * world, "parallelism": f"replicas x{world} (no collective)",
                   "l2": "per-step index rebuild and fresh problems (inputs re-read from HBM)"},
        "gpu_launches": int(launches),
        "batch": {k: v for k, v in res.items() if k not in ("timed_ms", "timed_launches")},
    }


def run_global(work, args, torch):
    from paper_2408_01654_b200 import ba
    graph = work["graph"]
    soa0 = {k: np.array(v) for k, v in graph.soa().items()}
    times = []
    reps = []
    for r in range(3):
        # identical starting state for every run
        graph._q.view[:] = soa0["frame_q"]
        graph._t.view[:] = soa0["frame_t"]
        graph._depth.view[:] = soa0["patch_depth"]
        graph._pose_ver += 1
        graph._patch_ver += 1
        graph.device()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        prob = ba.BAProblem(graph, work["free"])
        rep = ba.solve(prob, max_iterations=args.lm_iters, tolerance=1e-9)
        torch.cuda.synchronize()
        times.append((time.perf_counter() - t0) * 1e3)
        reps.append(rep)
        del prob
    rep = reps[-1]
    return {"ms": float(np.median(times[1:])), "runs_ms": times, "iterations": rep.iterations,
            "lm_attempts": rep.n_attempts, "backend": rep.backend,
            "iteration_ms": [x * 1e3 for x in rep.iteration_times],
            "initial_objective": rep.initial_objective, "final_objective": rep.final_objective,
            "includes": "BAProblem index build + native LM + write-back"}


def workload_config(args, graph, free, world):
    """The bench line's `config`: the workload named from host data only, so
    the reference arm (which runs a bounded sample of it on the CPU and
    describes the sample in cpu_baseline.sample) prints the same dict."""
    from paper_2408_01654_b200.synthetic import DESCRIPTIONS as DESC
    return {"workload": f"{args.config}: {DESC.get(args.config, args.config)} + corr on "
                        "the window/loop edges",
            "frames": int(graph.n_frames), "patches": int(graph.n_patches),
            "graph_edges": int(graph.n_edges), "free_poses": [int(free[0]), int(free[1])],
            "corr_window": args.window, "corr_levels": 2, "corr_channels": args.channels,
            "corr_dtype": args.feat_dtype,
            "parallelism": (f"edge-shard x{world} by depth row, one "
                            f"{args.dist_backend.upper()} all-reduce of the packed reduced "
                            "pose system per step" if world > 1 else "single GPU"),
            "l2": f"inputs larger than L2 (flow targets {graph.n_edges * 144 / 1e9:.2f} GB, "
                  "126 MB L2)"}


def run_reference(args):
    """Reference arm: the unmodified reference package (baseline/_ref) on the
    host cores -- each step one full LM iteration of the named sub-problem of
    the same workload (bench_ref.py); the numpy oracle port if the reference
    is not installed.  Rank 0 only under torchrun."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import bench_ref
    from paper_2408_01654_b200 import synthetic
    t0 = time.perf_counter()
    scene, graph, free = synthetic.make_config(args.config)
    gen_s = time.perf_counter() - t0
    soa = {k: np.array(v) for k, v in graph.soa().items()}
    prefix = min(REF_PREFIX, graph.n_frames)
    warm = max(args.warmup, 0)
    if bench_ref.reference_available():
        r = bench_ref.time_iterations(soa, prefix, args.steps, warm)
        kind = "reference"
    else:
        r = port_iterations(soa, prefix, args.steps, warm)
        kind = "port"
    value = r["value"]
    return {
        "impl": "reference",
        "metric": "patch-edges/sec for corr lookup + Gauss-Newton BA step; global loop-closure BA ms",
        "value": value, "unit": "patch-edges/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": warm, "ms_per_step": r["step_s"] * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator restated bit-exactly)",
        "config": workload_config(args, graph, free, int(os.environ.get("WORLD_SIZE", "1"))),
        "sample": {"workload": (f"{args.config} graph, global BA over its first {prefix} frames "
                                f"(the bounded sample of the ours arm's {graph.n_frames})"),
                   "E_ba": r["E"], "E_corr": 0,
                   "corr": "none: the reference has no correlation code (SPEC.md:14)"},
        "cpu_baseline": {"value": value, "unit": "patch-edges/s", "cores": r["cores"],
                         "kind": kind, "sample": r["sample"]},
        "reference_run": {k: r[k] for k in ("step_times_s", "objectives", "setup_s")},
        "e2e": {"value": value, "unit": "patch-edges/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "input_generation_s": gen_s,
    }


def main():
    import faulthandler
    # a stuck phase dumps every thread's stack to stderr (diagnostics only)
    faulthandler.dump_traceback_later(int(os.environ.get("DPV_BENCH_WATCHDOG_S", "420")),
                                      repeat=True, file=sys.stderr)
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        line = run_reference(args)
    elif args.config == "cfg5":
        line = run_replicas(args)
    else:
        line = run_ours(args)
    rank = int(os.environ.get("RANK", "0"))
    if rank == 0 and line is not None:
        text = json.dumps(line, default=float)
        print(text, flush=True)
        if args.json_out:
            with open(args.json_out, "w") as fh:
                fh.write(text + "\n")
    del world


if __name__ == "__main__":
    main()
