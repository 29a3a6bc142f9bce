"""The reference arm of bench.py: the UNMODIFIED reference package
(``patchslam``, installed by ``build()`` into the git-ignored baseline/_ref,
which travels to the GPU box) timed on this host's cores.

One reference *step* = one LM iteration exactly as ``patchslam.ba.solve``
runs it when the first damping attempt is accepted (ba.py:553-581):
``assemble`` at the current state -> the selected backend's linear solve at
lambda (``_BACKENDS[select_backend(problem)]``) -> ``_apply_step`` ->
``objective`` of the candidate; the state advances.  The index caches
(``_structure`` / ``_assembly_maps``) are built once before timing, as the
B200 arm's index build is.

Workload: a fully executed, named sub-problem of the benchmark graph -- the
global BA over the first ``prefix`` frames of the cfg3 graph (free range
(1, prefix-1), every edge among those frames) -- so a step takes seconds, not
the ~90 s of a full cfg3 iteration.  The graph is handed to the reference as
its own objects (``PatchGraph`` / ``Frame`` / ``Patch`` / ``Edge``), built from
this package's generator, whose output is SHA-256-identical to the
reference generator's (tests/golden/synth_hashes.json).
"""

from __future__ import annotations

import importlib.util
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(ROOT, "baseline", "_ref")


def reference_available() -> bool:
    if os.path.isdir(os.path.join(REF, "patchslam")) and REF not in sys.path:
        sys.path.append(REF)
    return importlib.util.find_spec("patchslam") is not None


def reference_graph(soa: dict, n_frames: int):
    """The first ``n_frames`` frames of a SoA graph (and every edge among
    them) as a reference ``patchslam.graph.PatchGraph``."""
    from patchslam.geometry import Intrinsics, Patch, Pose
    from patchslam.graph import LOOP, ODOMETRY, Edge, PatchGraph
    intr = Intrinsics(*[float(v) for v in soa["intr"]])
    g = PatchGraph(intr, int(soa["patch_size"]))
    off = np.asarray(soa["patch_offset"])
    for f in range(n_frames):
        lo, hi = int(off[f]), int(off[f + 1])
        lm = soa["patch_landmark"][lo:hi]
        patches = [Patch(f, soa["patch_grid"][k], float(soa["patch_depth"][k]),
                         None if lm[k - lo] < 0 else int(lm[k - lo])) for k in range(lo, hi)]
        g.add_frame(Pose(soa["frame_q"][f], soa["frame_t"][f]), float(f), patches)
    src, dst = np.asarray(soa["edge_src"]), np.asarray(soa["edge_dst"])
    keep = np.nonzero((src < n_frames) & (dst < n_frames))[0]
    tgt, conf, kind = soa["edge_target"], soa["edge_conf"], soa["edge_kind"]
    pat = soa["edge_patch"]
    g.edges = [Edge(int(src[e]), int(pat[e]), int(dst[e]), tgt[e], conf[e],
                    LOOP if kind[e] == 1 else ODOMETRY) for e in keep]
    return g


def time_iterations(soa: dict, prefix: int, steps: int, warmup: int) -> dict:
    """Build the prefix problem with the reference and time ``steps`` LM
    iterations (after ``warmup`` untimed ones)."""
    from patchslam import ba as rba
    t0 = time.perf_counter()
    graph = reference_graph(soa, prefix)
    problem = rba.BAProblem(graph, (1, prefix - 1))
    problem._structure()
    problem._assembly_maps()
    setup_s = time.perf_counter() - t0
    backend = rba.select_backend(problem)
    solver = rba._BACKENDS[backend]
    lam = problem.damping
    q, t, d = problem.state()
    obj0 = rba.objective(problem, (q, t, d))
    times, objs = [], []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        system = rba.assemble(problem, (q, t, d))
        dp, dd, _ = solver(system, lam)
        q, t, d = rba._apply_step(q, t, d, dp, dd, problem)
        obj = rba.objective(problem, (q, t, d))
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
            objs.append(obj)
    E = len(problem.edge_indices)
    step_s = float(np.median(times))
    return {
        "E": E, "P": int(problem.n_depths), "n_free": int(problem.n_free_poses),
        "backend": backend, "step_s": step_s, "step_times_s": times, "setup_s": setup_s,
        "initial_objective": float(obj0), "objectives": [float(o) for o in objs],
        "value": E / step_s, "unit": "patch-edges/s",
        "cores": os.cpu_count(),
        "threads": {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS")},
        "sample": (f"unmodified reference patchslam.ba (baseline/_ref): one LM iteration per step "
                   f"(assemble -> {backend} solve at lambda {lam:g} -> _apply_step -> candidate "
                   f"objective) on the global BA over the first {prefix} frames of the cfg3 graph "
                   f"(free range (1, {prefix - 1}), E = {E} edges); median of {len(times)} "
                   f"iterations after {warmup} warm-up; numpy elementwise single-threaded, "
                   f"LAPACK on all host threads"),
    }
