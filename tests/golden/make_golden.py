"""Generate the golden parity fixtures from the REAL reference package.

Run in the build container only (the reference tree does not exist on the GPU
box)::

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
        python tests/golden/make_golden.py [--with-cfg3]

Every fixture is produced by calling the reference's own public functions
(``patchslam.synthetic.generate``/``fill_flow``, ``patchslam.ba.*``,
``patchslam.block_cholesky.block_cholesky``, ``patchslam.geometry.reproject_grid``)
on seeded inputs, and stored as ``tests/golden/<case>.npz``.  The oracle
(``oracle/``) is pinned against these files by ``tests/test_oracle_golden.py``
and the CUDA path by the ``-m gpu`` parity tests.

Graph state is stored in the structure-of-arrays layout the B200 package uses
(see DESIGN.md "Data layout"): frame_q/frame_t, patch_offset/patch_grid/
patch_depth/patch_landmark, edge_src/edge_patch/edge_dst/edge_target/
edge_conf/edge_kind.
"""

from __future__ import annotations

import argparse
import copy
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from patchslam import ba  # noqa: E402  (reference, via PYTHONPATH)
from patchslam.block_cholesky import block_cholesky  # noqa: E402
from patchslam.errors import SingularSystem  # noqa: E402
from patchslam.geometry import Intrinsics, Patch, Pose, pinhole_rays, reproject_grid  # noqa: E402
from patchslam.graph import LOOP, PatchGraph  # noqa: E402
from patchslam.synthetic import OracleConfig, SceneSpec, fill_flow, generate  # noqa: E402


# ---------------------------------------------------------------------------
# reference objects -> SoA


def graph_soa(graph) -> dict:
    fq = np.stack([f.pose.q for f in graph.frames])
    ft = np.stack([f.pose.t for f in graph.frames])
    counts = [len(p) for p in graph.patches]
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    grids = np.stack([p.grid for plist in graph.patches for p in plist])
    depth = np.array([p.inverse_depth for plist in graph.patches for p in plist])
    lm = np.array([-1 if p.landmark_id is None else p.landmark_id
                   for plist in graph.patches for p in plist], dtype=np.int64)
    e = graph.edges
    out = {
        "intr": graph.intrinsics.as_array(),
        "patch_size": np.int64(graph.patch_size),
        "frame_q": fq, "frame_t": ft,
        "patch_offset": off, "patch_grid": grids, "patch_depth": depth,
        "patch_landmark": lm,
        "edge_src": np.array([x.src_frame for x in e], dtype=np.int64),
        "edge_patch": np.array([x.src_patch for x in e], dtype=np.int64),
        "edge_dst": np.array([x.dst_frame for x in e], dtype=np.int64),
        "edge_target": np.stack([x.target for x in e]) if e else np.zeros((0, 9, 2)),
        "edge_conf": np.stack([x.confidence for x in e]) if e else np.zeros((0, 2)),
        "edge_kind": np.array([1 if x.kind == LOOP else 0 for x in e], dtype=np.uint8),
    }
    return out


def perturb_poses(graph, sigma, seed, first=1, frame="world"):
    # restated from the reference test conftest (pkg/tests/conftest.py:28-32);
    # frame="camera" right-multiplies the same draws (the cfg4 recipe)
    rng = np.random.default_rng(seed)
    for f in graph.frames[first:]:
        noise = Pose.exp(rng.normal(0, sigma, 6))
        f.pose = noise * f.pose if frame == "world" else f.pose * noise


def dump_problem(prefix, out, graph, free_range, *, lam=1e-4, iters=2, tol=1e-12,
                 threshold=48, edge_indices=None):
    """All hot-path intermediates of one BAProblem, under ``prefix``."""
    g = copy.deepcopy(graph)
    problem = ba.BAProblem(g, free_range, edge_indices=edge_indices)
    out[prefix + "free_range"] = np.array(free_range, dtype=np.int64)
    if edge_indices is not None:
        out[prefix + "given_edge_indices"] = np.array(edge_indices, dtype=np.int64)
    out[prefix + "edge_indices"] = np.array(problem.edge_indices, dtype=np.int64)
    out[prefix + "depth_keys"] = np.array(problem.depth_keys, dtype=np.int64).reshape(-1, 2)
    out[prefix + "var_of"] = problem._var_of.astype(np.int64)
    out[prefix + "touched_fixed"] = np.array(problem.touched_fixed, dtype=np.int64)
    out[prefix + "scale_degenerate"] = np.bool_(problem.scale_degenerate)
    out[prefix + "active_patches"] = np.int64(problem.active_patch_count())
    st = problem._structure()
    for k in ("src", "dst", "depth_row", "rays", "target", "weight"):
        out[prefix + "st_" + k] = np.asarray(st[k])
    maps = problem._assembly_maps()
    for k, v in maps.items():
        out[prefix + "map_" + k] = np.asarray(v)
    q, t, d = problem.state()
    out[prefix + "state_d"] = d
    res, valid = ba.residuals(problem, (q, t, d))
    out[prefix + "res"] = res
    out[prefix + "valid"] = valid
    out[prefix + "objective"] = np.float64(ba.objective(problem, (q, t, d)))
    system = ba.assemble(problem, (q, t, d))
    for k in ("pair_keys", "pose_blocks", "schur_blocks", "depth_diag", "rhs_pose",
              "rhs_depth", "rhs_schur", "inc_var", "inc_row", "inc_block", "active"):
        out[prefix + "sys_" + k] = np.asarray(getattr(system, k))
    out[prefix + "sys_gradient_norm"] = np.float64(system.gradient_norm)
    if system.scale_pin is not None:
        out[prefix + "sys_pin_var"] = np.int64(system.scale_pin[0])
        out[prefix + "sys_pin_u"] = np.asarray(system.scale_pin[1])
    keys, blocks, rhs, cinv = system.reduced_system(lam)
    out[prefix + "red_lam"] = np.float64(lam)
    out[prefix + "red_blocks"] = blocks
    out[prefix + "red_rhs"] = rhs
    out[prefix + "red_cinv"] = cinv
    try:
        dp, dd, s1 = ba.solve_dense(system, lam)
        out[prefix + "dense_dp"] = dp
        out[prefix + "dense_dd"] = dd
        out[prefix + "dense_peak"] = np.int64(s1["peak_block_count"])
        dp2, dd2, s2 = ba.solve_block_sparse(system, lam)
        out[prefix + "bs_dp"] = dp2
        out[prefix + "bs_dd"] = dd2
        out[prefix + "bs_peak"] = np.int64(s2["peak_block_count"])
        cq, ct, cd = ba._apply_step(q, t, d, dp, dd, problem)
        out[prefix + "cand_q"] = cq
        out[prefix + "cand_t"] = ct
        out[prefix + "cand_d"] = cd
        out[prefix + "cand_objective"] = np.float64(ba.objective(problem, (cq, ct, cd)))
        out[prefix + "singular"] = np.bool_(False)
    except SingularSystem:
        out[prefix + "singular"] = np.bool_(True)
    # full LM solve on a fresh copy
    g2 = copy.deepcopy(graph)
    p2 = ba.BAProblem(g2, free_range, edge_indices=edge_indices)
    try:
        rep = ba.solve(p2, max_iterations=iters, tolerance=tol, backend_threshold=threshold)
        out[prefix + "lm_iters"] = np.int64(iters)
        out[prefix + "lm_tol"] = np.float64(tol)
        out[prefix + "lm_threshold"] = np.int64(threshold)
        out[prefix + "rep_iterations"] = np.int64(rep.iterations)
        out[prefix + "rep_initial"] = np.float64(rep.initial_objective)
        out[prefix + "rep_final"] = np.float64(rep.final_objective)
        out[prefix + "rep_backend"] = np.array(rep.backend)
        out[prefix + "rep_converged"] = np.bool_(rep.converged)
        out[prefix + "rep_gradient_norm"] = np.float64(rep.gradient_norm)
        out[prefix + "rep_unconstrained"] = np.int64(rep.unconstrained_depths)
        out[prefix + "rep_active"] = np.int64(rep.active_patches)
        out[prefix + "rep_final_damping"] = np.float64(rep.final_damping)
        out[prefix + "rep_step_norm"] = np.float64(rep.step_norm)
        after = graph_soa(g2)
        out[prefix + "after_frame_q"] = after["frame_q"]
        out[prefix + "after_frame_t"] = after["frame_t"]
        out[prefix + "after_patch_depth"] = after["patch_depth"]
        out[prefix + "lm_singular"] = np.bool_(False)
    except SingularSystem:
        out[prefix + "lm_singular"] = np.bool_(True)


def save(name, d):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **d)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB, {len(d)} arrays)")


def put_graph(out, graph, prefix="g_"):
    for k, v in graph_soa(graph).items():
        out[prefix + k] = v


# ---------------------------------------------------------------------------
# cases


def case_small():
    """conftest.small_scene (pkg/tests/conftest.py:10-16) perturbed as in test_ba.py:31-36."""
    spec = SceneSpec(kind="circle", n_frames=12, seed=5, n_landmarks=1500, look="inward")
    scene, graph = generate(spec, patches_per_frame=20, odometry_radius=4)
    fill_flow(graph, scene, OracleConfig())
    out = {}
    put_graph(out, graph, "gt_")          # ground-truth state (zero residual)
    perturb_poses(graph, 0.05, seed=11)
    put_graph(out, graph)
    dump_problem("p_", out, graph, (1, graph.n_frames - 1), iters=3)
    # non-degenerate: two fixed poses pin the scale (test_ba.py:222-231)
    g2 = copy.deepcopy(graph)
    dump_problem("q_", out, g2, (2, graph.n_frames - 1), iters=3)
    # threshold 0 forces the block-sparse backend on the same problem
    dump_problem("s_", out, graph, (1, graph.n_frames - 1), iters=3, threshold=0)
    # sub-range window with explicit edge list
    dump_problem("w_", out, graph, (5, 8), iters=2)
    save("small", out)


def case_window():
    """cfg1 shape reduced to 24 patches/frame (BASELINE.json configs[0])."""
    spec = SceneSpec(kind="circle", n_frames=16, seed=0, n_landmarks=3000, look="inward",
                     image_size=(640, 480), intrinsics=Intrinsics(320.0, 320.0, 320.0, 240.0))
    scene, graph = generate(spec, patches_per_frame=24, odometry_radius=13)
    fill_flow(graph, scene, OracleConfig(pixel_noise_sigma=0.3, outlier_fraction=0.05), seed=1)
    perturb_poses(graph, 0.02, seed=11)
    out = {}
    put_graph(out, graph)
    dump_problem("p_", out, graph, (1, 15), iters=2)
    save("window", out)


def case_loops():
    """bench-ba recipe (pkg/src/patchslam/cli.py:94-110) at 60 poses: block-sparse backend."""
    n_poses, patches, radius, seed = 60, 12, 5, 0
    spec = SceneSpec(kind="circle", n_frames=n_poses + 1, seed=seed,
                     n_landmarks=max(1200, 12 * n_poses), look="inward",
                     extent=max(10.0, n_poses / 8.0))
    scene, graph = generate(spec, patches_per_frame=patches, odometry_radius=radius)
    rng = np.random.default_rng(seed)
    loops = []
    for _ in range(max(2, n_poses // 60) + 2):
        old = int(rng.integers(0, max(1, n_poses // 4)))
        recent = int(rng.integers(3 * n_poses // 4, n_poses))
        loops.extend((old, k, recent) for k in range(min(patches, 32)))
    graph.add_edges(loops, kind=LOOP)
    fill_flow(graph, scene, OracleConfig(pixel_noise_sigma=0.3), seed=1)
    perturb_poses(graph, 0.02, seed=11)
    out = {}
    put_graph(out, graph)
    dump_problem("p_", out, graph, (1, n_poses), iters=3, tol=1e-9)
    save("loops", out)


def case_edges():
    """Edge cases: self-edges, a zero-confidence patch, outliers, cells behind the camera."""
    spec = SceneSpec(kind="circle", n_frames=8, seed=3, n_landmarks=800, look="inward")
    scene, graph = generate(spec, patches_per_frame=10, odometry_radius=3)
    graph.add_edges([(2, 1, 2), (5, 3, 5)])          # self edges (graph.py:144-165 allows them)
    fill_flow(graph, scene, OracleConfig(pixel_noise_sigma=0.5, outlier_fraction=0.1), seed=4)
    for e in graph.edges:
        if e.src_frame == 0 and e.src_patch == 0:
            e.confidence = np.zeros(2)           # test_ba.py:135-148 pattern
    perturb_poses(graph, 0.03, seed=7)
    # push one frame so that some reprojected cells land behind it
    f = graph.frames[6]
    f.pose = Pose(f.pose.q, f.pose.t + 6.0 * (Pose(f.pose.q).rotation_matrix()[:, 2]))
    out = {}
    put_graph(out, graph)
    dump_problem("p_", out, graph, (1, graph.n_frames - 1), iters=2)
    # singular: zero information everywhere (test_ba.py:170-178)
    g0 = copy.deepcopy(graph)
    for e in g0.edges:
        e.confidence = np.zeros(2)
    put_graph(out, g0, "z_")
    dump_problem("z_p_", out, g0, (1, g0.n_frames - 1), iters=2)
    save("edges", out)


def case_reproject():
    """Random poses/patches through reproject_grid with Jacobians (geometry.py:478-529)."""
    rng = np.random.default_rng(15)
    intr = Intrinsics(320.0, 320.0, 256.0, 192.0)
    n = 400
    poses_i = [Pose.exp(rng.normal(0, 0.3, 6)) for _ in range(n)]
    poses_j = [Pose.exp(rng.normal(0, 0.3, 6)) for _ in range(n)]
    d = rng.uniform(0.05, 1.0, n)
    centers = rng.uniform([64, 48], [448, 336], (n, 2))
    grids = np.stack([Patch.square(0, c, 1.0).grid for c in centers])
    rays = pinhole_rays(grids, intr)
    ri = np.stack([p.rotation_matrix() for p in poses_i])
    rj = np.stack([p.rotation_matrix() for p in poses_j])
    ti = np.stack([p.t for p in poses_i])
    tj = np.stack([p.t for p in poses_j])
    # a few edges deliberately behind the target camera
    tj[:10] = ti[:10] + 20.0 * ri[:10, :, 2]
    pix, valid, jp, jd = reproject_grid(rays, d, ri, ti, rj, tj, intr, jacobians=True)
    out = {"intr": intr.as_array(), "grid": grids, "rays": rays, "d": d,
           "qi": np.stack([p.q for p in poses_i]), "ti": ti,
           "qj": np.stack([p.q for p in poses_j]), "tj": tj,
           "rot_i": ri, "rot_j": rj,
           "pix": pix, "valid": valid, "j_pose": jp, "j_depth": jd}
    save("reproject", out)


def _random_block_spd(n, rng, extra):
    # same construction as pkg/tests/test_block_cholesky.py:8-24 (restated)
    keys = {(j, j) for j in range(n)} | {(j, j + 1) for j in range(n - 1)}
    for _ in range(extra):
        a, b = sorted(rng.integers(0, n, 2))
        if a != b:
            keys.add((int(a), int(b)))
    keys = sorted(keys)
    blocks = []
    for a, b in keys:
        blk = rng.normal(size=(6, 6))
        blk = blk @ blk.T + 6 * n * np.eye(6) if a == b else 0.3 * blk
        blocks.append(blk)
    return np.array(keys), np.stack(blocks)


def case_cholesky():
    rng = np.random.default_rng(0)
    out = {}
    for c in range(12):
        n = int(rng.integers(2, 60))
        keys, blocks = _random_block_spd(n, rng, n // 2)
        rhs = rng.normal(size=(n, 6))
        fac = block_cholesky(keys, blocks, n)
        out[f"c{c}_n"] = np.int64(n)
        out[f"c{c}_keys"] = keys
        out[f"c{c}_blocks"] = blocks
        out[f"c{c}_rhs"] = rhs
        out[f"c{c}_x"] = fac.solve(rhs)
        out[f"c{c}_block_count"] = np.int64(fac.block_count)
    save("cholesky", out)


# ---------------------------------------------------------------------------
# synthetic-generator hashes (inputs of configs 1-3)


def case_detect():
    """Proximity loop-closure candidates (pkg/src/patchslam/loop.py:51-85):
    camera centres of a few synthetic trajectories that revisit themselves,
    reference detect() output in its distance order (stable for ties)."""
    from patchslam.loop import ProximityConfig, detect, resolve_threshold
    out = {}
    k = 0
    for kind, n, gap, thr, newest in [("circle", 120, 30, None, None),
                                      ("square-loop", 200, 31, None, None),
                                      ("circle", 90, 40, 0.9, 85),
                                      ("circle", 60, 40, None, 30),
                                      ("line", 150, 30, 3.0, None)]:
        spec = SceneSpec(kind=kind, n_frames=n, seed=k, n_landmarks=4 * n, look="forward",
                         extent=12.0, overshoot=0.2)
        scene, graph = generate(spec, patches_per_frame=2, odometry_radius=3)
        cfg = ProximityConfig(distance_threshold=thr, min_temporal_gap=gap)
        pairs = detect(graph, cfg, newest=newest)
        out[f"d{k}_centers"] = graph.camera_centers()
        out[f"d{k}_gap"] = np.int64(gap)
        out[f"d{k}_threshold"] = np.float64(resolve_threshold(graph, cfg))
        out[f"d{k}_newest"] = np.int64(-1 if newest is None else newest)
        out[f"d{k}_pairs"] = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
        k += 1
    out["n_cases"] = np.int64(k)
    save("detect", out)


def soa_hashes(graph) -> dict:
    h = {}
    for k, v in graph_soa(graph).items():
        a = np.ascontiguousarray(np.asarray(v))
        h[k] = hashlib.sha256(a.tobytes()).hexdigest()
    return h


def synth_cfg(name):
    """Reference inputs for the benchmark configs (SURVEY.md 8d common recipe)."""
    if name == "cfg1":
        spec = SceneSpec(kind="circle", n_frames=16, seed=0, n_landmarks=3000, look="inward",
                         image_size=(640, 480), intrinsics=Intrinsics(320.0, 320.0, 320.0, 240.0))
        loops = 0
    elif name == "cfg2":
        spec = SceneSpec(kind="circle", n_frames=40, seed=0, n_landmarks=6000, look="inward",
                         image_size=(752, 480),
                         intrinsics=Intrinsics(458.654, 457.296, 367.215, 248.375))
        loops = 0
    elif name == "cfg3":
        n = 2000
        spec = SceneSpec(kind="circle", n_frames=n, seed=0, n_landmarks=72 * n, look="inward",
                         image_size=(640, 480), intrinsics=Intrinsics(320.0, 320.0, 320.0, 240.0),
                         extent=n / 8.0)
        loops = n
    elif name == "cfg4":
        n = 4500
        spec = SceneSpec(kind="square-loop", n_frames=n, seed=0, n_landmarks=72 * n,
                         look="forward", image_size=(1226, 370),
                         intrinsics=Intrinsics(718.856, 718.856, 607.193, 185.216), extent=440.0)
        loops = n
    elif name == "mid":
        n = 120
        spec = SceneSpec(kind="circle", n_frames=n, seed=0, n_landmarks=max(1200, 12 * n) * 6,
                         look="inward", image_size=(640, 480),
                         intrinsics=Intrinsics(320.0, 320.0, 320.0, 240.0), extent=max(10.0, n / 8.0))
        loops = n
    else:
        raise KeyError(name)
    t0 = time.time()
    scene, graph = generate(spec, patches_per_frame=96, odometry_radius=13)
    if loops:
        rng = np.random.default_rng(0)
        tri = []
        for _ in range(max(2, loops // 60)):
            old = int(rng.integers(0, max(1, loops // 4)))
            recent = int(rng.integers(3 * loops // 4, loops))
            tri.extend((old, k, recent) for k in range(32))
        graph.add_edges(tri, kind=LOOP)
    fill_flow(graph, scene, OracleConfig(pixel_noise_sigma=0.3), seed=1)
    perturb_poses(graph, 0.02, seed=11, frame="camera" if name == "cfg4" else "world")
    print(f"  {name}: {graph.n_frames} frames, {len(graph.edges)} edges, "
          f"{time.time() - t0:.1f}s")
    return spec, graph


def case_synth(with_cfg3, names=None):
    names = names or (["cfg1", "cfg2", "mid"] + (["cfg3"] if with_cfg3 else []))
    path = os.path.join(HERE, "synth_hashes.json")
    table = json.load(open(path)) if os.path.exists(path) else {}
    for name in names:
        _, graph = synth_cfg(name)
        table[name] = {"n_frames": graph.n_frames, "n_edges": len(graph.edges),
                       "sha256": soa_hashes(graph)}
    with open(path, "w") as fh:
        json.dump(table, fh, indent=1, sort_keys=True)
    print(f"wrote {path}")


def case_fixture():
    """Text fixture written by the reference's own writer (graph.py:268-296):
    a small perturbed scene plus loop edges, one frame without dense features
    and landmark extras; the SoA state beside it pins the parser."""
    from patchslam.graph import write_graph
    spec = SceneSpec(kind="circle", n_frames=6, seed=3, n_landmarks=600, look="inward")
    scene, graph = generate(spec, patches_per_frame=8, odometry_radius=2)
    graph.add_edges([(5, k, 0) for k in range(3)], kind=LOOP)
    fill_flow(graph, scene, OracleConfig(outlier_fraction=0.2), seed=2)
    perturb_poses(graph, 0.03, seed=4)
    graph.frames[2].has_dense_features = False
    out = {}
    put_graph(out, graph)
    out["g_timestamp"] = np.array([f.timestamp for f in graph.frames])
    out["g_keyframe"] = np.array([f.is_keyframe for f in graph.frames])
    out["g_features"] = np.array([f.has_dense_features for f in graph.frames])
    extras = [f"landmark {i} {x!r} {y!r} {z!r}"
              for i, (x, y, z) in enumerate(np.asarray(scene.landmarks)[:3].tolist())]
    write_graph(graph, os.path.join(HERE, "graph_fixture.txt"), extras)
    save("fixture", out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--with-cfg3", action="store_true")
    ap.add_argument("--only", default=None)
    ap.add_argument("--synth-names", default=None, help="e.g. cfg4 (hash table entries to add)")
    args = ap.parse_args()
    cases = {"small": case_small, "window": case_window, "loops": case_loops,
             "edges": case_edges, "reproject": case_reproject, "cholesky": case_cholesky,
             "detect": case_detect, "fixture": case_fixture,
             "synth": lambda: case_synth(args.with_cfg3, args.synth_names and
                                         args.synth_names.split(","))}
    for name, fn in cases.items():
        if args.only and name not in args.only.split(","):
            continue
        t0 = time.time()
        fn()
        print(f"{name}: {time.time() - t0:.1f}s", file=sys.stderr)
