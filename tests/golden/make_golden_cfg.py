"""Golden vectors at the BASELINE configurations, produced by the REAL reference.

Run in the build container only (the reference tree does not exist on the GPU
box); cfg3 takes about 15 minutes and ~30 GB of host memory::

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
        python tests/golden/make_golden_cfg.py cfg1 cfg2 cfg3

For each config (SURVEY.md 8(d) recipe: ``generate`` -> bench-ba LOOP edges ->
``fill_flow(sigma=0.3, seed=1)`` -> ``perturb_poses(0.02, seed=11)``) the
reference's own hot-path functions are called on the full problem and the
results are written to ``tests/golden/cfg_<name>.npz``:

* ``hash_<k>``: SHA-256 of every index / structure array the reference builds
  (``BAProblem`` ba.py:60-98, ``_structure`` ba.py:124-141,
  ``_assembly_maps`` ba.py:147-216) -- the CUDA path must be bit-exact;
* the starting objective (ba.py:244-253);
* the assembled system (ba.py:328-440), the damped reduced system
  (ba.py:303-319), the block-sparse solve (ba.py:475-487), back-substitution
  (ba.py:321-325) and the candidate state / objective (ba.py:521-531);
* the state after ``ba.solve(max_iterations=2)`` (ba.py:534-605) and its
  ``BAReport``.

Arrays with at most ``FULL_LIMIT`` elements are stored whole.  Larger ones are
stored as a seeded sample of rows (``smp_<k>_idx`` / ``smp_<k>_val``) plus
full-array checksums ``sum_<k>`` = [sum, sum |x|, max |x|] so that a wrong
entry anywhere still shows.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import synth_cfg  # noqa: E402  (reference recipe, same as make_golden)
from patchslam import ba  # noqa: E402

FULL_LIMIT = 60_000
SAMPLE_ROWS = 4096

FREE = {"cfg1": lambda n: (1, 15), "cfg2": lambda n: (n - 22, n - 1),
        "cfg3": lambda n: (1, n - 1)}


def sha(a) -> str:
    a = np.ascontiguousarray(np.asarray(a))
    return hashlib.sha256(a.tobytes()).hexdigest()


def put(out, key, a, rng):
    a = np.asarray(a, dtype=np.float64)
    if a.size <= FULL_LIMIT:
        out["full_" + key] = a
        return
    rows = a.shape[0]
    idx = np.sort(rng.choice(rows, size=min(SAMPLE_ROWS, rows), replace=False)).astype(np.int64)
    out["smp_" + key + "_idx"] = idx
    out["smp_" + key + "_val"] = a[idx]
    out["sum_" + key] = np.array([a.sum(), np.abs(a).sum(), np.abs(a).max()])


def dump(name):
    t0 = time.time()
    spec, graph = synth_cfg(name)
    free = FREE[name](graph.n_frames)
    rng = np.random.default_rng(12345)
    out = {"free_range": np.array(free, dtype=np.int64), "n_edges_graph": np.int64(len(graph.edges))}
    tm = {}

    t = time.time()
    problem = ba.BAProblem(graph, free)
    out["hash_edge_indices"] = np.array(sha(np.array(problem.edge_indices, dtype=np.int64)))
    out["hash_depth_keys"] = np.array(sha(np.array(problem.depth_keys, dtype=np.int64).reshape(-1, 2)))
    out["hash_var_of"] = np.array(sha(problem._var_of.astype(np.int64)))
    out["n_edges"] = np.int64(len(problem.edge_indices))
    out["n_depths"] = np.int64(problem.n_depths)
    out["touched_fixed"] = np.array(problem.touched_fixed, dtype=np.int64)
    out["scale_degenerate"] = np.bool_(problem.scale_degenerate)
    out["active_patches"] = np.int64(problem.active_patch_count())
    st = problem._structure()
    for k in ("src", "dst", "depth_row", "rays", "target", "weight"):
        out["hash_st_" + k] = np.array(sha(st[k]))
    maps = problem._assembly_maps()
    for k, v in maps.items():
        v = np.asarray(v)
        out["hash_map_" + k] = np.array(sha(v))
        out["len_map_" + k] = np.int64(v.shape[0]) if v.ndim else np.int64(0)
    tm["index"] = time.time() - t
    print(f"  {name}: index {tm['index']:.1f}s", flush=True)

    q, tt, d = problem.state()
    t = time.time()
    out["objective"] = np.float64(ba.objective(problem, (q, tt, d)))
    tm["objective"] = time.time() - t
    t = time.time()
    system = ba.assemble(problem, (q, tt, d))
    tm["assemble"] = time.time() - t
    print(f"  {name}: assemble {tm['assemble']:.1f}s", flush=True)
    out["hash_sys_pair_keys"] = np.array(sha(system.pair_keys))
    out["hash_sys_inc_var"] = np.array(sha(system.inc_var))
    out["hash_sys_inc_row"] = np.array(sha(system.inc_row))
    out["hash_sys_active"] = np.array(sha(system.active))
    for k in ("pose_blocks", "schur_blocks", "depth_diag", "rhs_pose", "rhs_depth",
              "rhs_schur", "inc_block"):
        put(out, "sys_" + k, getattr(system, k), rng)
    out["sys_gradient_norm"] = np.float64(system.gradient_norm)
    out["sys_unconstrained"] = np.int64(system.unconstrained_depths)
    if system.scale_pin is not None:
        out["sys_pin_var"] = np.int64(system.scale_pin[0])
        out["sys_pin_u"] = np.asarray(system.scale_pin[1])
    lam = 1e-4
    _, blocks, rhs, cinv = system.reduced_system(lam)
    out["red_lam"] = np.float64(lam)
    put(out, "red_blocks", blocks, rng)
    put(out, "red_rhs", rhs, rng)
    put(out, "red_cinv", cinv, rng)
    backend = ba.select_backend(problem)
    out["backend"] = np.array(backend)
    t = time.time()
    dp, dd, stats = ba._BACKENDS[backend](system, lam)
    tm["linear_solve"] = time.time() - t
    out["peak_block_count"] = np.int64(stats["peak_block_count"])
    put(out, "dp", dp, rng)
    put(out, "dd", dd, rng)
    cq, ct, cd = ba._apply_step(q, tt, d, dp, dd, problem)
    put(out, "cand_q", cq, rng)
    put(out, "cand_t", ct, rng)
    put(out, "cand_d", cd, rng)
    t = time.time()
    out["cand_objective"] = np.float64(ba.objective(problem, (cq, ct, cd)))
    tm["cand_objective"] = time.time() - t
    del system, blocks
    print(f"  {name}: solve+cand {tm['linear_solve'] + tm['cand_objective']:.1f}s", flush=True)

    # 2 LM iterations on the same problem (its caches are state-independent)
    iters = 2
    t = time.time()
    rep = ba.solve(problem, max_iterations=iters, tolerance=1e-12)
    tm["lm_solve"] = time.time() - t
    out["lm_iters"] = np.int64(iters)
    out["rep_iterations"] = np.int64(rep.iterations)
    out["rep_initial"] = np.float64(rep.initial_objective)
    out["rep_final"] = np.float64(rep.final_objective)
    out["rep_backend"] = np.array(rep.backend)
    out["rep_final_damping"] = np.float64(rep.final_damping)
    out["rep_gradient_norm"] = np.float64(rep.gradient_norm)
    out["rep_step_norm"] = np.float64(rep.step_norm)
    q2, t2, d2 = problem.state()
    put(out, "after_q", q2, rng)
    put(out, "after_t", t2, rng)
    put(out, "after_d", d2, rng)
    for k, v in tm.items():
        out["time_" + k] = np.float64(v)
    out["cpu_count"] = np.int64(os.cpu_count())
    path = os.path.join(HERE, f"cfg_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB) in {time.time() - t0:.0f}s; "
          f"times {tm}", flush=True)


if __name__ == "__main__":
    for n in sys.argv[1:] or ["cfg1", "cfg2"]:
        dump(n)
