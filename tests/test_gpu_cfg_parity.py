"""GPU parity at the BASELINE configurations against the REAL reference.

``tests/golden/cfg_<name>.npz`` were written by ``make_golden_cfg.py``, which
runs the reference package (``patchslam.ba``) on the full cfg1 (16-frame
window), cfg2 (22-frame EuRoC window) and cfg3 (2000-frame global
loop-closure BA, 4.98 M edges, 1999 free poses) problems.  The package's
generator reproduces the reference inputs bit-for-bit (SHA-256 pinned in
``tests/golden/synth_hashes.json``), so both sides see identical inputs.

Tolerances (float64 throughout; "of max" = relative to the array's max |x|):

* every index / structure array (edge selection, depth keys, var map,
  structure rays / targets / weights, all ``_assembly_maps`` arrays, pair
  keys, incidences, active flags): **bit-exact** (SHA-256);
* starting objective: rel 1e-10;
* pose / Schur / coupling blocks, rhs, depth diagonal, reduced system:
  1e-9 of max (sampled rows exactly compared at that tolerance, plus full-array
  checksums sum / sum|x| / max|x| at rel 1e-9);
* block-sparse solve dp and back-substituted dd: 1e-7 of max;
* candidate poses / depths 1e-7 of max, candidate objective rel 1e-6;
* ``solve(max_iterations=2)``: same iteration count and backend, final
  objective rel 1e-6, poses / depths 1e-7 of max.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from golden_check import check, sha

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2408_01654_b200 import ba, synthetic  # noqa: E402
from paper_2408_01654_b200.graph import PatchGraph  # noqa: E402

CFGS = [c for c in ("cfg1", "cfg2", "cfg3")
        if os.path.exists(os.path.join(GOLDEN, f"cfg_{c}.npz"))]


@pytest.fixture(scope="module", params=CFGS)
def case(request):
    name = request.param
    z = dict(np.load(os.path.join(GOLDEN, f"cfg_{name}.npz"), allow_pickle=False))
    _, graph, free = synthetic.make_config(name)
    assert tuple(free) == tuple(z["free_range"])
    assert graph.n_edges == int(z["n_edges_graph"])
    soa = {k: np.array(v) for k, v in graph.soa().items()}
    return name, z, graph, soa, tuple(free)


def test_index_structure_bit_exact(case):
    name, z, graph, soa, free = case
    prob = ba.BAProblem(graph, free)
    assert sha(np.array(prob.edge_indices, dtype=np.int64)) == str(z["hash_edge_indices"])
    assert sha(np.array(prob.depth_keys, dtype=np.int64).reshape(-1, 2)) == str(z["hash_depth_keys"])
    assert sha(prob._var_of.astype(np.int64)) == str(z["hash_var_of"])
    assert prob.touched_fixed == z["touched_fixed"].tolist()
    assert prob.scale_degenerate == bool(z["scale_degenerate"])
    assert prob.n_depths == int(z["n_depths"])
    assert prob.active_patch_count() == int(z["active_patches"])
    st = prob._structure()
    for k in ("src", "dst", "depth_row", "rays", "target", "weight"):
        assert sha(st[k]) == str(z["hash_st_" + k]), k
    del st
    maps = prob._assembly_maps()
    keys = sorted(k[len("hash_map_"):] for k in z if k.startswith("hash_map_"))
    assert sorted(maps) == keys
    for k in keys:
        assert sha(np.asarray(maps[k])) == str(z["hash_map_" + k]), k


def test_objective_assembly_reduced_system(case):
    name, z, graph, soa, free = case
    prob = ba.BAProblem(graph, free)
    assert ba.objective(prob) == pytest.approx(float(z["objective"]), rel=1e-10)
    sysm = ba.assemble(prob)
    assert sha(sysm.pair_keys) == str(z["hash_sys_pair_keys"])
    assert sha(sysm.inc_var) == str(z["hash_sys_inc_var"])
    assert sha(sysm.inc_row) == str(z["hash_sys_inc_row"])
    assert sha(sysm.active) == str(z["hash_sys_active"])
    for k in ("pose_blocks", "schur_blocks", "depth_diag", "rhs_pose", "rhs_depth",
              "rhs_schur", "inc_block"):
        check(z, "sys_" + k, getattr(sysm, k), 1e-9, 1e-9)
    assert sysm.gradient_norm == pytest.approx(float(z["sys_gradient_norm"]), rel=1e-8)
    assert sysm.unconstrained_depths == int(z["sys_unconstrained"])
    if "sys_pin_var" in z:
        assert sysm.scale_pin[0] == int(z["sys_pin_var"])
        np.testing.assert_allclose(sysm.scale_pin[1], z["sys_pin_u"], rtol=0, atol=1e-14)
    else:
        assert sysm.scale_pin is None
    _, blocks, rhs, cinv = sysm.reduced_system(float(z["red_lam"]))
    check(z, "red_blocks", blocks, 1e-9, 1e-9)
    check(z, "red_rhs", rhs, 1e-9, 1e-9)
    check(z, "red_cinv", cinv, 1e-9, 1e-12)


def test_linear_solve_and_candidate(case):
    name, z, graph, soa, free = case
    prob = ba.BAProblem(graph, free)
    sysm = ba.assemble(prob)
    lam = float(z["red_lam"])
    backend = ba.select_backend(prob)
    assert backend == str(z["backend"])
    dp, dd, stats = ba._BACKENDS[backend](sysm, lam)
    assert stats["peak_block_count"] == int(z["peak_block_count"])
    check(z, "dp", dp, 1e-7, 1e-9)
    check(z, "dd", dd, 1e-7, 1e-9)
    q, t, d = prob.state()
    cq, ct, cd = ba._apply_step(q, t, d, dp, dd, prob)
    check(z, "cand_q", cq, 1e-7, 1e-9)
    check(z, "cand_t", ct, 1e-7, 1e-9)
    check(z, "cand_d", cd, 1e-7, 1e-9)
    assert ba.objective(prob, (cq, ct, cd)) == pytest.approx(float(z["cand_objective"]), rel=1e-6)


def test_lm_two_iterations(case):
    name, z, graph, soa, free = case
    g = PatchGraph.from_soa({k: np.array(v) for k, v in soa.items()})
    prob = ba.BAProblem(g, free)
    rep = ba.solve(prob, max_iterations=int(z["lm_iters"]), tolerance=1e-12)
    assert rep.backend == str(z["rep_backend"])
    assert rep.iterations == int(z["rep_iterations"])
    assert rep.initial_objective == pytest.approx(float(z["rep_initial"]), rel=1e-10)
    assert rep.final_objective == pytest.approx(float(z["rep_final"]), rel=1e-6)
    assert rep.final_damping == pytest.approx(float(z["rep_final_damping"]))
    # the LM driver's packed per-attempt read-back (k_lm_scalars): the last
    # accepted step's norm and the last assembly's gradient max
    assert rep.step_norm == pytest.approx(float(z["rep_step_norm"]), rel=1e-5)
    assert rep.gradient_norm == pytest.approx(float(z["rep_gradient_norm"]), rel=1e-5)
    q, t, d = prob.state()
    check(z, "after_q", q, 1e-7, 1e-9)
    check(z, "after_t", t, 1e-7, 1e-9)
    check(z, "after_d", d, 1e-7, 1e-9)
