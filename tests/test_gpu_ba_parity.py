"""GPU parity of the BA hot path against the reference's golden vectors.

Every case of tests/golden (produced by the real reference, make_golden.py)
is replayed through the package's public API, which runs the sm_100a kernels
through the C-ABI.  Tolerances (stated per field, float64 throughout):

* index construction (edge selection, depth keys, touched frames, union keys,
  incidences, Schur pairs, structure rays/targets/weights): bit-exact;
* residuals: elementwise rel 1e-9 (near-zero depths amplify rounding);
  objective rel 1e-11;
* Hessian / Schur blocks, rhs, coupling blocks: 1e-9 of the array's max;
* pose / depth updates: 1e-7 of max (ill-conditioned reduced systems);
* full LM: same iteration count / backend, final objective rel 1e-6,
  poses and depths 1e-7.
"""

import numpy as np
import pytest

from conftest import BA_CASES, golden_graph

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2408_01654_b200 import ba, block_cholesky, geometry  # noqa: E402
from paper_2408_01654_b200.errors import SingularSystem  # noqa: E402
from paper_2408_01654_b200.graph import PatchGraph  # noqa: E402


def close(a, b, rel, abs_=0.0):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    assert a.shape == b.shape, (a.shape, b.shape)
    if a.size == 0:
        return
    scale = max(1.0, float(np.abs(b).max()))
    err = float(np.abs(a - b).max())
    assert err <= abs_ + rel * scale, f"max err {err:.3e} (scale {scale:.3e})"


def close_elem(a, b, rel, abs_):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    bad = np.abs(a - b) > abs_ + rel * np.abs(b)
    assert not bad.any(), f"{bad.sum()} elements off"


def make(z, gp, pp):
    g = PatchGraph.from_soa(golden_graph(z, gp))
    given = z.get(pp + "given_edge_indices")
    return g, ba.BAProblem(g, tuple(z[pp + "free_range"]), edge_indices=given)


def test_reproject_grid(golden):
    z = golden("reproject")
    pix, valid, jp, jd = geometry.reproject_grid(z["rays"], z["d"], z["rot_i"], z["ti"],
                                                 z["rot_j"], z["tj"], z["intr"], jacobians=True)
    assert np.array_equal(valid, z["valid"])
    close(pix, z["pix"], 1e-13, 1e-12)
    close(jp, z["j_pose"], 1e-12, 1e-12)
    close(jd, z["j_depth"], 1e-12, 1e-12)
    p2, v2 = geometry.reproject_grid(z["rays"], z["d"], z["rot_i"], z["ti"], z["rot_j"],
                                     z["tj"], z["intr"])
    assert np.array_equal(p2, pix) and np.array_equal(v2, valid)


@pytest.mark.parametrize("fx,gp,pp", BA_CASES)
def test_index_bit_exact(golden, fx, gp, pp):
    z = golden(fx)
    _, prob = make(z, gp, pp)
    assert prob.edge_indices == z[pp + "edge_indices"].tolist()
    assert np.array_equal(np.array(prob.depth_keys).reshape(-1, 2), z[pp + "depth_keys"])
    assert np.array_equal(prob._var_of, z[pp + "var_of"])
    assert prob.touched_fixed == z[pp + "touched_fixed"].tolist()
    assert prob.scale_degenerate == bool(z[pp + "scale_degenerate"])
    assert prob.active_patch_count() == int(z[pp + "active_patches"])
    st = prob._structure()
    for k in ("src", "dst", "depth_row", "rays", "target", "weight"):
        assert np.array_equal(st[k], z[pp + "st_" + k]), k
    mp = prob._assembly_maps()
    for k, v in mp.items():
        assert np.array_equal(np.asarray(v), z[pp + "map_" + k]), k


@pytest.mark.parametrize("fx,gp,pp", BA_CASES)
def test_residuals_objective_assembly(golden, fx, gp, pp):
    z = golden(fx)
    _, prob = make(z, gp, pp)
    res, valid = ba.residuals(prob)
    assert np.array_equal(valid, z[pp + "valid"])
    close_elem(np.where(valid[..., None], res, 0), np.where(valid[..., None], z[pp + "res"], 0),
               1e-9, 1e-9)
    assert ba.objective(prob) == pytest.approx(float(z[pp + "objective"]), rel=1e-11, abs=1e-12)
    sysm = ba.assemble(prob)
    assert np.array_equal(sysm.pair_keys, z[pp + "sys_pair_keys"])
    assert np.array_equal(sysm.inc_var, z[pp + "sys_inc_var"])
    assert np.array_equal(sysm.inc_row, z[pp + "sys_inc_row"])
    assert np.array_equal(sysm.active, z[pp + "sys_active"])
    for k in ("pose_blocks", "schur_blocks", "depth_diag", "rhs_pose", "rhs_depth",
              "rhs_schur", "inc_block"):
        close(getattr(sysm, k), z[pp + "sys_" + k], 1e-9, 1e-9)
    assert sysm.gradient_norm == pytest.approx(float(z[pp + "sys_gradient_norm"]), rel=1e-8)
    if pp + "sys_pin_var" in z:
        close(sysm.scale_pin[1], z[pp + "sys_pin_u"], 1e-14, 1e-14)
    else:
        assert sysm.scale_pin is None
    keys, blocks, rhs, cinv = sysm.reduced_system(float(z[pp + "red_lam"]))
    close(blocks, z[pp + "red_blocks"], 1e-9, 1e-9)
    close(rhs, z[pp + "red_rhs"], 1e-9, 1e-9)
    close(cinv, z[pp + "red_cinv"], 1e-9, 1e-12)


@pytest.mark.parametrize("fx,gp,pp", BA_CASES)
def test_solves_and_step(golden, fx, gp, pp):
    z = golden(fx)
    _, prob = make(z, gp, pp)
    sysm = ba.assemble(prob)
    lam = float(z[pp + "red_lam"])
    if bool(z[pp + "singular"]):
        with pytest.raises(SingularSystem):
            ba.solve_dense(sysm, lam)
        with pytest.raises(SingularSystem):
            ba.solve_block_sparse(sysm, lam)
        return
    dp, dd, s1 = ba.solve_dense(sysm, lam)
    close(dp, z[pp + "dense_dp"], 1e-7, 1e-9)
    close(dd, z[pp + "dense_dd"], 1e-7, 1e-9)
    dp2, dd2, s2 = ba.solve_block_sparse(sysm, lam)
    close(dp2, z[pp + "bs_dp"], 1e-7, 1e-9)
    close(dd2, z[pp + "bs_dd"], 1e-7, 1e-9)
    assert s1["peak_block_count"] == int(z[pp + "dense_peak"])
    assert s2["peak_block_count"] == int(z[pp + "bs_peak"])
    close(sysm.back_substitute(z[pp + "dense_dp"], lam), z[pp + "dense_dd"], 1e-9, 1e-12)
    q, t, d = prob.state()
    cq, ct, cd = ba._apply_step(q, t, d, z[pp + "dense_dp"], z[pp + "dense_dd"], prob)
    close(cq, z[pp + "cand_q"], 1e-14, 1e-14)
    close(ct, z[pp + "cand_t"], 1e-13, 1e-13)
    close(cd, z[pp + "cand_d"], 1e-14, 1e-14)
    assert ba.objective(prob, (cq, ct, cd)) == pytest.approx(float(z[pp + "cand_objective"]),
                                                            rel=1e-10, abs=1e-12)


@pytest.mark.parametrize("fx,gp,pp", BA_CASES)
def test_lm_solve(golden, fx, gp, pp):
    z = golden(fx)
    g, prob = make(z, gp, pp)
    if bool(z[pp + "lm_singular"]):
        before = g.soa()["frame_q"].copy()
        with pytest.raises(SingularSystem):
            ba.solve(prob, max_iterations=2)
        assert np.array_equal(g.soa()["frame_q"], before)    # no write-back on failure
        return
    rep = ba.solve(prob, int(z[pp + "lm_iters"]), float(z[pp + "lm_tol"]),
                   backend_threshold=int(z[pp + "lm_threshold"]))
    assert rep.backend == str(z[pp + "rep_backend"])
    assert rep.iterations == int(z[pp + "rep_iterations"])
    assert rep.initial_objective == pytest.approx(float(z[pp + "rep_initial"]), rel=1e-11)
    assert rep.final_objective == pytest.approx(float(z[pp + "rep_final"]), rel=1e-6, abs=1e-10)
    assert rep.unconstrained_depths == int(z[pp + "rep_unconstrained"])
    assert rep.active_patches == int(z[pp + "rep_active"])
    assert rep.final_damping == pytest.approx(float(z[pp + "rep_final_damping"]))
    soa = g.soa()
    close(soa["frame_q"], z[pp + "after_frame_q"], 1e-7, 1e-9)
    close(soa["frame_t"], z[pp + "after_frame_t"], 1e-7, 1e-9)
    close(soa["patch_depth"], z[pp + "after_patch_depth"], 1e-7, 1e-9)


def test_block_cholesky(golden):
    z = golden("cholesky")
    c = 0
    while f"c{c}_n" in z:
        fac = block_cholesky.block_cholesky(z[f"c{c}_keys"], z[f"c{c}_blocks"], int(z[f"c{c}_n"]))
        assert fac.block_count == int(z[f"c{c}_block_count"])
        close(fac.solve(z[f"c{c}_rhs"]), z[f"c{c}_x"], 1e-10, 1e-10)
        c += 1
    with pytest.raises(SingularSystem):
        block_cholesky.block_cholesky(np.array([[0, 0], [1, 1]]),
                                      np.stack([np.eye(6), -np.eye(6)]), 2)
    with pytest.raises(SingularSystem):
        block_cholesky.block_cholesky(np.array([[0, 0]]), np.eye(6)[None], 2)


@pytest.mark.parametrize("case", [c for c in BA_CASES if c[0] in ("loops", "window")])
def test_grouped_schur_matches_golden(golden, case, monkeypatch):
    """The opt-in grouped Schur path (per-group SYRK W W^T on DMMA,
    DPV_SCHUR_GROUPED=1) gives the reference's Schur blocks and rhs_schur."""
    monkeypatch.setenv("DPV_SCHUR_GROUPED", "1")
    name, gp, pp = case
    z = golden(name)
    g, prob = make(z, gp, pp)
    sys_ = ba.assemble(prob)
    close(sys_.schur_blocks, z[pp + "sys_schur_blocks"], 1e-9, 1e-9)
    close(sys_.rhs_schur, z[pp + "sys_rhs_schur"], 1e-9, 1e-9)


def test_lm_solve_tile_plan_fallback(golden, monkeypatch):
    """When the banded+border plan is impossible (forced here with
    DPV_SPD_FAIL) the solve falls back to the tile-plan factorisation and the
    LM trajectory is unchanged (block-sparse golden problem, 60 poses)."""
    monkeypatch.setenv("DPV_SPD_FAIL", "1")
    z = golden("loops")
    g, prob = make(z, "g_", "p_")
    rep = ba.solve(prob, int(z["p_lm_iters"]), float(z["p_lm_tol"]),
                   backend_threshold=int(z["p_lm_threshold"]))
    assert rep.iterations == int(z["p_rep_iterations"])
    assert rep.final_objective == pytest.approx(float(z["p_rep_final"]), rel=1e-6, abs=1e-10)
    close(g.soa()["frame_t"], z["p_after_frame_t"], 1e-7, 1e-9)
