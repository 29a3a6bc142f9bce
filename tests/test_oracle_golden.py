"""Pin the CPU oracle against golden vectors produced by the real reference.

The fixtures come from tests/golden/make_golden.py (reference patchslam calls);
these tests need no GPU and no reference tree.
"""

import numpy as np
import pytest

from conftest import BA_CASES, golden_graph
from oracle import ba_oracle as O
from oracle.geometry_oracle import quat_to_rot, reproject


def close(a, b, rel=1e-10, abs_=1e-10):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    assert a.shape == b.shape, (a.shape, b.shape)
    if a.size == 0:
        return
    scale = max(1.0, float(np.abs(b).max()))
    err = float(np.abs(a - b).max())
    assert err <= abs_ + rel * scale, f"max err {err:.3e} (scale {scale:.3e})"


def close_elem(a, b, rel, abs_):
    """Elementwise |a-b| <= abs + rel*|b| (for arrays with huge dynamic range)."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    assert a.shape == b.shape
    bad = np.abs(a - b) > abs_ + rel * np.abs(b)
    assert not bad.any(), f"{bad.sum()} elements off; worst rel {np.max(np.abs(a-b)/np.maximum(np.abs(b),1e-300)):.3e}"


def test_reproject_matches_reference(golden):
    z = golden("reproject")
    rot_i = quat_to_rot(z["qi"])
    rot_j = quat_to_rot(z["qj"])
    close(rot_i, z["rot_i"], 1e-15, 1e-15)
    pix, valid, jp, jd = reproject(z["rays"], z["d"], rot_i, z["ti"], rot_j, z["tj"], z["intr"],
                                   jacobians=True)
    assert (valid == z["valid"]).all()
    assert (~valid).sum() >= 10 * 9 - 5  # the planted behind-camera edges
    close(pix, z["pix"], 1e-13, 1e-12)
    close(jp, z["j_pose"], 1e-12, 1e-12)
    close(jd, z["j_depth"], 1e-12, 1e-12)


@pytest.mark.parametrize("fx,gp,pp", BA_CASES)
def test_problem_index_bit_exact(golden, fx, gp, pp):
    z = golden(fx)
    g = golden_graph(z, gp)
    prob = O.OracleProblem(g, tuple(z[pp + "free_range"]),
                           edge_indices=z.get(pp + "given_edge_indices"))
    assert np.array_equal(prob.edge_indices, z[pp + "edge_indices"])
    assert np.array_equal(prob.depth_keys(), z[pp + "depth_keys"])
    assert np.array_equal(prob.var_of, z[pp + "var_of"])
    assert np.array_equal(prob.touched_fixed, z[pp + "touched_fixed"])
    assert bool(prob.scale_degenerate) == bool(z[pp + "scale_degenerate"])
    assert prob.active_patch_count() == int(z[pp + "active_patches"])
    st = prob.structure()
    for k in ("src", "dst", "depth_row"):
        assert np.array_equal(st[k], z[pp + "st_" + k]), k
    assert np.array_equal(st["rays"], z[pp + "st_rays"])        # same IEEE ops
    assert np.array_equal(st["target"], z[pp + "st_target"])
    assert np.array_equal(st["weight"], z[pp + "st_weight"])
    mp = prob.maps()
    for k, v in mp.items():
        ref = z[pp + "map_" + k]
        assert np.array_equal(np.asarray(v), ref), k


@pytest.mark.parametrize("fx,gp,pp", BA_CASES)
def test_residuals_and_assembly(golden, fx, gp, pp):
    z = golden(fx)
    g = golden_graph(z, gp)
    prob = O.OracleProblem(g, tuple(z[pp + "free_range"]))
    state = prob.state()
    res, valid = O.residuals(prob, state)
    assert np.array_equal(valid, z[pp + "valid"])
    close_elem(np.where(valid[..., None], res, 0), np.where(valid[..., None], z[pp + "res"], 0),
               1e-9, 1e-9)
    obj = O.objective(prob, state)
    assert obj == pytest.approx(float(z[pp + "objective"]), rel=1e-11, abs=1e-12)
    sys_ = O.assemble(prob, state)
    assert np.array_equal(sys_.pair_keys, z[pp + "sys_pair_keys"])
    assert np.array_equal(sys_.inc_var, z[pp + "sys_inc_var"])
    assert np.array_equal(sys_.inc_row, z[pp + "sys_inc_row"])
    assert np.array_equal(sys_.active, z[pp + "sys_active"])
    for k in ("pose_blocks", "schur_blocks", "depth_diag", "rhs_pose", "rhs_depth",
              "rhs_schur", "inc_block"):
        close(getattr(sys_, k), z[pp + "sys_" + k], 1e-9, 1e-9)
    assert sys_.gradient_norm == pytest.approx(float(z[pp + "sys_gradient_norm"]), rel=1e-8)
    if pp + "sys_pin_var" in z:
        assert sys_.scale_pin is not None
        close(sys_.scale_pin[1], z[pp + "sys_pin_u"], 1e-14, 1e-14)
    else:
        assert sys_.scale_pin is None
    keys, blocks, rhs, cinv = sys_.reduced_system(float(z[pp + "red_lam"]))
    close(blocks, z[pp + "red_blocks"], 1e-9, 1e-9)
    close(rhs, z[pp + "red_rhs"], 1e-9, 1e-9)
    close(cinv, z[pp + "red_cinv"], 1e-9, 1e-12)


@pytest.mark.parametrize("fx,gp,pp", BA_CASES)
def test_solves_and_step(golden, fx, gp, pp):
    z = golden(fx)
    g = golden_graph(z, gp)
    prob = O.OracleProblem(g, tuple(z[pp + "free_range"]))
    state = prob.state()
    sys_ = O.assemble(prob, state)
    lam = float(z[pp + "red_lam"])
    if bool(z[pp + "singular"]):
        with pytest.raises(O.OracleSingular):
            O.solve_dense(sys_, lam)
        with pytest.raises(O.OracleSingular):
            O.solve_block_sparse(sys_, lam)
        return
    dp, dd, s1 = O.solve_dense(sys_, lam)
    close(dp, z[pp + "dense_dp"], 1e-7, 1e-9)
    close(dd, z[pp + "dense_dd"], 1e-7, 1e-9)
    dp2, dd2, s2 = O.solve_block_sparse(sys_, lam)
    close(dp2, z[pp + "bs_dp"], 1e-7, 1e-9)
    close(dd2, z[pp + "bs_dd"], 1e-7, 1e-9)
    assert s1["peak_block_count"] == int(z[pp + "dense_peak"])
    assert s2["peak_block_count"] == int(z[pp + "bs_peak"])
    cq, ct, cd = O.apply_step(*state, z[pp + "dense_dp"], z[pp + "dense_dd"], prob)
    close(cq, z[pp + "cand_q"], 1e-14, 1e-14)
    close(ct, z[pp + "cand_t"], 1e-13, 1e-13)
    close(cd, z[pp + "cand_d"], 1e-14, 1e-14)
    assert O.objective(prob, (cq, ct, cd)) == pytest.approx(float(z[pp + "cand_objective"]),
                                                           rel=1e-10, abs=1e-12)


@pytest.mark.parametrize("fx,gp,pp", BA_CASES)
def test_lm_solve(golden, fx, gp, pp):
    z = golden(fx)
    g = golden_graph(z, gp)
    prob = O.OracleProblem(g, tuple(z[pp + "free_range"]))
    if bool(z[pp + "lm_singular"]):
        with pytest.raises(O.OracleSingular):
            O.lm_solve(prob, max_iterations=2)
        return
    rep = O.lm_solve(prob, int(z[pp + "lm_iters"]), float(z[pp + "lm_tol"]),
                     threshold=int(z[pp + "lm_threshold"]))
    assert rep.backend == str(z[pp + "rep_backend"])
    assert rep.iterations == int(z[pp + "rep_iterations"])
    assert rep.initial_objective == pytest.approx(float(z[pp + "rep_initial"]), rel=1e-11)
    assert rep.final_objective == pytest.approx(float(z[pp + "rep_final"]), rel=1e-6, abs=1e-10)
    assert rep.unconstrained_depths == int(z[pp + "rep_unconstrained"])
    assert rep.active_patches == int(z[pp + "rep_active"])
    assert rep.final_damping == pytest.approx(float(z[pp + "rep_final_damping"]))
    close(g["frame_q"], z[pp + "after_frame_q"], 1e-7, 1e-9)
    close(g["frame_t"], z[pp + "after_frame_t"], 1e-7, 1e-9)
    close(g["patch_depth"], z[pp + "after_patch_depth"], 1e-7, 1e-9)


def test_block_cholesky_matches_reference(golden):
    z = golden("cholesky")
    c = 0
    while f"c{c}_n" in z:
        n = int(z[f"c{c}_n"])
        fac = O.block_cholesky(z[f"c{c}_keys"], z[f"c{c}_blocks"], n)
        assert fac.block_count == int(z[f"c{c}_block_count"])
        close(fac.solve(z[f"c{c}_rhs"]), z[f"c{c}_x"], 1e-10, 1e-10)
        c += 1
    assert c >= 10


def test_block_cholesky_singular_cases():
    with pytest.raises(O.OracleSingular):
        O.block_cholesky(np.array([[0, 0], [1, 1]]), np.stack([np.eye(6), -np.eye(6)]), 2)
    with pytest.raises(O.OracleSingular):
        O.block_cholesky(np.array([[0, 0]]), np.eye(6)[None], 2)


def test_detect_oracle_matches_reference(golden):
    """oracle/loop_oracle.py reproduces the reference's proximity candidates
    (loop.py:64-85) in order, on the reference's own fixtures."""
    from oracle import loop_oracle
    z = golden("detect")
    for k in range(int(z["n_cases"])):
        c = z[f"d{k}_centers"]
        newest = int(z[f"d{k}_newest"])
        pairs = loop_oracle.detect(c, int(z[f"d{k}_gap"]), float(z[f"d{k}_threshold"]),
                                   None if newest < 0 else newest)
        assert np.array_equal(np.asarray(pairs, dtype=np.int64).reshape(-1, 2), z[f"d{k}_pairs"])
