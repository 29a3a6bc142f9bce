"""Batched replicas (SURVEY 8(d) cfg5, 8(e) "replicas only"): ba.solve_batch
runs independent problems concurrently (one stream + host worker each,
dpv_problem_create_batch / dpv_lm_solve_batch).  Every problem must come out
exactly as a lone ba.solve leaves it (bit-identical: same kernels, same
fixed-order reductions), match the reference goldens with test_lm_solve's
tolerances, and a singular problem must not disturb the others."""

import numpy as np
import pytest

from conftest import BA_CASES, golden_graph

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2408_01654_b200 import ba  # noqa: E402
from paper_2408_01654_b200.errors import SingularSystem  # noqa: E402
from paper_2408_01654_b200.graph import PatchGraph  # noqa: E402


def close(a, b, rel, abs_):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    scale = max(1.0, float(np.abs(b).max()))
    assert float(np.abs(a - b).max()) <= abs_ + rel * scale


def make(z, gp, pp):
    g = PatchGraph.from_soa(golden_graph(z, gp))
    given = z.get(pp + "given_edge_indices")
    return g, ba.BAProblem(g, tuple(z[pp + "free_range"]), edge_indices=given)


def settings(z, pp):
    if bool(z[pp + "lm_singular"]):         # test_lm_solve: solve(prob, max_iterations=2)
        return (2, 1e-9, ba.DEFAULT_BACKEND_THRESHOLD)
    return (int(z[pp + "lm_iters"]), float(z[pp + "lm_tol"]), int(z[pp + "lm_threshold"]))


@pytest.mark.parametrize("threads", [0, 1, 3])
def test_solve_batch_matches_solve_and_goldens(golden, threads):
    cases = [(golden(fx), gp, pp) for fx, gp, pp in BA_CASES]
    lone, batch = [], []
    for z, gp, pp in cases:
        lone.append(make(z, gp, pp))
        batch.append(make(z, gp, pp))
    ref = []
    for (g, prob), (z, gp, pp) in zip(lone, cases):
        it, tol, th = settings(z, pp)
        try:
            ref.append(ba.solve(prob, it, tol, backend_threshold=th))
        except SingularSystem as e:
            ref.append(e)
    st = [settings(z, pp) for z, _, pp in cases]
    out = ba.solve_batch([p for _, p in batch], [s[0] for s in st], [s[1] for s in st],
                         backend_threshold=[s[2] for s in st], threads=threads)
    assert len(out) == len(cases)
    for (z, gp, pp), (gl, _), (gb, _), r0, r1 in zip(cases, lone, batch, ref, out):
        if bool(z[pp + "lm_singular"]):
            assert isinstance(r0, SingularSystem) and isinstance(r1, SingularSystem)
            assert np.array_equal(gb.soa()["frame_q"], z[gp + "frame_q"])   # not written
            continue
        assert not isinstance(r1, Exception), r1
        assert (r1.iterations, r1.backend, r1.n_attempts) == (r0.iterations, r0.backend,
                                                              r0.n_attempts)
        assert r1.final_objective == r0.final_objective
        assert r1.final_damping == r0.final_damping
        for k in ("frame_q", "frame_t", "patch_depth"):
            assert np.array_equal(gb.soa()[k], gl.soa()[k]), k
        assert r1.final_objective == pytest.approx(float(z[pp + "rep_final"]), rel=1e-6,
                                                   abs=1e-10)
        close(gb.soa()["frame_t"], z[pp + "after_frame_t"], 1e-7, 1e-9)
        close(gb.soa()["patch_depth"], z[pp + "after_patch_depth"], 1e-7, 1e-9)


def test_build_batch_index_matches_lone_build(golden):
    z = golden("window")
    probs = [make(z, "g_", "p_")[1] for _ in range(4)]
    ba.build_batch(probs, threads=4)
    lone = make(z, "g_", "p_")[1]
    for p in probs:
        assert p.edge_indices == lone.edge_indices
        mp, ml = p._assembly_maps(), lone._assembly_maps()
        for k in ml:
            assert np.array_equal(np.asarray(mp[k]), np.asarray(ml[k])), k


def test_solve_batch_empty():
    assert ba.solve_batch([]) == []
