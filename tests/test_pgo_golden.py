"""CPU checks of the pose-graph golden vectors (written by the real reference,
tests/golden/make_golden_pgo.py) and of the host-side Similarity value type
the device PGO packs (no GPU needed)."""

import os

import numpy as np

from conftest import GOLDEN
from paper_2408_01654_b200 import posegraph as PG

Z = dict(np.load(os.path.join(GOLDEN, "pgo.npz")))


def test_golden_shapes_and_reference_outcomes():
    assert Z["exp_v"].shape == (20, 7) and Z["exp_s"].shape == (20, 8)
    assert Z["rj_J"].shape == (30, 7, 7)
    # reference posegraph tests' acceptance criteria hold on the stored results
    assert float(Z["chain_obj"]) < 1e-16 and float(Z["loop_obj"]) < 1e-12
    s = Z["drift_out"][:, 7]
    assert abs(s[0] - 1.0) < 1e-12 and np.all(np.diff(np.log(s)) > 0)
    for name in ("chain", "loop", "drift", "noisy"):
        assert int(Z[f"{name}_iters"]) <= int(Z[f"{name}_maxit"])
        q = Z[f"{name}_out"][:, 3:7]
        assert np.allclose(np.linalg.norm(q, axis=1), 1.0, atol=1e-12)


def test_host_similarity_group_laws():
    rng = np.random.default_rng(0)
    a = PG.Similarity(rng.normal(size=4), rng.normal(size=3), 1.7)
    b = PG.Similarity(rng.normal(size=4), rng.normal(size=3), 0.4)
    e = a * a.inverse()
    assert np.allclose(e.t, 0, atol=1e-12) and abs(e.s - 1) < 1e-12
    assert np.allclose(np.abs(e.q), [0, 0, 0, 1], atol=1e-12)
    x = rng.normal(size=3)
    # (a b)^-1 = b^-1 a^-1
    lhs, rhs = (a * b).inverse(), b.inverse() * a.inverse()
    assert np.allclose(lhs.t, rhs.t) and np.isclose(lhs.s, rhs.s)
    assert np.allclose(PG._pack([a])[0], np.r_[a.t, a.q, a.s])
    del x


def test_problem_validation():
    s = PG.Similarity.identity()
    try:
        PG.PoseGraphProblem([s, s], [], [])
        raise AssertionError("expected ValueError")
    except ValueError:
        pass
    try:
        PG.PoseGraphProblem([s, s], [s], [(0, 0, s)])
        raise AssertionError("expected ValueError")
    except ValueError:
        pass
