"""Host-side checks of the batched-replica API (no GPU): settings are
validated per problem before any device work, and the C-ABI exports the
batch entry points with the signatures the binding declares."""

import numpy as np
import pytest

from conftest import golden_graph, load_golden

from paper_2408_01654_b200 import ba
from paper_2408_01654_b200.graph import PatchGraph


def _problems(k):
    z = load_golden("window")
    return [ba.BAProblem(PatchGraph.from_soa(golden_graph(z, "g_")), tuple(z["p_free_range"]))
            for _ in range(k)]


def test_solve_batch_empty():
    assert ba.solve_batch([]) == []


def test_solve_batch_rejects_mismatched_settings():
    probs = _problems(2)
    with pytest.raises(ValueError, match="one entry per problem"):
        ba.solve_batch(probs, max_iterations=[2])
    with pytest.raises(ValueError, match="one entry per problem"):
        ba.solve_batch(probs, tolerance=np.array([1e-9, 1e-9, 1e-9]))


def test_solve_batch_unknown_backend():
    with pytest.raises(KeyError):
        ba.solve_batch(_problems(1), backend="qr")


def test_batch_signatures_declared():
    from paper_2408_01654_b200 import _lib
    for name in ("dpv_problem_create_batch", "dpv_lm_solve_batch"):
        assert name in _lib.SIGNATURES
