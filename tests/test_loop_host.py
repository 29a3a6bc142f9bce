"""Host-side loop-closure logic (no GPU): the closure triple order
(reference loop.py:98-106) and the configuration checks (loop.py:35-43)."""

import importlib.util

import numpy as np
import pytest

from paper_2408_01654_b200 import errors
from paper_2408_01654_b200.loop import ProximityConfig, closure_triples


def triples_loop(counts, matched, anchor, cap):
    # the reference's nested loop, written out (loop.py:98-106)
    out = []
    for old in matched:
        for k in range(int(counts[old])):
            if len(out) >= cap:
                break
            out.append((old, k, anchor))
        if len(out) >= cap:
            break
    return out


@pytest.mark.parametrize("seed", range(20))
def test_closure_triples_match_reference_loop(seed):
    rng = np.random.default_rng(seed)
    counts = rng.integers(0, 120, size=50)
    matched = rng.choice(50, size=int(rng.integers(0, 8)), replace=False).tolist()
    cap = int(rng.choice([1, 7, 96, 288, 10_000]))
    assert closure_triples(counts, matched, 49, cap) == triples_loop(counts, matched, 49, cap)


def test_config_validation():
    ProximityConfig().validate()
    for kw in ({"min_temporal_gap": 13}, {"backend_range": 1}, {"max_edges_per_closure": 0}):
        with pytest.raises(errors.ConfigError):
            ProximityConfig(**kw).validate()
    assert issubclass(errors.ConfigError, errors.PatchSlamError)
    assert issubclass(errors.ConfigError, ValueError)


@pytest.mark.skipif(importlib.util.find_spec("patchslam") is None,
                    reason="reference package not importable")
def test_errors_are_reference_subclasses():
    import patchslam.errors as ref
    for name in ("PatchSlamError", "SingularSystem", "ConfigError", "ParseError",
                 "NonPositiveDepth", "IndexOutOfRange"):
        assert issubclass(getattr(errors, name), getattr(ref, name)), name
    try:
        raise errors.SingularSystem("x")
    except ref.SingularSystem:
        pass
    e = errors.ParseError("bad token", "f.txt", 3)
    assert str(e) == str(ref.ParseError("bad token", "f.txt", 3))
