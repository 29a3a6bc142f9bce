"""Patch-graph text fixtures (reference graph.py:9-20,
264-357).  tests/golden/graph_fixture.txt was written by the reference's own
write_graph (make_golden.py case_fixture) with fixture.npz holding the same
graph's arrays: parsing must reproduce them bit-exactly, and writing the
parsed graph must reproduce the reference's text line for line."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden

from paper_2408_01654_b200 import fixture
from paper_2408_01654_b200.errors import IndexOutOfRange, ParseError

PATH = os.path.join(GOLDEN, "graph_fixture.txt")


def test_parse_reference_fixture_bit_exact():
    z = load_golden("fixture")
    with open(PATH) as fh:
        g, extras = fixture.parse_graph_lines(fh, PATH)
    soa = g.soa()
    for k in ("intr", "patch_size", "frame_q", "frame_t", "patch_offset", "patch_grid",
              "patch_depth", "patch_landmark", "edge_src", "edge_patch", "edge_dst",
              "edge_target", "edge_conf"):
        assert np.array_equal(np.asarray(soa[k]), z["g_" + k]), k
    assert np.array_equal(np.asarray(soa["edge_kind"]), z["g_edge_kind"])
    assert int(np.sum(soa["edge_kind"] == 1)) == 3          # the loop edges
    assert np.array_equal(g._ts.view, z["g_timestamp"])
    assert np.array_equal(g._kf.view, z["g_keyframe"])
    assert np.array_equal(g._feat.view, z["g_features"])
    assert [tok[0] for _, tok in extras] == ["landmark"] * 3


def test_write_reproduces_reference_text():
    g = fixture.read_graph(PATH)
    with open(PATH) as fh:
        ref = [ln.rstrip("\n") for ln in fh]
    ours = fixture.graph_to_lines(g)
    assert ours == ref[:len(ours)]
    assert all(ln.startswith("landmark") for ln in ref[len(ours):])


def test_round_trip(tmp_path):
    g = fixture.read_graph(PATH)
    p = tmp_path / "g.txt"
    fixture.write_graph(g, p, ["landmark 0 1.0 2.0 3.0"])
    g2, extras = fixture.parse_graph_lines(open(p), str(p))
    for k, v in g.soa().items():
        assert np.array_equal(np.asarray(v), np.asarray(g2.soa()[k])), k
    assert extras == [(len(fixture.graph_to_lines(g)) + 1, ["landmark", "0", "1.0", "2.0", "3.0"])]


def test_parse_errors():
    with pytest.raises(ParseError, match="missing intrinsics"):
        fixture.parse_graph_lines(["meta patch_size 3"])
    with pytest.raises(ParseError) as ei:
        fixture.parse_graph_lines(["intrinsics 1 1 0 0", "frame 0 x 1 1 0 0 0 0 0 0 1"], "f.txt")
    assert ei.value.line == 2 and ei.value.path == "f.txt"
    with pytest.raises(ParseError, match="non-contiguous"):
        fixture.parse_graph_lines(["intrinsics 1 1 0 0", "frame 1 0.0 1 1 0 0 0 0 0 0 1"])
    with pytest.raises(ParseError, match="unknown edge kind"):
        fixture.parse_graph_lines(["intrinsics 1 1 0 0", "edge 0 0 0 sideways 1 1"])
    with pytest.raises(IndexOutOfRange):
        fixture.parse_graph_lines(["intrinsics 1 1 0 0", "frame 0 0.0 1 1 0 0 0 0 0 0 1",
                                   "edge 0 0 0 odometry 1 1 " + " ".join(["0"] * 18)])
