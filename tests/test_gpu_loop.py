"""GPU proximity loop-closure detection (dpv_proximity_detect) against the
reference's own candidates (tests/golden/detect.npz, loop.py:64-85):
bit-exact pairs in the reference order (distance, ties by insertion), plus a
larger trajectory checked against the oracle, and loop.close on a synthetic
graph (edges inserted as the reference does, global BA lowers the objective)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import loop_oracle  # noqa: E402
from paper_2408_01654_b200 import loop, synthetic  # noqa: E402


class _G:
    def __init__(self, centers):
        self._c = centers
        self.n_frames = len(centers)

    def camera_centers(self):
        return self._c


def test_detect_matches_reference(golden):
    z = golden("detect")
    for k in range(int(z["n_cases"])):
        c = z[f"d{k}_centers"]
        newest = int(z[f"d{k}_newest"])
        cfg = loop.ProximityConfig(distance_threshold=float(z[f"d{k}_threshold"]),
                                   min_temporal_gap=int(z[f"d{k}_gap"]))
        pairs = loop.detect(_G(c), cfg, newest=None if newest < 0 else newest)
        assert np.array_equal(np.asarray(pairs, dtype=np.int64).reshape(-1, 2),
                              z[f"d{k}_pairs"]), k


def test_detect_large_trajectory_matches_oracle():
    rng = np.random.default_rng(5)
    t = np.linspace(0, 6 * np.pi, 3000)
    c = np.stack([np.cos(t) * 20, 0.01 * t, np.sin(t) * 20], 1) + rng.normal(0, 0.02, (3000, 3))
    cfg = loop.ProximityConfig(min_temporal_gap=50)
    thr = loop.resolve_threshold(_G(c), cfg)
    ref = loop_oracle.detect(c, 50, thr)
    got = loop.detect(_G(c), cfg)
    assert len(ref) > 1000
    assert got == ref


def test_close_inserts_loop_edges_and_solves():
    spec = synthetic.SceneSpec(kind="circle", n_frames=70, seed=3, n_landmarks=3000,
                               look="inward", extent=12.0)
    scene, graph = synthetic.generate(spec, 24, 5)
    synthetic.fill_flow(graph, scene, synthetic.OracleConfig(pixel_noise_sigma=0.3), seed=1)
    synthetic.perturb_poses(graph, 0.01, seed=4)
    cfg = loop.ProximityConfig(min_temporal_gap=30, odometry_radius=5, max_edges_per_closure=48)
    cands = loop.detect(graph, cfg)
    assert cands
    n0 = graph.n_edges
    oracle = synthetic.make_flow_oracle(scene, synthetic.OracleConfig(pixel_noise_sigma=0.3))
    ev = loop.close(graph, cands, oracle, cfg)
    assert ev.anchor == max(r for _, r in cands)
    assert len(ev.edge_indices) == min(48, 24 * len(ev.matched))
    assert graph.n_edges == n0 + len(ev.edge_indices)
    assert ev.report.final_objective < ev.report.initial_objective
