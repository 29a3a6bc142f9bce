import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
# the reference package installed by build() (git-ignored, travels to the GPU
# box): makes the drop-in exception hierarchy and the reference-suite shim
# tests (test_gpu_reference_suite.py) available; nothing on the product path
# computes with it
REF = os.path.join(ROOT, "baseline", "_ref")
if os.path.isdir(os.path.join(REF, "patchslam")) and REF not in sys.path:
    sys.path.append(REF)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False))


def golden_graph(z, prefix="g_"):
    """SoA graph dict (writable copies) from a golden fixture."""
    n = len(prefix)
    return {k[n:]: np.array(v) for k, v in z.items() if k.startswith(prefix)
            and k[n:] in GRAPH_KEYS}


GRAPH_KEYS = ("intr", "patch_size", "frame_q", "frame_t", "patch_offset", "patch_grid",
              "patch_depth", "patch_landmark", "edge_src", "edge_patch", "edge_dst",
              "edge_target", "edge_conf", "edge_kind")

# (fixture, graph prefix, problem prefix)
BA_CASES = [("small", "g_", "p_"), ("small", "g_", "q_"), ("small", "g_", "s_"),
            ("small", "g_", "w_"), ("window", "g_", "p_"), ("loops", "g_", "p_"),
            ("edges", "g_", "p_"), ("edges", "z_", "z_p_")]


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load_golden(name)
        return cache[name]
    return get
