"""The numpy oracle pinned to the reference at the BASELINE window configs.

``tests/golden/cfg_cfg1.npz`` / ``cfg_cfg2.npz`` hold the real reference's
results on the full cfg1 (16-frame, 22,464-edge) and cfg2 (22-frame EuRoC
window, 54,912-edge) problems (``make_golden_cfg.py``).  The oracle is test
infrastructure (the checker of the CUDA path); this pins it at those sizes
with the same tolerances the GPU test uses (``test_gpu_cfg_parity.py``).
CPU only.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import ba_oracle as O
from paper_2408_01654_b200 import synthetic
from golden_check import check, sha

CFGS = [c for c in ("cfg1", "cfg2") if os.path.exists(os.path.join(GOLDEN, f"cfg_{c}.npz"))]


@pytest.fixture(scope="module", params=CFGS)
def case(request):
    name = request.param
    z = dict(np.load(os.path.join(GOLDEN, f"cfg_{name}.npz"), allow_pickle=False))
    _, graph, free = synthetic.make_config(name)
    soa = {k: np.array(v) for k, v in graph.soa().items()}
    return name, z, soa, tuple(free)


def test_oracle_index_and_system(case):
    name, z, soa, free = case
    p = O.OracleProblem(soa, free)
    assert sha(np.asarray(p.edge_indices, dtype=np.int64)) == str(z["hash_edge_indices"])
    assert sha(np.asarray(p.depth_keys(), dtype=np.int64).reshape(-1, 2)) == str(z["hash_depth_keys"])
    st = p.structure()
    for k in ("src", "dst", "depth_row", "rays", "target", "weight"):
        assert sha(st[k]) == str(z["hash_st_" + k]), k
    maps = p.maps()
    for k, v in maps.items():
        if "hash_map_" + k in z:
            assert sha(np.asarray(v)) == str(z["hash_map_" + k]), k
    assert O.objective(p) == pytest.approx(float(z["objective"]), rel=1e-10)
    s = O.assemble(p)
    for k in ("pose_blocks", "schur_blocks", "depth_diag", "rhs_pose", "rhs_depth",
              "rhs_schur", "inc_block"):
        check(z, "sys_" + k, getattr(s, k), 1e-9, 1e-9)
    _, blocks, rhs, cinv = s.reduced_system(float(z["red_lam"]))
    check(z, "red_blocks", blocks, 1e-9, 1e-9)
    check(z, "red_rhs", rhs, 1e-9, 1e-9)


def test_oracle_lm(case):
    name, z, soa, free = case
    p = O.OracleProblem(soa, free)
    rep = O.lm_solve(p, int(z["lm_iters"]), 1e-12)
    assert rep.iterations == int(z["rep_iterations"])
    assert rep.final_objective == pytest.approx(float(z["rep_final"]), rel=1e-6)
    q, t, d = p.state()
    check(z, "after_q", q, 1e-7, 1e-9)
    check(z, "after_t", t, 1e-7, 1e-9)
    check(z, "after_d", d, 1e-7, 1e-9)
