"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): a 60-pose loop-closure global BA (block-sparse backend ->
spd.cu's flag dataflow, both levels), a cfg1-shaped window BA (small dense
solver), a two-level bf16 correlation (corr_tma.cu mbarriers / TMA), a Sim(3)
pose-graph LM (pgo.cu + the dense K4c engine) and device input generation
(synth.cu).

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import golden_graph, load_golden  # noqa: E402
from paper_2408_01654_b200 import _lib, ba, corr  # noqa: E402
from paper_2408_01654_b200.graph import PatchGraph  # noqa: E402


def main():
    torch.cuda.set_device(0)
    l0 = _lib.lib().dpv_launch_count()
    z = load_golden("loops")
    g = PatchGraph.from_soa(golden_graph(z, "g_"))
    rep = ba.solve(ba.BAProblem(g, tuple(z["p_free_range"])), 2, 1e-12)
    print("loops:", rep.to_line())
    z = load_golden("window")
    g = PatchGraph.from_soa(golden_graph(z, "g_"))
    rep = ba.solve(ba.BAProblem(g, tuple(z["p_free_range"])), 2, 1e-12)
    print("window:", rep.to_line())
    rng = np.random.default_rng(0)
    C, E = 128, 256
    f = torch.as_tensor((rng.normal(size=(2, 32, 40, C)) / np.sqrt(C)), device="cuda").bfloat16()
    gm = torch.as_tensor((rng.normal(size=(16, 9, C)) / np.sqrt(C)), device="cuda").bfloat16()
    coords = torch.as_tensor(rng.uniform(0, [40, 32], size=(E, 1, 2))
                             + rng.uniform(-0.5, 0.5, (E, 9, 2)), device="cuda")
    ii = torch.as_tensor(rng.integers(0, 16, E).astype(np.int32), device="cuda")
    jj = torch.as_tensor(rng.integers(0, 2, E).astype(np.int32), device="cuda")
    out = corr.corr(gm, corr.pyramid(f), coords, ii, jj)
    torch.cuda.synchronize()
    print("corr:", tuple(out.shape), float(out.abs().sum()))
    # Sim(3) pose-graph LM (pgo.cu) on a golden problem, device input
    # generation (synth.cu: visibility, flow oracle, initial targets)
    from paper_2408_01654_b200 import posegraph as PG
    from paper_2408_01654_b200 import synthetic
    zp = dict(np.load(os.path.join(ROOT, "tests", "golden", "pgo.npz")))
    sims = lambda a: [PG.Similarity(r[3:7], r[0:3], float(r[7])) for r in a]   # noqa: E731
    loops = [(int(j), int(k), d) for (j, k), d in zip(zp["loop_loops"], sims(zp["loop_loopsim"]))]
    prob = PG.PoseGraphProblem(sims(zp["loop_nodes"]), sims(zp["loop_odo"]), loops)
    rep = PG.optimize(prob, 10)
    print("pgo:", rep.iterations, rep.final_objective)
    spec = synthetic.SceneSpec(kind="circle", n_frames=12, seed=1, n_landmarks=2000,
                               look="inward")
    scene, graph = synthetic.generate(spec, patches_per_frame=16, odometry_radius=3,
                                      initial_targets=True)
    synthetic.fill_flow(graph, scene, synthetic.OracleConfig(pixel_noise_sigma=0.3,
                                                             outlier_fraction=0.1), seed=1)
    print("synth:", graph.n_edges, float(np.abs(graph._tgt.view).sum()))
    print("kernels launched:", _lib.lib().dpv_launch_count() - l0)


if __name__ == "__main__":
    main()
