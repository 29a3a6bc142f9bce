"""GPU test of the edge-sharded global BA (dist.py): two ranks share cuda:0
through the gloo backend (NCCL needs one GPU per rank; the driver's boxes
have one).  The sharded LM must reproduce the single-process ba.solve."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def graph_and_range():
    from paper_2408_01654_b200 import synthetic
    spec = synthetic.SceneSpec(kind="circle", n_frames=70, seed=0, n_landmarks=5000,
                               look="inward", extent=12.0)
    scene, graph = synthetic.generate(spec, patches_per_frame=24, odometry_radius=6,
                                      initial_targets=False)
    synthetic.add_loop_edges(graph, 70, 24, seed=0)
    synthetic.fill_flow(graph, scene, synthetic.OracleConfig(pixel_noise_sigma=0.3), seed=1)
    synthetic.perturb_poses(graph, 0.02, seed=11)
    return graph, (1, 69)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2408_01654_b200.dist import ShardedProblem
    graph, free = graph_and_range()
    sp = ShardedProblem(graph, free)
    rep, q, t, d = sp.solve(max_iterations=4, tolerance=1e-12)
    depth = sp.gather_depths(d)
    if rank == 0:
        out["rep"] = {k: v for k, v in rep.items() if k != "iteration_times"}
        out["t"] = t.cpu().numpy()
        out["depth"] = depth.cpu().numpy()
    dist.destroy_process_group()


def test_sharded_solve_matches_single_gpu():
    from paper_2408_01654_b200 import ba
    graph, free = graph_and_range()
    prob = ba.BAProblem(graph, free)
    ref = ba.solve(prob, max_iterations=4, tolerance=1e-12)
    soa = graph.soa()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, _port(), out), nprocs=2, join=True)
        res = dict(out)
    rep = res["rep"]
    assert rep["iterations"] == ref.iterations
    assert rep["initial_objective"] == pytest.approx(ref.initial_objective, rel=1e-10)
    assert rep["final_objective"] == pytest.approx(ref.final_objective, rel=1e-8)
    assert np.abs(res["t"] - soa["frame_t"]).max() < 1e-8
    assert np.abs(res["depth"] - soa["patch_depth"]).max() < 1e-8
