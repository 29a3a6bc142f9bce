"""Multi-process (gloo, world size 2, CPU) tests of the sharded global BA's
host-side logic: depth-row partitioning and the all-reduce of the reduced
pose system.  The shard assembly is evaluated with the CPU oracle (the CUDA
kernels need a GPU); the reduction plumbing is the same torch.distributed
code path the NCCL run uses."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2408_01654_b200 import synthetic
from paper_2408_01654_b200.dist import allreduce_packed, shard_rows


def small_graph():
    spec = synthetic.SceneSpec(kind="circle", n_frames=24, seed=2, n_landmarks=2500,
                               look="inward")
    scene, graph = synthetic.generate(spec, patches_per_frame=16, odometry_radius=4,
                                      initial_targets=False)
    synthetic.add_loop_edges(graph, 24, 16, seed=0)
    synthetic.fill_flow(graph, scene, synthetic.OracleConfig(pixel_noise_sigma=0.3), seed=1)
    synthetic.perturb_poses(graph, 0.02, seed=11)
    return graph


def test_shard_rows_partition():
    graph = small_graph()
    free = (1, graph.n_frames - 1)
    for world in (1, 2, 3, 5):
        shards, bounds = shard_rows(graph, free, world)
        allidx = np.sort(np.concatenate(shards))
        src = graph._src.view
        dst = graph._dst.view
        inside = ((src >= 1) & (src <= free[1])) | ((dst >= 1) & (dst <= free[1]))
        assert np.array_equal(allidx, np.nonzero(inside)[0])         # cover, disjoint
        gid = graph.patch_offset()[src] + graph._pat.view
        owners = {}
        for r, s in enumerate(shards):
            for g in np.unique(gid[s]):
                assert owners.setdefault(int(g), r) == r                # rows never straddle
        sizes = [len(s) for s in shards]
        assert max(sizes) - min(sizes) <= max(200, 0.2 * max(sizes))  # balanced


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import ba_oracle as O
    graph = small_graph()
    soa = {k: np.array(v) for k, v in graph.soa().items()}
    free = (1, graph.n_frames - 1)
    shards, _ = shard_rows(graph, free, world)
    full = O.OracleProblem(soa, free)
    union = full.maps()["union_keys"]
    prob = O.OracleProblem(soa, free, edge_indices=shards[rank])
    sysm = O.assemble(prob)
    # place the shard's blocks on the global pattern, then all-reduce
    keys = prob.maps()["union_keys"]
    where = np.searchsorted(union, keys)
    assert np.array_equal(union[where], keys)
    pose = np.zeros((len(union), 6, 6))
    schur = np.zeros((len(union), 6, 6))
    pose[where] = sysm.pose_blocks
    schur[where] = sysm.schur_blocks
    # the packed buffer of dist.allreduce_packed: ONE all-reduce carries the
    # pose system and every rank's depth-gradient max (one slot per rank)
    buf = torch.from_numpy(np.concatenate([pose.ravel(), schur.ravel(), sysm.rhs_pose.ravel(),
                                           sysm.rhs_schur.ravel(), np.full(8, np.nan)]))
    n_sys = buf.numel() - 8
    depth_g = np.abs(sysm.rhs_depth[sysm.active]).max() if sysm.active.any() else 0.0
    grad = allreduce_packed(buf, buf[n_sys:], buf[2 * len(union) * 36:2 * len(union) * 36
                                                  + 6 * full.n_free],
                            torch.tensor(depth_g, dtype=torch.float64), rank, world, dist)
    buf = buf[:n_sys]
    obj = torch.tensor([O.objective(prob)], dtype=torch.float64)
    dist.all_reduce(obj)
    if rank == 0:
        ref = O.assemble(full)
        W = len(union)
        got = buf.numpy()
        out["pose"] = np.abs(got[:W * 36] - ref.pose_blocks.ravel()).max() / max(
            1.0, np.abs(ref.pose_blocks).max())
        out["schur"] = np.abs(got[W * 36:2 * W * 36] - ref.schur_blocks.ravel()).max() / max(
            1.0, np.abs(ref.schur_blocks).max())
        n6 = 6 * full.n_free
        out["rhs"] = np.abs(got[2 * W * 36:2 * W * 36 + n6] - ref.rhs_pose.ravel()).max() / max(
            1.0, np.abs(ref.rhs_pose).max())
        out["rhs_schur"] = np.abs(got[2 * W * 36 + n6:] - ref.rhs_schur.ravel()).max() / max(
            1.0, np.abs(ref.rhs_schur).max())
        out["obj"] = abs(obj.item() - O.objective(full)) / O.objective(full)
        out["grad"] = abs(float(grad) - ref.gradient_norm) / ref.gradient_norm
    dist.destroy_process_group()


def test_sharded_reduction_equals_full_system():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for k, v in res.items():
        assert v < 1e-10, (k, v)
