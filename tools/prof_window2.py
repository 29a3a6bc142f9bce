"""Phase and kernel breakdown of one cfg2 window step (host wall clock with
syncs + per-kernel CUDA-event totals from the library's timing hooks)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_01654_b200 import _lib, ba, synthetic  # noqa: E402

scene, graph, free = synthetic.make_config("cfg2")
soa0 = {k: np.array(v) for k, v in graph.soa().items()}


def reset():
    graph._q.view[:] = soa0["frame_q"]
    graph._t.view[:] = soa0["frame_t"]
    graph._depth.view[:] = soa0["patch_depth"]
    graph._pose_ver += 1
    graph._patch_ver += 1
    graph.device()
    torch.cuda.synchronize()


def phases():
    out = {}
    t = time.perf_counter()

    def lap(k):
        nonlocal t
        torch.cuda.synchronize()
        now = time.perf_counter()
        out[k] = (now - t) * 1e3
        t = now
    prob = ba.BAProblem(graph, free)
    prob._ensure()
    lap("build")
    ap = prob.active_patch_count()
    lap("active_patch_count")
    q, tt, d = prob.device_state()
    lap("device_state")
    rep = ba.solve_device(prob, q, tt, d, 2, 1e-12, active_patches=ap)
    lap("lm_solve")
    prob.write_back(q, tt, d)
    lap("write_back")
    return out, rep


for _ in range(3):
    reset()
    phases()
res = []
for _ in range(10):
    reset()
    res.append(phases()[0])
print({k: round(float(np.median([r[k] for r in res])), 3) for k in res[0]})
reset()
_lib.timing_enable(True)
o, rep = phases()
tm = _lib.timing_collect()
_lib.timing_enable(False)
print("attempts", rep.n_attempts, "iterations", rep.iterations, "lm iteration_times", rep.iteration_times)
tot = 0
for k, (ms, n) in sorted(tm.items(), key=lambda x: -x[1][0]):
    tot += ms
    print(f"  {k:24s} {ms*1e3:8.1f} us  x{n}")
print("kernel total us", round(tot * 1e3, 1))
