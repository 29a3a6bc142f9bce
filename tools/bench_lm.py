"""Where the global-BA time goes: ba.solve(8 LM iterations) on cfg3 with
per-kernel CUDA-event timing; prints wall vs summed kernel time.

    python tools/bench_lm.py
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_01654_b200 import _lib, ba, synthetic  # noqa: E402


def main():
    torch.cuda.set_device(0)
    scene, graph, free = synthetic.make_config(os.environ.get("CFG", "cfg3"))
    soa0 = {k: np.array(v) for k, v in graph.soa().items()}

    def reset():
        graph._q.view[:] = soa0["frame_q"]
        graph._t.view[:] = soa0["frame_t"]
        graph._depth.view[:] = soa0["patch_depth"]
        graph._pose_ver += 1
        graph._patch_ver += 1
        graph.device()
        torch.cuda.synchronize()

    for timed in (False, False, True):
        reset()
        if timed:
            _lib.timing_enable(True)
        t0 = time.perf_counter()
        prob = ba.BAProblem(graph, free)
        ta = time.perf_counter()
        prob._ensure()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        if timed:
            tb = _lib.timing_collect()
            print(f"BAProblem() python {1e3 * (ta - t0):.1f} ms, _ensure {1e3 * (t1 - ta):.1f} ms, "
                  f"build kernels {sum(v[0] for v in tb.values()):.1f} ms "
                  f"({sum(v[1] for v in tb.values())} timed launches)")
        rep = ba.solve(prob, max_iterations=8, tolerance=1e-9)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        if timed:
            tm = _lib.timing_collect()
            _lib.timing_enable(False)
            tot = sum(v[0] for v in tm.values())
            print(f"build {1e3 * (t1 - t0):.1f} ms, solve {1e3 * (t2 - t1):.1f} ms wall, "
                  f"kernels {tot:.1f} ms, attempts {rep.n_attempts}")
            for k, v in sorted(tm.items(), key=lambda kv: -kv[1][0])[:25]:
                print(f"  {k:22s} {v[0]:8.3f} ms  {v[1]:5d} launches")
        else:
            print(f"build {1e3 * (t1 - t0):.1f} ms, solve {1e3 * (t2 - t1):.1f} ms, "
                  f"iters {[round(1e3 * x, 2) for x in rep.iteration_times]}")


if __name__ == "__main__":
    main()
