"""Index-build phase times at a config (DPV_BUILD_PROFILE=1 prints them)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2408_01654_b200 import ba, synthetic  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
scene, graph, free = synthetic.make_config(cfg)
graph.device()
for r in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = ba.BAProblem(graph, free)
    p._ensure()
    torch.cuda.synchronize()
    print(f"build {cfg} run {r}: {(time.perf_counter() - t0) * 1e3:.2f} ms", file=sys.stderr)
    del p
