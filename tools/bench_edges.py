"""Isolated timing of the edge-pass kernels on a config's problem
(objective; assemble chain with per-kernel CUDA-event times).

    python tools/bench_edges.py [--config cfg3]
"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_01654_b200 import _lib, ba, synthetic  # noqa: E402


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    t0 = time.time()
    scene, graph, free = synthetic.make_config(a.config)
    prob = ba.BAProblem(graph, free)
    h = prob._ensure()
    q, t, d = prob.device_state()
    lib = _lib.lib()
    P = _lib.ptr
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    s = _lib.stream_ptr
    print(f"setup {time.time() - t0:.1f}s")
    ms = timeit(lambda: lib.dpv_objective(h, P(q), P(t), P(d), P(out), s()))
    print(f"objective: {ms:.3f} ms  value {out.item():.12e}")
    _lib.timing_enable(True)
    ms = timeit(lambda: lib.dpv_assemble(h, P(q), P(t), P(d), s()))
    tm = _lib.timing_collect()
    _lib.timing_enable(False)
    print(f"assemble chain: {ms:.3f} ms")
    for name, (tot, cnt) in sorted(tm.items(), key=lambda kv: -kv[1][0]):
        print(f"  {name:20s} {tot / max(cnt, 1):.3f} ms x {cnt}")

if __name__ == "__main__":
    main()
