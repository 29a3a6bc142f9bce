"""Isolated timing of the edge-pass kernels on the cfg3 problem (objective,
assemble chain) for kernel-variant tuning.

    python tools/bench_edges.py [--config cfg3] [--variants 0,1,2,3,4]
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
    ap.add_argument("--variants", default="0")
    ap.add_argument("--asm-variants", default="0")
    ap.add_argument("--key-variants", default="0,1,2,3,4")
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
    ref = None
    for v in a.variants.split(","):
        os.environ["DPV_OBJ_VARIANT"] = v
        ms = timeit(lambda: lib.dpv_objective(h, P(q), P(t), P(d), P(out), s()))
        val = out.item()
        ref = val if ref is None else ref
        print(f"objective variant {v}: {ms:.3f} ms  value {val:.12e}  rel {abs(val - ref) / ref:.1e}")
    for v in a.asm_variants.split(","):
        os.environ["DPV_ASM_VARIANT"] = v
        _lib.timing_enable(True)
        ms = timeit(lambda: lib.dpv_assemble(h, P(q), P(t), P(d), s()))
        tm = _lib.timing_collect()
        _lib.timing_enable(False)
        ae = tm.get("assemble_edges", (0, 1))
        inc = tm.get("incidences", (0, 1))
        print(f"assemble variant {v}: chain {ms:.3f} ms, k_assemble_edges {ae[0] / ae[1]:.3f} ms, "
              f"incidences {inc[0] / inc[1]:.3f} ms (DPV_INC_VARIANT="
              f"{os.environ.get('DPV_INC_VARIANT', '0')})")
    for v in a.key_variants.split(","):
        os.environ["DPV_KEY_VARIANT"] = v
        _lib.timing_enable(True)
        ms = timeit(lambda: lib.dpv_assemble(h, P(q), P(t), P(d), s()))
        tm = _lib.timing_collect()
        _lib.timing_enable(False)
        kb = tm.get("key_blocks", (0, 1))
        vs = tm.get("var_schur", (0, 1))
        print(f"    var_schur {vs[0] / vs[1]:.3f} ms")
        gs = tm.get("group_syrk", (0, 1))
        print(f"key variant {v}: chain {ms:.3f} ms, k_key_blocks {kb[0] / kb[1]:.3f} ms, group_syrk {gs[0] / gs[1]:.3f} ms")


if __name__ == "__main__":
    main()
