"""Isolated K1 timing: cfg3-shaped correlation (E_corr edges, 52 feature
frames of 120x160x128 bf16, 2 levels) through the shipped TMA kernel.

    python tools/bench_corr.py [--edges 47232] [--frames 52] [--sorted 1]
"""
import argparse
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_01654_b200 import corr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--edges", type=int, default=47232)
    ap.add_argument("--frames", type=int, default=52)
    ap.add_argument("--patches", type=int, default=192000)
    ap.add_argument("--sorted", type=int, default=1)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    H, W, C = 120, 160, 128
    g = torch.Generator(device="cuda").manual_seed(0)
    fmap = (torch.randn((a.frames, H, W, C), generator=g, device="cuda") / math.sqrt(C)).bfloat16()
    pyr = corr.pyramid(fmap)
    gmap = (torch.randn((a.patches, 9, C), generator=g, device="cuda") / math.sqrt(C)).bfloat16()
    E = a.edges
    base = torch.rand((E, 1, 2), generator=g, device="cuda", dtype=torch.float64) * \
        torch.tensor([W, H], device="cuda", dtype=torch.float64)
    offs = torch.stack(torch.meshgrid(torch.arange(3.0), torch.arange(3.0), indexing="xy"),
                       -1).reshape(1, 9, 2).to("cuda", torch.float64) * 0.25
    coords = base + offs
    ii = torch.randint(0, a.patches, (E,), generator=g, device="cuda", dtype=torch.int32)
    jj = torch.randint(0, a.frames, (E,), generator=g, device="cuda", dtype=torch.int32)
    if a.sorted:
        jj, _ = torch.sort(jj)
    out = torch.empty((E, 2, 9, 7, 7), dtype=torch.float32, device="cuda")
    hbm_bytes = E * (144 + 8 + 2 * 441 * 4) + E * 9 * C * 2 + sum(p.numel() * 2 for p in pyr)
    for mode in ("tma",):
        for _ in range(3):
            corr.corr(gmap, pyr, coords, ii, jj, out=out)
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(a.reps):
            corr.corr(gmap, pyr, coords, ii, jj, out=out)
        t1.record()
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1) / a.reps
        print(f"{mode}: {ms:.3f} ms per 2-level corr of {E} edges; algorithmic "
              f"{hbm_bytes / 1e6:.0f} MB -> {hbm_bytes / ms / 1e6:.0f} GB/s; "
              f"{E * 2 * 9 * 64 * C * 2 / ms / 1e9:.1f} TFLOP/s (tap dots)")


if __name__ == "__main__":
    main()
