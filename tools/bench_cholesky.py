"""Microbenchmark of the dense FP64 Cholesky engine (K4c) via dpv_cholesky_solve.

    python tools/bench_cholesky.py [N] [reps]
Random diagonally dominant SPD matrix; reports wall time per solve, the
per-kernel event breakdown, achieved TFLOP/s (N^3/3) and the residual.
"""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_01654_b200 import _lib  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 11994
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    g = torch.Generator(device="cuda").manual_seed(0)
    a0 = torch.rand((N, N), generator=g, device="cuda", dtype=torch.float64)
    a0 = a0 + a0.T
    a0.diagonal().add_(2.0 * N + 1.0)
    b0 = torch.rand(N, generator=g, device="cuda", dtype=torch.float64)
    status = torch.zeros(8, dtype=torch.int32, device="cuda")
    lib = _lib.lib()
    times = []
    for r in range(reps + 1):
        a = a0.clone()
        b = b0.clone()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        _lib.check(lib.dpv_cholesky_solve(_lib.ptr(a), _lib.ptr(b), N, _lib.ptr(status),
                                          _lib.stream_ptr()), "solve")
        e1.record()
        torch.cuda.synchronize()
        if r:
            times.append(e0.elapsed_time(e1) * 1e-3)
    res = (a0 @ b - b0).abs().max().item() / b0.abs().max().item()
    # per-kernel split (note: dpv_cholesky_solve also copies the matrix)
    _lib.timing_enable(True)
    a = a0.clone()
    b = b0.clone()
    _lib.check(lib.dpv_cholesky_solve(_lib.ptr(a), _lib.ptr(b), N, _lib.ptr(status),
                                      _lib.stream_ptr()), "solve")
    tim = _lib.timing_collect()
    _lib.timing_enable(False)
    t = sorted(times)[len(times) // 2]
    print(f"N={N} median {t * 1e3:.2f} ms  {N ** 3 / 3 / t / 1e12:.2f} TFLOP/s (N^3/3)  "
          f"rel residual {res:.2e} status {status[0].item()}")
    for k, (ms, c) in sorted(tim.items(), key=lambda kv: -kv[1][0]):
        print(f"  {k:16s} {ms:9.3f} ms  {c:5d} launches  {ms / c * 1e3:9.2f} us/launch")
    # reference point: torch.linalg.cholesky (cuSOLVER) for context only
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    torch.linalg.cholesky(a0)
    torch.cuda.synchronize()
    print(f"  [context] torch.linalg.cholesky (cuSOLVER potrf): {(time.perf_counter() - t0) * 1e3:.2f} ms")


if __name__ == "__main__":
    main()
