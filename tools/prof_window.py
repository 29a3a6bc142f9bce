"""cProfile of one cfg5 window step (host-side cost breakdown)."""
import argparse
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

args = argparse.Namespace(channels=128, feat_dtype="bf16")
bench.run_batch(args, torch, n_seq=1, reps=1)
pr = cProfile.Profile()
pr.enable()
bench.run_batch(args, torch, n_seq=1, reps=3)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
