"""cfg5 replicas leg of bench.py on its own: python tools/bench_batch.py [n_seq]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
th = int(sys.argv[2]) if len(sys.argv) > 2 else 0
args = argparse.Namespace(channels=128, feat_dtype="bf16")
print(json.dumps(bench.run_batch(args, torch, n_seq=n, threads=th)))
