#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_corr.py -x -q 2>&1 | tail -3
python tools/bench_corr.py 2>&1 | tail -5
