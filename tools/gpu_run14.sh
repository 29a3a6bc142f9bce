#!/bin/bash
set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_batch.py -x -q 2>&1 | tail -5
python tools/prof_window.py 2>&1 | head -70
