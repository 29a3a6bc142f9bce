#!/bin/bash
python -m pytest tests/test_gpu_ba_parity.py tests/test_gpu_batch.py -x -q 2>&1 | tail -2
mkdir -p gpurun_out
python tools/prof_window2.py 2>&1 | tail -14
DPV_SMALL_V1=1 python tools/prof_window2.py 2>&1 | head -3
