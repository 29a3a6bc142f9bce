#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_ba_parity.py tests/test_gpu_batch.py tests/test_gpu_spd.py -x -q 2>&1 | tail -3
python tools/prof_window2.py 2>&1 | tail -14
DPV_SMALL_V1=1 python tools/prof_window2.py 2>&1 | grep small_solve
