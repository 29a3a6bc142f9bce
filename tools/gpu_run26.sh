#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_ba_parity.py tests/test_gpu_batch.py tests/test_gpu_spd.py -x -q 2>&1 | tail -2
python tools/prof_build.py cfg3 2>&1 | grep build
python tools/prof_build.py cfg2 2>&1 | grep build
