#!/bin/bash
# batched replicas: tests + cfg5 leg
set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_batch.py tests/test_gpu_ba_parity.py tests/test_gpu_spd.py -x -q 2>&1 | tail -15
for n in 1 8 16; do timeout 600 python tools/bench_batch.py $n 2>&1 | tail -1; done
