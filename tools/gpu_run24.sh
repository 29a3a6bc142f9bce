#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_ba_parity.py tests/test_gpu_batch.py -x -q 2>&1 | tail -2
python tools/bench_edges.py --asm-variants 8,9,10,11,0 --key-variants 0 2>&1 | grep "assemble variant"
