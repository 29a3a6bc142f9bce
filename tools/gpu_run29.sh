#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_ba_parity.py -x -q 2>&1 | tail -1
python tools/bench_edges.py --asm-variants 0 --key-variants 0 2>&1 | grep "assemble variant"
DPV_INC_VARIANT=1 python tools/bench_edges.py --asm-variants 0 --key-variants 0 2>&1 | grep "assemble variant"
