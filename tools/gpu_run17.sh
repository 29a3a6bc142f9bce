#!/bin/bash
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:k_assemble_edges_stg -s 3 -c 1 -o gpurun_out/asm_stg -f python tools/bench_edges.py --asm-variants 0 --key-variants 0 > gpurun_out/ncu17.log 2>&1
tail -3 gpurun_out/ncu17.log
