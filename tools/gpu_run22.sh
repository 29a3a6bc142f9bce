#!/bin/bash
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:k_small_solve2 -s 2 -c 1 -o gpurun_out/small -f python tools/prof_window2.py > gpurun_out/ncu22.log 2>&1
tail -2 gpurun_out/ncu22.log
