#!/bin/bash
mkdir -p gpurun_out
nproc
for a in "1 0" "8 1" "8 8" "8 4"; do python tools/bench_batch.py $a 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print({k:d[k] for k in ('sequences','ms_per_batch','sequential_ms','phase_ms')})"; done
