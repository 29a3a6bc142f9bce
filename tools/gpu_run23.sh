#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/prof_window2.py 2>&1 | head -1
python tools/bench_batch.py 8 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print({k:d[k] for k in ('sequences','ms_per_batch','window_steps_per_s','sequential_ms','phase_ms')})"
