#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1500 python bench.py --config cfg4 --steps 5 --warmup 3 --no-e2e --no-cpu --no-batch --json-out gpurun_out/bench_cfg4.json > gpurun_out/bench_cfg4.log 2>&1; echo cfg4=$?
