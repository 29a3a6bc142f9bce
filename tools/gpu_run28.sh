#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python bench.py --steps 5 --no-e2e --no-cpu --no-batch --json-out gpurun_out/b28.json > /dev/null 2>&1; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/b28.json'));g=d['global_ba'];print('step',d['ms_per_step'],'global',g['ms'],g['runs_ms'],g['iteration_ms'][:3])"
DPV_SPD_SYNC_PLAN=1 python bench.py --steps 5 --no-e2e --no-cpu --no-batch --json-out gpurun_out/b28s.json > /dev/null 2>&1
python -c "import json;d=json.load(open('gpurun_out/b28s.json'));g=d['global_ba'];print('sync plan: global',g['ms'],g['iteration_ms'][:3])"
