#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -1
python bench.py --steps 10 --no-e2e --no-cpu --no-batch --json-out gpurun_out/b30.json > /dev/null 2>&1; echo bench=$?
python -c "
import json;d=json.load(open('gpurun_out/b30.json'));g=d['global_ba']
print('step',d['ms_per_step'],'value',d['value'],'global',g['ms'])
for k in ("rows","incidences","key_blocks","var_rhs","back_substitute","assemble_edges","spd_factor"): print(k, round(d['kernels'][k]['ms_per_step'],4))"
