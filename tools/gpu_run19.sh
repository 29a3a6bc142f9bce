#!/bin/bash
mkdir -p gpurun_out
for cfg in "0 start" "1 start" "0 solve" "1 solve"; do
  set -- $cfg
  DPV_BENCH_HIPRIO=$1 DPV_BENCH_CORR_AT=$2 python bench.py --steps 20 --no-global --no-e2e --no-cpu --json-out gpurun_out/b19_$1_$2.json > /dev/null 2>&1
  python -c "import json;d=json.load(open('gpurun_out/b19_$1_$2.json'));print('$1 $2', round(d['ms_per_step'],4), 'corr', round(d['kernels']['corr']['ms_per_step'],3), 'factor', round(d['kernels']['spd_factor']['ms_per_step'],3))"
done
