#!/bin/bash
for v in 0 1; do DPV_VAR_RHS_CTA=$v python bench.py --steps 10 --no-e2e --no-cpu --no-batch --no-global --json-out gpurun_out/b35_$v.json > /dev/null 2>&1; python -c "
import json;d=json.load(open('gpurun_out/b35_$v.json'));print('$v', d['ms_per_step'], d['kernels']['var_rhs']['ms_per_step'])"; done
