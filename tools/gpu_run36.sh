#!/bin/bash
for cfg in "0 0" "1 0" "0 1"; do set -- $cfg
DPV_KEY_CTA=$1 DPV_BSUB_WARP=$2 python bench.py --steps 10 --no-e2e --no-cpu --no-batch --no-global --json-out gpurun_out/b36.json > /dev/null 2>&1; python -c "
import json;d=json.load(open('gpurun_out/b36.json'));k=d['kernels'];print('$1 $2', round(d['ms_per_step'],4), 'key', round(k['key_blocks']['ms_per_step'],4), 'bsub', round(k['back_substitute']['ms_per_step'],4))"; done
