#!/bin/bash
mkdir -p gpurun_out
python bench.py --steps 10 --no-e2e --no-cpu --no-batch --no-global --json-out gpurun_out/b31g.json 2>&1 | grep -i "graph\|error" | head -5
python bench.py --steps 10 --no-e2e --no-cpu --no-batch --no-global --no-graph --json-out gpurun_out/b31e.json > /dev/null 2>&1
python -c "
import json
for f in ('b31g','b31e'):
    d=json.load(open('gpurun_out/%s.json'%f)); print(f, d['ms_per_step'], d['value'], d['gpu_launches'], d['config'].get('cuda_graph'))"
