DPV_PLAN_DEBUG=1 timeout 1500 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu --no-e2e --json-out gpurun_out/bench_cfg4.json > gpurun_out/bench_cfg4.log 2>&1; echo cfg4=$?
