timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --json-out gpurun_out/bench10.json > gpurun_out/bench10.log 2>&1; echo bench=$?
