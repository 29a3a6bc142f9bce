set -x
export DPV_PLAN_DEBUG=1
timeout 300 python -m pytest tests/test_gpu_spd.py -x -q > gpurun_out/spd_test.log 2>&1; echo spd=$?
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --json-out gpurun_out/bench2.json > gpurun_out/bench2.log 2>&1; echo bench=$?
