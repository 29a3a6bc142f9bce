timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --json-out gpurun_out/bench5.json > gpurun_out/bench5.log 2>&1; echo bench=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_assemble_edges|k_key_blocks|k_objective|k_key_blocks" -c 1 -o gpurun_out/full_r01b python bench.py --steps 1 --warmup 1 --no-global --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
