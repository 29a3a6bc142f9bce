set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py --json-out gpurun_out/bench.json > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-global --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_corr|k_assemble_edges|k_key_blocks|k_objective" -c 5 -o gpurun_out/full_r01 python bench.py --steps 1 --warmup 1 --no-global --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
