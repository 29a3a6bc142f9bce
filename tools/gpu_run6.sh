timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py --json-out gpurun_out/bench6.json > gpurun_out/bench6.log 2>&1; echo bench=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_assemble_edges|k_objective_seg|k_corr_mma|k_key_blocks|k_spd_factor|k_incidences|k_coords_sel" -c 9 -o gpurun_out/full_r01c python bench.py --steps 1 --warmup 1 --no-global --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 600 -c 1200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-global --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
