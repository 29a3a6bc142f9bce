set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2a_gputest.log 2>&1; tail -15 gpurun_out/r2a_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r2a_smoke.log 2>&1; tail -3 gpurun_out/r2a_smoke.log
timeout 900 python bench.py --json-out gpurun_out/r2a_bench.json > gpurun_out/r2a_bench.log 2>&1; tail -c 1500 gpurun_out/r2a_bench.log
timeout 900 python bench.py --impl reference > gpurun_out/r2a_bench_ref.log 2>&1; tail -c 800 gpurun_out/r2a_bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2a_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r2a_ncu_bench.log 2>&1; tail -3 gpurun_out/r2a_ncu_bench.log
