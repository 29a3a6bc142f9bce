mkdir -p gpurun_out
PYTHONFAULTHANDLER=1 timeout -s ABRT 600 python bench.py --json-out gpurun_out/r2m_bench.json > gpurun_out/r2m_bench.log 2> gpurun_out/r2m_bench.err; echo "bench rc=$?"
PYTHONFAULTHANDLER=1 timeout -s ABRT 600 python bench.py --config cfg4 --no-cpu --json-out gpurun_out/r2m_bench_cfg4.json > /dev/null 2> gpurun_out/r2m_bench_cfg4.err; echo "cfg4 rc=$?"
PYTHONFAULTHANDLER=1 timeout -s ABRT 300 python bench.py --config cfg5 --json-out gpurun_out/r2m_bench_cfg5.json > /dev/null 2> gpurun_out/r2m_bench_cfg5.err; echo "cfg5 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2m_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-global --no-cpu > /dev/null 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_key_blocks|k_corr_tma|k_incidences2|k_rows" -c 4 -o gpurun_out/r2m_full python bench.py --steps 2 --warmup 3 --no-e2e --no-global --no-cpu --no-graph > /dev/null 2>&1; echo "ncu full rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2m_ref.log 2>&1; tail -c 400 gpurun_out/r2m_ref.log
