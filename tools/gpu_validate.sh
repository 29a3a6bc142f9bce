# The round's GPU validation in one call (what the r02 numbers in profiles/ come from):
#   /usr/local/graft/bin/gpurun --timeout 4000 -- 'bash tools/gpu_validate.sh'
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -2
PYTHONFAULTHANDLER=1 timeout -s ABRT 600 python bench.py --json-out gpurun_out/bench.json > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?"
PYTHONFAULTHANDLER=1 timeout -s ABRT 600 python bench.py --config cfg4 --no-cpu --json-out gpurun_out/bench_cfg4.json > /dev/null 2> gpurun_out/bench_cfg4.err; echo "cfg4 rc=$?"
PYTHONFAULTHANDLER=1 timeout -s ABRT 300 python bench.py --config cfg5 --json-out gpurun_out/bench_cfg5.json > /dev/null 2> gpurun_out/bench_cfg5.err; echo "cfg5 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "reference rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-global --no-cpu > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spd_factor|k_assemble_edges_stg|k_key_blocks|k_incidences2|k_rows" -s 40 -c 8 -o gpurun_out/full python bench.py --steps 2 --warmup 3 --no-e2e --no-global --no-cpu --no-graph > /dev/null 2>&1; echo "ncu full rc=$?"
# compute-sanitizer is closed on this GPU pool (profiles/sanitize_r02.txt); set SANITIZE=1 where it is allowed
if [ "${SANITIZE:-0}" = 1 ]; then for t in memcheck racecheck synccheck; do timeout 1500 compute-sanitizer --tool $t --print-limit 10 python tools/sanitize_case.py > gpurun_out/san_$t.txt 2>&1; echo "$t: $(grep -E 'SUMMARY' gpurun_out/san_$t.txt)"; done; fi
