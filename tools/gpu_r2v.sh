mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2v_gputest.log 2>&1; tail -2 gpurun_out/r2v_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -2
PYTHONFAULTHANDLER=1 timeout -s ABRT 600 python bench.py --json-out gpurun_out/r2v_bench.json > gpurun_out/r2v_bench.log 2> gpurun_out/r2v_bench.err; echo "bench rc=$?"
for t in memcheck racecheck synccheck; do timeout 1500 compute-sanitizer --tool $t --print-limit 10 python tools/sanitize_case.py > gpurun_out/r2v_san_$t.txt 2>&1; echo "$t: $(grep -E 'SUMMARY' gpurun_out/r2v_san_$t.txt)"; done
