set -x
python -m pytest tests -m gpu -q -x > gpurun_out/r2_gputest2.log 2>&1; tail -3 gpurun_out/r2_gputest2.log
python bench.py --json-out gpurun_out/r2_bench2.json > gpurun_out/r2_bench2.log 2>&1; tail -c 600 gpurun_out/r2_bench2.log
./tools/spd_micro > gpurun_out/r2_spd_micro.txt 2>&1; cat gpurun_out/r2_spd_micro.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_case.py > gpurun_out/r2_san_memcheck.txt 2>&1; tail -5 gpurun_out/r2_san_memcheck.txt
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_case.py > gpurun_out/r2_san_racecheck.txt 2>&1; tail -5 gpurun_out/r2_san_racecheck.txt
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_case.py > gpurun_out/r2_san_synccheck.txt 2>&1; tail -5 gpurun_out/r2_san_synccheck.txt
python bench.py --impl reference > gpurun_out/r2_bench2_ref.log 2>&1; tail -c 800 gpurun_out/r2_bench2_ref.log
