mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pgo.py tests/test_gpu_corr.py tests/test_gpu_spd.py -q -x > gpurun_out/r2j_tests.log 2>&1; tail -15 gpurun_out/r2j_tests.log
timeout 900 python -m pytest tests/test_gpu_reference_suite.py -q -x -k posegraph > gpurun_out/r2j_refsuite.log 2>&1; tail -15 gpurun_out/r2j_refsuite.log
timeout 120 compute-sanitizer --tool racecheck --print-limit 3 tools/corr_micro_default 3000 0 24 32 6 1 2>&1 | tail -3
timeout 1200 compute-sanitizer --tool racecheck --print-limit 5 python tools/sanitize_case.py > gpurun_out/r2j_san_racecheck.txt 2>&1; tail -3 gpurun_out/r2j_san_racecheck.txt
