timeout 300 python -m pytest tests/test_gpu_corr.py -x -q > gpurun_out/corr_test.log 2>&1; echo corrtest=$?
timeout 300 python tools/bench_corr.py > gpurun_out/corr.txt 2>&1; echo bc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_corr_tma -c 1 -o gpurun_out/corr_tma python tools/bench_corr.py --reps 1 > gpurun_out/corr_ncu.log 2>&1; echo ncu=$?
