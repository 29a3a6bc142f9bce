timeout 600 python -m pytest tests/test_gpu_ba_parity.py tests/test_gpu_dist.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python tools/bench_edges.py --key-variants 0 > gpurun_out/edges.txt 2>&1
DPV_SCHUR_PAIRS=1 python tools/bench_edges.py --key-variants 0 >> gpurun_out/edges.txt 2>&1
