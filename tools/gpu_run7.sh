export DPV_PLAN_DEBUG=1
timeout 300 python -m pytest tests/test_gpu_spd.py tests/test_gpu_ba_parity.py tests/test_gpu_dist.py -x -q > gpurun_out/spd_test.log 2>&1; echo spd=$?
for G in 0; do
  if [ $G = 0 ]; then unset DPV_SPD_CHAINS; else export DPV_SPD_CHAINS=$G; fi
  DPV_SPD_PROFILE=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-global --no-e2e --json-out gpurun_out/bench_g$G.json > gpurun_out/bench_g$G.log 2>&1; echo bench$G=$?
done
