mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2b_gputest.log 2>&1; tail -4 gpurun_out/r2b_gputest.log
PYTHONFAULTHANDLER=1 timeout -s ABRT 600 python bench.py --json-out gpurun_out/r2b_bench.json > gpurun_out/r2b_bench.log 2> gpurun_out/r2b_bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/r2b_bench.err
./tools/spd_micro > gpurun_out/r2b_spd_micro.txt 2>&1; cat gpurun_out/r2b_spd_micro.txt
DPV_SPD_PROFILE=1 timeout 300 python bench.py --no-e2e --no-global --no-cpu --steps 2 --warmup 3 > /dev/null 2> gpurun_out/r2b_spd_profile.txt; grep "\[spd\]" gpurun_out/r2b_spd_profile.txt | tail -8
