mkdir -p gpurun_out
for b in tools/corr_micro_*; do timeout 60 $b 47232 0; done 2>&1 | tee gpurun_out/r2e_corr_variants.txt
./tools/spd_micro > gpurun_out/r2e_spd_micro.txt 2>&1; ./tools/spd_micro_v2 >> gpurun_out/r2e_spd_micro.txt 2>&1; ./tools/spd_micro_v3 >> gpurun_out/r2e_spd_micro.txt 2>&1; cat gpurun_out/r2e_spd_micro.txt
timeout 600 python -m pytest tests/test_gpu_corr.py tests/test_gpu_spd.py tests/test_gpu_ba_parity.py -q -x > gpurun_out/r2e_tests.log 2>&1; tail -3 gpurun_out/r2e_tests.log
timeout 120 python tools/bench_corr.py 2>&1 | tail -2
PYTHONFAULTHANDLER=1 timeout -s ABRT 300 python bench.py --no-e2e --no-cpu --json-out gpurun_out/r2e_bench.json > gpurun_out/r2e_bench.log 2> gpurun_out/r2e_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/r2e_bench.json'));print(d['ms_per_step'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()}, d['global_ba']['ms'])"
