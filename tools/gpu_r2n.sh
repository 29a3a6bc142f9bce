mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ba_parity.py tests/test_gpu_cfg_parity.py tests/test_gpu_batch.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r2n_tests.log 2>&1; tail -3 gpurun_out/r2n_tests.log
PYTHONFAULTHANDLER=1 timeout -s ABRT 600 python bench.py --no-e2e --no-cpu --json-out gpurun_out/r2n_bench.json > /dev/null 2> gpurun_out/r2n_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/r2n_bench.json'));print(d['ms_per_step'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()}, d['global_ba']['ms'])"
