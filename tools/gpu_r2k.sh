mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_synth.py -q -x > gpurun_out/r2k_synth.log 2>&1; tail -15 gpurun_out/r2k_synth.log
PYTHONFAULTHANDLER=1 timeout -s ABRT 600 python bench.py --json-out gpurun_out/r2k_bench.json > gpurun_out/r2k_bench.log 2> gpurun_out/r2k_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/r2k_bench.json'));print(d['ms_per_step'], d['input_generation_s'], d['global_ba']['ms'], d['e2e']['ms_per_step'], d['kernels']['corr']['ms_per_step'], d['kernels']['spd_factor']['ms_per_step'])"
