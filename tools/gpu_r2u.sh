mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_spd.py tests/test_gpu_ba_parity.py tests/test_gpu_cfg_parity.py -q -x 2>&1 | tail -1
PYTHONFAULTHANDLER=1 timeout -s ABRT 600 python bench.py --no-e2e --no-cpu --json-out gpurun_out/r2u_bench.json > /dev/null 2> gpurun_out/r2u_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/r2u_bench.json'));print(d['ms_per_step'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items() if k.startswith('spd')}, d['global_ba']['ms'])"
DPV_SPD_PROFILE=1 timeout 300 python bench.py --no-e2e --no-global --no-cpu --steps 2 --warmup 3 > /dev/null 2> gpurun_out/r2u_prof.txt; grep "\[spd\]" gpurun_out/r2u_prof.txt | tail -4
