mkdir -p gpurun_out
for args in "47232 0" "3000 0 24 32 6 1" "47232 0 120 160 52 1"; do timeout 20 tools/corr_micro_default $args || echo "micro $args rc=$?"; done 2>&1 | tee gpurun_out/r2h_micro.txt
timeout 120 compute-sanitizer --tool racecheck --print-limit 3 tools/corr_micro_default 3000 0 24 32 6 1 2>&1 | tail -4
timeout 120 compute-sanitizer --tool memcheck --print-limit 3 tools/corr_micro_default 47232 0 120 160 52 1 2>&1 | tail -3
for a in "wide 3000 128" "wide 2000 64" "wide 1500 256"; do timeout 30 python tools/corr_hang.py $a || echo "lib $a -> rc=$?"; done 2>&1
timeout 300 python -m pytest tests/test_gpu_corr.py tests/test_gpu_spd.py -q -x 2>&1 | tail -2
PYTHONFAULTHANDLER=1 timeout -s ABRT 300 python bench.py --no-e2e --no-cpu --json-out gpurun_out/r2h_bench.json > gpurun_out/r2h_bench.log 2> gpurun_out/r2h_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/r2h_bench.json'));print(d['ms_per_step'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()}, d['global_ba']['ms'])"
