mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_corr.py -q -x > gpurun_out/r2c_corrtest.log 2>&1; tail -2 gpurun_out/r2c_corrtest.log
timeout 120 python tools/bench_corr.py > gpurun_out/r2c_bench_corr.txt 2>&1; tail -5 gpurun_out/r2c_bench_corr.txt
for i in 1 2 3; do
PYTHONFAULTHANDLER=1 timeout -s ABRT 240 python bench.py --json-out gpurun_out/r2c_bench$i.json > gpurun_out/r2c_bench$i.log 2> gpurun_out/r2c_bench$i.err; echo "bench $i rc=$?"; grep -v "^\[bench" gpurun_out/r2c_bench$i.err | tail -30
python -c "import json;d=json.load(open('gpurun_out/r2c_bench$i.json'));print(d['ms_per_step'], d['kernels']['corr']['ms_per_step'], d['global_ba']['ms'])"
done
