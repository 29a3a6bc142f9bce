mkdir -p gpurun_out
for v in 0 1 2 3 4 5; do
DPV_KB_EXP=$v timeout 300 python bench.py --no-e2e --no-global --no-cpu --steps 4 --warmup 3 --json-out gpurun_out/r2q_kb$v.json > /dev/null 2>&1
python -c "import json;d=json.load(open('gpurun_out/r2q_kb$v.json'));print('variant $v', d['ms_per_step'], d['kernels']['key_blocks']['ms_per_step'])"
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_corr_tma -s 2 -c 1 -o gpurun_out/r2q_corr python tools/bench_corr.py > /dev/null 2>&1; echo "ncu rc=$?"
