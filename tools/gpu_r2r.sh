mkdir -p gpurun_out
for g in 0 4 5 8; do
if [ $g = 0 ]; then unset DPV_SPD_CHAINS; else export DPV_SPD_CHAINS=$g; fi
DPV_PLAN_DEBUG=1 timeout 300 python bench.py --no-e2e --no-global --no-cpu --steps 4 --warmup 3 --json-out gpurun_out/r2r_g$g.json > /dev/null 2> gpurun_out/r2r_g$g.err
grep "spd plan n=" gpurun_out/r2r_g$g.err | head -1 | cut -c1-200
python -c "import json;d=json.load(open('gpurun_out/r2r_g$g.json'));print('G=$g', d['ms_per_step'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items() if k.startswith('spd')})"
done
