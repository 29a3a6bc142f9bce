DPV_SPD_PROFILE=1 timeout 300 python bench.py --no-e2e --no-global --no-cpu --steps 2 --warmup 3 > /dev/null 2> gpurun_out/r2t_prof.txt; grep "\[spd\]" gpurun_out/r2t_prof.txt | tail -6
