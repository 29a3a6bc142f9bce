mkdir -p gpurun_out
for b in tools/corr_micro_default tools/corr_micro_np*; do timeout 20 $b 47232 0 || echo "$b rc=$?"; done 2>&1 | tee gpurun_out/r2i_micro.txt
timeout 120 compute-sanitizer --tool racecheck --print-limit 2 tools/corr_micro_default 3000 0 24 32 6 0 2>&1 | tail -3
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_case.py > gpurun_out/r2i_san_memcheck.txt 2>&1; tail -4 gpurun_out/r2i_san_memcheck.txt
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_case.py > gpurun_out/r2i_san_racecheck.txt 2>&1; tail -4 gpurun_out/r2i_san_racecheck.txt
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_case.py > gpurun_out/r2i_san_synccheck.txt 2>&1; tail -4 gpurun_out/r2i_san_synccheck.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spd_factor|k_assemble_edges_stg|k_key_blocks|k_corr_tma|k_incidences2" -s 40 -c 6 -o gpurun_out/r2i_full python bench.py --steps 2 --warmup 3 --no-e2e --no-global --no-cpu --no-graph > gpurun_out/r2i_ncu.log 2>&1; tail -3 gpurun_out/r2i_ncu.log
