mkdir -p gpurun_out
timeout 180 compute-sanitizer --tool memcheck --print-limit 5 tools/corr_micro_200_4_1_3 47232 0 120 160 52 1 > gpurun_out/r2g_memcheck.txt 2>&1; head -60 gpurun_out/r2g_memcheck.txt
timeout 180 compute-sanitizer --tool racecheck --print-limit 5 tools/corr_micro_200_4_1_3 3000 0 24 32 6 1 > gpurun_out/r2g_racecheck.txt 2>&1; head -40 gpurun_out/r2g_racecheck.txt
timeout 180 compute-sanitizer --tool synccheck --print-limit 5 tools/corr_micro_200_4_1_3 3000 0 24 32 6 1 > gpurun_out/r2g_synccheck.txt 2>&1; head -40 gpurun_out/r2g_synccheck.txt
