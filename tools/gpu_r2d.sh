mkdir -p gpurun_out
for b in tools/corr_micro_*; do timeout 60 $b 47232 0; timeout 60 $b 47232 1; done 2>&1 | tee gpurun_out/r2d_corr_variants.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_corr_tma -s 3 -c 1 -o gpurun_out/r2d_corr_full tools/corr_micro_200_4_1 47232 0 > gpurun_out/r2d_ncu.log 2>&1; tail -2 gpurun_out/r2d_ncu.log
