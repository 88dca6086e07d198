./tools/gemm_bench 11264 128 > gpurun_out/gb.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gemm_nt -s 2 -c 1 -o gpurun_out/prof_gemm_bench ./tools/gemm_bench 11264 128 > gpurun_out/ncu_gb.log 2>&1
echo rc=$?
