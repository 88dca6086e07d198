./tools/potrf_bench > gpurun_out/pb15.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_potrf_diag -s 1 -c 1 -o gpurun_out/prof_potrf2 ./tools/potrf_bench > gpurun_out/ncu15.log 2>&1
echo rc=$?
