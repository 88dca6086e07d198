timeout 300 python tools/profile_step.py 2 0 > gpurun_out/plain13.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_potrf_diag -s 10 -c 1 -o gpurun_out/prof_potrf python tools/profile_step.py 2 0 > gpurun_out/ncu13.log 2>&1
echo rc=$?
