timeout 300 python tools/profile_step.py 2 0 > gpurun_out/plain9.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_solve_coop -c 1 -o gpurun_out/prof_solve python tools/profile_step.py 2 0 > gpurun_out/ncu9.log 2>&1
echo rc=$?
