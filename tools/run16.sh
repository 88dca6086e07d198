timeout 300 python tools/profile_step.py 2 0 > gpurun_out/plain16.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_far|k_near_gl" -c 2 -o gpurun_out/prof_far python tools/profile_step.py 2 0 > gpurun_out/ncu16.log 2>&1
echo rc=$?
