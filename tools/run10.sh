timeout 300 python tools/profile_step.py 2 0 > gpurun_out/plain10.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01b.csv python tools/profile_step.py 2 0 > gpurun_out/ncu10.log 2>&1
echo rc=$?
