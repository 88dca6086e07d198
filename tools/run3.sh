set -x
make -s -C oracle _build/libgbem_oracle.so
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 300 python tools/profile_step.py 2 1 > gpurun_out/step.log 2>&1; cat gpurun_out/step.log
timeout 300 python tools/profile_step.py 2 0 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python tools/profile_step.py 2 0 > gpurun_out/ncu1.log 2>&1
echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_far|k_near_warp|k_potrf_diag|k_coplanar" -c 4 -o gpurun_out/prof_r01_asm python tools/profile_step.py 2 0 > gpurun_out/ncu2.log 2>&1
echo "ncu2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_nt" -s 3 -c 2 -o gpurun_out/prof_r01_gemm python tools/profile_step.py 2 0 > gpurun_out/ncu3.log 2>&1
echo "ncu3 rc=$?"
ls -la gpurun_out
