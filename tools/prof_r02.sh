#!/bin/bash
# Round-2 profiling session (one GPU): launch list of the bench step (config 3,
# single-partition factor: ncu cannot profile kernels launched into green
# contexts), full captures of the trailing update at a config-3 K = 256 shape,
# the sharded solve's row-block product and the dominant far-field kernel.
set -x
mkdir -p gpurun_out
export GBEM_NO_CLOCKS=1
GBEM_NO_GREEN=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_launches.csv python bench.py --steps 1 --warmup 1 --no-sharded --no-cpu-baseline \
  > gpurun_out/r02_launch_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_syrk_gen --launch-skip 2 --launch-count 1 \
  -o gpurun_out/r02_syrk_k256 tools/gemm_bench 16384 256 > gpurun_out/r02_syrk.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_gemm_nt_sk --launch-skip 13 --launch-count 1 \
  -o gpurun_out/r02_gemm_sk tools/pcg_gemm_bench 12032 96200 > gpurun_out/r02_gemm_sk.log 2>&1
ncu --set full --import-source on --clock-control none -k "regex:k_far<9>" --launch-count 1 \
  -o gpurun_out/r02_kfar9_c3 python tools/prof_assembly.py 3 1 > gpurun_out/r02_kfar_c3.log 2>&1
ls -la gpurun_out
