#!/bin/bash
# scratch experiment driver (one gpurun call)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pairs.py tests/test_gpu_assembly.py tests/test_gpu_near_contact.py tests/test_gpu_golden.py tests/test_gpu_configs.py -m gpu -x -q > gpurun_out/exp1_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/exp1_tests.log
python tools/far_ab.py 2,3 4 2>&1 | tee gpurun_out/exp1_far_minb4.log
for mb in 5 6; do
  touch paper_2203_11733_b200/csrc/gbem_assembly.cu
  GBEM_NVCC_EXTRA="-DGBEM_FAST_MINB=$mb" python -m paper_2203_11733_b200.build > /dev/null 2>&1
  echo "GBEM_FAST_MINB=$mb"
  python tools/far_ab.py 2,3 4 2>&1 | tee gpurun_out/exp1_far_minb$mb.log
done
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -o /tmp/gemm_bench tools/gemm_bench.cu -lcublas 2> gpurun_out/exp1_gemm_build.log
for shape in "20000 640" "20000 256" "8000 640"; do /tmp/gemm_bench $shape; done 2>&1 | tee gpurun_out/exp1_gemm.log
ncu --set full --import-source on --clock-control none -k regex:k_syrk_gen --launch-skip 2 --launch-count 1 \
  -o gpurun_out/exp1_syrk_k640 -f /tmp/gemm_bench 20000 640 > gpurun_out/exp1_syrk_ncu.log 2>&1; echo "ncu rc=$?"
