#!/bin/bash
# scratch: A/B of assembly build variants.  usage: exp3.sh "<flags A>" "<flags B>" ...
mkdir -p gpurun_out
for fl in "$@"; do
  touch paper_2203_11733_b200/csrc/gbem_assembly.cu
  GBEM_NVCC_EXTRA="$fl" python -m paper_2203_11733_b200.build > /dev/null 2>&1 || echo "build failed"
  echo "FLAGS=$fl"
  python tools/far_ab.py 2,3 4 2>&1
done | tee gpurun_out/exp3.log
touch paper_2203_11733_b200/csrc/gbem_assembly.cu
python -m paper_2203_11733_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_pairs.py tests/test_gpu_assembly.py tests/test_gpu_near_contact.py tests/test_gpu_golden.py tests/test_gpu_configs.py -m gpu -x -q > gpurun_out/exp3_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/exp3_tests.log
