#!/bin/bash
# k_far CTAs-per-SM sweep: rebuild the assembly unit with GBEM_FAR_MINB=N, time configs 2 and 3
for mb in "$@"; do
  touch paper_2203_11733_b200/csrc/gbem_assembly.cu
  GBEM_NVCC_EXTRA="-DGBEM_FAR_MINB=$mb" python -m paper_2203_11733_b200.build > /dev/null 2>&1
  echo "GBEM_FAR_MINB=$mb"
  tools/far_ab.sh
done
touch paper_2203_11733_b200/csrc/gbem_assembly.cu
python -m paper_2203_11733_b200.build > /dev/null 2>&1
