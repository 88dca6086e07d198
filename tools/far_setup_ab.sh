#!/bin/bash
# far-field cost split (config-2 k_far device time; results of the variants are wrong):
#   GBEM_FAR_SETUP_ONLY=1: queue / plan / panel loads, decode, store only
#   GBEM_FAR_SETUP_ONLY=2: + the three node lists (far_list + emit_list)
#   full kernel
for v in 1 2; do
  touch paper_2203_11733_b200/csrc/gbem_assembly.cu
  GBEM_NVCC_EXTRA="-DGBEM_FAR_SETUP_ONLY=$v" python -m paper_2203_11733_b200.build > /dev/null 2>&1
  python tools/prof_assembly.py 2 2 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read().strip().splitlines()[-1]); print('variant $v far_ms', d['ms_far'])"
done
touch paper_2203_11733_b200/csrc/gbem_assembly.cu
python -m paper_2203_11733_b200.build > /dev/null 2>&1
python tools/prof_assembly.py 2 2 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read().strip().splitlines()[-1]); print('full far_ms', d['ms_far'])"
