#!/bin/bash
# far-field setup cost: time k_far with the node loop compiled out (results wrong)
touch paper_2203_11733_b200/csrc/gbem_assembly.cu
GBEM_NVCC_EXTRA="-DGBEM_FAR_SETUP_ONLY" python -m paper_2203_11733_b200.build > /dev/null 2>&1
python tools/prof_assembly.py 2 2 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read().strip().splitlines()[-1]); print('setup-only far_ms', d['ms_far'])"
touch paper_2203_11733_b200/csrc/gbem_assembly.cu
python -m paper_2203_11733_b200.build > /dev/null 2>&1
python tools/prof_assembly.py 2 2 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read().strip().splitlines()[-1]); print('full far_ms', d['ms_far'])"
