#!/bin/bash
# assembly A/B driver: phase times on configs 2, 3 (and 5 with arg "5"), then the assembly parity tests
mkdir -p gpurun_out
python tools/far_ab.py ${1:-2,3} 4 2>&1 | tee gpurun_out/far_ab.log
timeout 1200 python -m pytest tests/test_gpu_pairs.py tests/test_gpu_assembly.py tests/test_gpu_near_contact.py tests/test_gpu_golden.py tests/test_gpu_configs.py tests/test_gpu_block.py -m gpu -x -q > gpurun_out/far_ab_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/far_ab_tests.log
