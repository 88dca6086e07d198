timeout 600 python tools/asm_only.py 5 0.25 4 2>&1 | tail -3
timeout 900 python tools/asm_only.py 5 1.0 16 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_assembly.py -x -q -m gpu 2>&1 | tail -2
