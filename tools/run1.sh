set -x
make -s -C oracle _build/libgbem_oracle.so 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_pairs.py tests/test_gpu_assembly.py -x -q -m gpu 2>&1 | tail -40
