./tools/potrf_bench
make -s -C oracle _build/libgbem_oracle.so
timeout 1200 python -m pytest tests/test_gpu_assembly.py tests/test_gpu_extract.py -x -q -m gpu 2>&1 | tail -2
timeout 300 python tools/profile_step.py 2 2 2>&1 | tail -1
timeout 300 python tools/profile_step.py 3 1 2>&1 | tail -1
