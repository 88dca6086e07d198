./tools/gemm_bench 11264 128
./tools/gemm_bench 11264 256
make -s -C oracle _build/libgbem_oracle.so
timeout 1200 python -m pytest tests/test_gpu_assembly.py -x -q -m gpu 2>&1 | tail -3
timeout 300 python tools/profile_step.py 2 2 2>&1 | tail -1
