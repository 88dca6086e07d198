timeout 300 python tools/profile_step.py 2 2 2>&1 | tail -1
timeout 300 python tools/profile_step.py 3 1 2>&1 | tail -1
make -s -C oracle _build/libgbem_oracle.so
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
