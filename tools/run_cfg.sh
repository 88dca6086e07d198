timeout 900 python -m pytest tests/test_gpu_configs.py -x -q 2>&1 | tail -5
timeout 1800 python tools/run_configs.py 3 4 5 2>&1 | tail -6
