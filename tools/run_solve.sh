timeout 900 python -m pytest tests/test_gpu_pcg.py tests/test_gpu_extract.py tests/test_gpu_assembly.py -x -q 2>&1 | tail -2
for R in 6 16 17 64; do python tools/solve_bench.py 11340 $R 2>&1 | tail -1; done
GBEM_SOLVE_BLOCKED_MIN=1 python tools/solve_bench.py 11340 6 2>&1 | tail -1
GBEM_SOLVE_BLOCKED_MIN=1 python tools/solve_bench.py 11340 1 2>&1 | tail -1
python tools/solve_bench.py 12025 64 2>&1 | tail -1
timeout 900 python tools/run_configs.py 3 4 2>&1 | tail -3
