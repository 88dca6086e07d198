./tools/solve_phase_bench 11340 6 | tail -3
for R in 1 6 16; do python tools/solve_bench.py 11340 $R 2>&1 | tail -1; done
timeout 600 python -m pytest tests/test_gpu_pcg.py tests/test_gpu_extract.py -x -q 2>&1 | tail -2
