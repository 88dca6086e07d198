for R in 1 2 6 16 17; do python tools/solve_bench.py 11340 $R 2>&1 | tail -1; done
for d in 1 2 4; do GBEM_SOLVE_DBG=$d python tools/solve_bench.py 11340 6 2>&1 | tail -1; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
