python tools/solve_bench.py 11340 6 2>&1 | tail -1
python tools/solve_bench.py 25000 17 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
GBEM_NO_CLOCKS=1 python bench.py 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phases_ms'], d['max_residual'], d['roofline']['frac'])"
