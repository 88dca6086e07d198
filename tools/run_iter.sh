# one build -> measure iteration under gpurun (scratch driver; outputs in gpurun_out/)
mkdir -p gpurun_out
T=${1:-c}

timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests_$T.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/tests_$T.log
GBEM_FACTOR_PROFILE=1 timeout 300 python tools/solve_bench.py 11340 6 > gpurun_out/fprof_$T.log 2>&1; tail -2 gpurun_out/fprof_$T.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_$T.json')); print(d['ms_per_step'], d['phases_ms'], d['e2e']['seconds_per_extraction'], d['max_residual'], d['roofline']['frac'])"
