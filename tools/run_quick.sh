# quick iteration: parity tests + factor profile + bench phases (scratch driver)
mkdir -p gpurun_out
T=${1:-q}
timeout 600 python -m pytest tests/test_gpu_pairs.py tests/test_gpu_assembly.py tests/test_gpu_extract.py tests/test_gpu_pcg.py tests/test_gpu_golden.py -x -q > gpurun_out/tests_$T.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/tests_$T.log
GBEM_FACTOR_PROFILE=1 timeout 300 python tools/solve_bench.py 11340 6 > gpurun_out/fprof_$T.log 2>&1; tail -2 gpurun_out/fprof_$T.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_$T.json')); print(d['ms_per_step'], d['phases_ms'], d['e2e']['seconds_per_extraction'], d['assembly']['far_evals'], d['roofline_secondary']['frac'], d['max_residual'])"
