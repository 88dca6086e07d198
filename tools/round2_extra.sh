#!/bin/bash
# Round-2 supplementary runs: config-2 bench line, compute-sanitizer on the look-ahead backward
# sweep, full-size configs 3 and 4 (direct + sharded path at N = 1).
mkdir -p gpurun_out
GBEM_NO_CLOCKS=1 python bench.py --config 2 --steps 20 --warmup 5 --no-sharded --no-cpu-baseline > gpurun_out/r02c_bench_config2.json 2> gpurun_out/r02c_bench_config2.err; echo "config2 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r02c_bench_config2.json')); print(d['ms_per_step'], d['phases_ms'], d['roofline']['achieved'])"
timeout 1200 compute-sanitizer --tool memcheck python tools/sanitize_bwd.py > gpurun_out/r02c_sanitize_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -4 gpurun_out/r02c_sanitize_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck python tools/sanitize_bwd.py > gpurun_out/r02c_sanitize_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -4 gpurun_out/r02c_sanitize_racecheck.log
timeout 1500 python tools/run_configs.py 3 4 > gpurun_out/r02c_configs.jsonl 2> gpurun_out/r02c_configs.err; echo "configs rc=$?"
cut -c1-1200 gpurun_out/r02c_configs.jsonl
