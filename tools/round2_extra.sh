#!/bin/bash
# Round-2 supplementary runs: config-2 bench line, full-size configs 3 and 4 (direct + sharded path
# at N = 1).  compute-sanitizer is closed on this GPU pool.
TAG=${1:-r02e}
mkdir -p gpurun_out
GBEM_NO_CLOCKS=1 python bench.py --config 2 --steps 20 --warmup 5 --no-sharded --no-cpu-baseline > gpurun_out/${TAG}_bench_config2.json 2> gpurun_out/${TAG}_bench_config2.err; echo "config2 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/${TAG}_bench_config2.json')); print(d['ms_per_step'], d['phases_ms'], d['roofline']['achieved'])"
timeout 1500 python tools/run_configs.py 3 4 > gpurun_out/${TAG}_configs.jsonl 2> gpurun_out/${TAG}_configs.err; echo "configs rc=$?"
cut -c1-1200 gpurun_out/${TAG}_configs.jsonl
