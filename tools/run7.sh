make -s -C oracle _build/libgbem_oracle.so
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 300 python tools/profile_step.py 2 2 2>&1 | tail -1
timeout 300 python tools/profile_step.py 3 1 2>&1 | tail -1
timeout 600 python bench.py --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err; tail -2 gpurun_out/bench_r01b.err; cat gpurun_out/bench_r01b.json
