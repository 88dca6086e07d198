make -s -C oracle _build/libgbem_oracle.so
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python __graft_entry__.py 2>&1 | tail -1
timeout 600 python bench.py --steps 5 --warmup 3 --cpu-seconds 15 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json; tail -2 gpurun_out/bench_ref.err
