set -x
make -s -C oracle _build/libgbem_oracle.so
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -30
python __graft_entry__.py 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
