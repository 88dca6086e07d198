python tools/matvec_bench.py 2>&1 | tail -5
python -m pytest tests/test_gpu_pcg.py tests/test_gpu_extract.py tests/test_gpu_assembly.py -q -x -m gpu 2>&1 | tail -15
