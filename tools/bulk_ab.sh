#!/bin/bash
# trailing update: bulk-copy staged kernel (k_syrk_bulk) against the cp.async kernel and cublasDsyrk
mkdir -p gpurun_out
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -o /tmp/gemm_bench tools/gemm_bench.cu -lcublas
for shape in "26000 1536" "33000 640" "12000 1024" "8000 256" "4000 256"; do timeout 300 env GEMM_BENCH_SHORT=1 /tmp/gemm_bench $shape | grep -E "gen 64x64 w2x2 st2 min4|bulk|max_abs|cublasDsyrk"; done 2>&1 | tee gpurun_out/bulk_ab.log
