#!/bin/bash
# ceiling experiment: the update kernel without its barrier / without its loads (results invalid, timing only)
mkdir -p gpurun_out
for v in "" "-DGBEM_EXP_NOSYNC" "-DGBEM_EXP_NOSYNC -DGBEM_EXP_NOLOAD"; do
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -DGBEM_GEN_PAD=4 $v -o /tmp/gemm_bench_x tools/gemm_bench.cu -lcublas
echo "VARIANT=$v"
for shape in "26000 1536" "12000 1024" "8000 256"; do /tmp/gemm_bench_x $shape | grep -E "gen 64x64 w2x2 st2 min4|gen 64x64 w2x2 st3 min4|cublasDsyrk"; done
done 2>&1 | tee gpurun_out/sync_ab.log
