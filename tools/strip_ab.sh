#!/bin/bash
mkdir -p gpurun_out
for w in 0 16 8 32; do
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -DGBEM_SYRK_STRIP=$w -o /tmp/gemm_bench_$w tools/gemm_bench.cu -lcublas
echo "STRIP=$w"
for shape in "26000 1536" "33000 640" "12000 1024"; do /tmp/gemm_bench_$w $shape | grep -E "gen 64x64 w2x2 st2 min4|max_abs"; done
done 2>&1 | tee gpurun_out/strip_ab.log
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_syrk_gen --launch-skip 2 --launch-count 1 /tmp/gemm_bench_16 26000 1536 2>&1 | grep -E "dram__|gpu__time" | tee -a gpurun_out/strip_ab.log
KNOBS="A=1" bash tools/factor_knobs.sh 3
KNOBS="A=1" bash tools/factor_knobs.sh 2
