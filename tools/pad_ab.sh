#!/bin/bash
# A/B of the update kernel's shared-memory slab padding (fragment-load bank conflicts)
mkdir -p gpurun_out
for w in 8 4 12; do
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -DGBEM_GEN_PAD=$w -o /tmp/gemm_bench_p$w tools/gemm_bench.cu -lcublas
echo "PAD=$w"
for shape in "26000 1536" "33000 640" "12000 1024" "8000 256"; do /tmp/gemm_bench_p$w $shape | grep -E "gen 64x64 w2x2 st2 min4|max_abs"; done
done 2>&1 | tee gpurun_out/pad_ab.log
for w in 8 4; do
ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_ld.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,gpu__time_duration.sum --clock-control none -k regex:k_syrk_gen --launch-skip 2 --launch-count 1 /tmp/gemm_bench_p$w 26000 1536 2>&1 | grep -E "l1tex|smsp|sm__|gpu__time" | tee -a gpurun_out/pad_ab.log
done
