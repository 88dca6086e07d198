#!/bin/bash
# ncu --set full capture of the trailing-update kernel (k_syrk_bulk<16, 3, 4, true>, the factorisation's) at a super-block shape, summarised on the box
mkdir -p gpurun_out
M=${1:-26000}; K=${2:-1536}
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -o /tmp/gemm_bench tools/gemm_bench.cu -lcublas
GEMM_BENCH_SHORT=1 /tmp/gemm_bench $M $K | grep -E "gen 64x64 w2x2 st2 min4|bulk-split bks16|cublas" 
GEMM_BENCH_BULK_ONLY=1 ncu --set full --import-source on --clock-control none -k regex:k_syrk_bulk --launch-skip 2 --launch-count 1 \
  -o gpurun_out/syrk_${M}_${K} -f /tmp/gemm_bench $M $K > gpurun_out/syrk_ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/syrk_${M}_${K}.ncu-rep > gpurun_out/syrk_${M}_${K}_summary.txt
python tools/ncu_stalls.py gpurun_out/syrk_${M}_${K}.ncu-rep 25 >> gpurun_out/syrk_${M}_${K}_summary.txt
ncu -i gpurun_out/syrk_${M}_${K}.ncu-rep --page details 2>/dev/null | grep -E "Issue Slots Busy|One or More Eligible|No Eligible|Active Warps Per Scheduler|Eligible Warps Per|Cycles Per Issued|Executed Ipc Active|highest-utilized|DRAM Throughput|L2 Cache Throughput|L1/TEX Cache Throughput|Achieved Occupancy|Bank conflict|bank conflict" >> gpurun_out/syrk_${M}_${K}_summary.txt
rm -f gpurun_out/syrk_${M}_${K}.ncu-rep
cat gpurun_out/syrk_${M}_${K}_summary.txt | cut -c1-170
