#!/bin/bash
mkdir -p gpurun_out
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/issue_bench tools/issue_bench.cu && /tmp/issue_bench | tee gpurun_out/issue_bench.log
