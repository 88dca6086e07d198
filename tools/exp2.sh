#!/bin/bash
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k_far_orth<.int.2, .int.3, .int.3>" --launch-count 1 \
  -o gpurun_out/exp2_far_orth233 -f python tools/prof_assembly.py 3 1 > gpurun_out/exp2_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/exp2_ncu.log
