#!/bin/bash
# Round-2 measured pipeline (run under gpurun from the repo root; TAG names the outputs):
#   1. GPU tests, 2. bench (ours, then the reference arm), 3. ncu launch list of the same
#   bench step (config 3, single-partition factor: ncu cannot profile kernels launched into
#   green contexts), 4. ncu --set full captures of the dominant far-field kernels and the
#   classifier from one config-3 assembly.
# Each ncu step runs only after the same command exited 0 without ncu.
TAG=${1:-r02b}
SKIP_TESTS=${2:-0}
mkdir -p gpurun_out
if [ "$SKIP_TESTS" != "1" ]; then
  timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/tests_$TAG.log 2>&1; echo "tests rc=$?"
  tail -3 gpurun_out/tests_$TAG.log
fi
timeout 1500 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; rc=$?; echo "bench rc=$rc"
cut -c1-1500 gpurun_out/bench_$TAG.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
if [ $rc -eq 0 ]; then
  export GBEM_NO_CLOCKS=1
  GBEM_NO_GREEN=1 timeout 900 python bench.py --steps 1 --warmup 1 --no-sharded --no-cpu-baseline > gpurun_out/plain_$TAG.log 2>&1 && \
  GBEM_NO_GREEN=1 timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 1 --no-sharded --no-cpu-baseline \
    > gpurun_out/ncu_list_$TAG.log 2>&1
  echo "launch list rc=$?"
  python tools/launch_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launch_summary.txt 2>&1
  head -40 gpurun_out/${TAG}_launch_summary.txt
  timeout 300 python tools/prof_assembly.py 3 1 > gpurun_out/asm_plain_$TAG.log 2>&1 && \
  SECS="--section SpeedOfLight --section ComputeWorkloadAnalysis --section Occupancy --section LaunchStats --section WarpStateStats --section SchedulerStats --section MemoryWorkloadAnalysis"
  # every far-field launch of the assembly's first chunk with the pipe / occupancy / stall sections (no source)
  timeout 1200 ncu $SECS --clock-control none --kernel-name-base demangled --kernel-name "regex:k_far" -c 80 \
    -o gpurun_out/prof_${TAG}_far_all -f python tools/prof_assembly.py 3 1 > gpurun_out/ncu_${TAG}_far_all.log 2>&1
  echo "ncu far_all rc=$?"
  python tools/ncu_far_all.py gpurun_out/prof_${TAG}_far_all.ncu-rep 80 > gpurun_out/${TAG}_ncu_far_kernels.txt 2>&1
  rm -f gpurun_out/prof_${TAG}_far_all.ncu-rep
  : > gpurun_out/${TAG}_ncu_summary.txt
  for KS in "k_classify<.bool.0>:classify0" "k_classify<.bool.1>:classify1" "k_far_orth<.int.2, .int.3, .int.3>:far_orth233"; do
    K=${KS%%:*}; NAME=${KS##*:}
    timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      --kernel-name "regex:$K" -c 1 -o gpurun_out/prof_${TAG}_$NAME -f \
      python tools/prof_assembly.py 3 1 > gpurun_out/ncu_${TAG}_$NAME.log 2>&1
    echo "ncu $K rc=$?"
    python tools/ncu_summary.py gpurun_out/prof_${TAG}_$NAME.ncu-rep >> gpurun_out/${TAG}_ncu_summary.txt 2>&1
    python tools/ncu_stalls.py gpurun_out/prof_${TAG}_$NAME.ncu-rep 15 >> gpurun_out/${TAG}_ncu_summary.txt 2>&1
    ncu -i gpurun_out/prof_${TAG}_$NAME.ncu-rep --page details 2>/dev/null | grep -E "Issue Slots Busy|One or More Eligible|Active Warps Per Scheduler|Eligible Warps Per|Cycles Per Issued|Executed Ipc Active|highest-utilized|DRAM Throughput|Achieved Occupancy" >> gpurun_out/${TAG}_ncu_summary.txt
    case "$NAME" in far_orth233) ;; *) rm -f gpurun_out/prof_${TAG}_$NAME.ncu-rep ;; esac
  done
  # the look-ahead backward sweep's kernels (graph nodes) from one bench step
  GBEM_NO_GREEN=1 timeout 900 ncu $SECS --clock-control none --kernel-name-base demangled --kernel-name "regex:k_bwd_step|k_bwd_bulk" -s 20 -c 4 \
    -o gpurun_out/prof_${TAG}_bwd -f python bench.py --steps 1 --warmup 0 --no-sharded --no-cpu-baseline > gpurun_out/ncu_${TAG}_bwd.log 2>&1
  echo "ncu bwd rc=$?"
  python tools/ncu_summary.py gpurun_out/prof_${TAG}_bwd.ncu-rep >> gpurun_out/${TAG}_ncu_summary.txt 2>&1
  rm -f gpurun_out/prof_${TAG}_bwd.ncu-rep
  gzip -f gpurun_out/${TAG}_launches.csv
  du -sh gpurun_out
fi
