#!/bin/bash
# Measured pipeline for one round (run under gpurun from the repo root):
#   1. GPU tests, 2. bench (ours, then reference arm), 3. ncu launch list of the
#   same bench command, 4. one ncu --set full capture of each top kernel.
# Each ncu step runs only after the same command exited 0 without ncu.
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/tests_$TAG.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/tests_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; rc=$?; echo "bench rc=$rc"
cat gpurun_out/bench_$TAG.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
if [ $rc -eq 0 ]; then
  export GBEM_NO_GREEN=1  # ncu cannot profile kernels launched into green contexts
  timeout 1200 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain_$TAG.log 2>&1 && \
  timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list_$TAG.log 2>&1
  echo "launch list rc=$?"
  python tools/launch_summary.py gpurun_out/launches_$TAG.csv > gpurun_out/launch_summary_$TAG.txt 2>&1
  head -30 gpurun_out/launch_summary_$TAG.txt
  for KS in "k_syrk_gen:1" "k_far<\(int\)9>:1" "k_potrf_diag:200" "k_bwd_flow:2" "k_near_gl:2" "k_classify:2" "k_trsm_rows:200" "k_symv_upper:1"; do
    K=${KS%%:*}; S=${KS##*:}
    NAME=$(echo "$K" | tr -cd 'a-z_0-9')
    timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      --kernel-name "regex:$K" -s $S -c 1 -o gpurun_out/prof_${TAG}_$NAME -f \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_${TAG}_$NAME.log 2>&1
    echo "ncu $K rc=$?"
  done
  python tools/ncu_collect.py $TAG gpurun_out > gpurun_out/ncu_collect_$TAG.log 2>&1; echo "collect rc=$?"
  # keep the two dominant captures; the rest are summarised in gpurun_out/${TAG}_ncu_summary.txt
  for f in gpurun_out/prof_${TAG}_*.ncu-rep; do
    case "$f" in *k_syrk_gen*|*k_far*) ;; *) rm -f "$f" ;; esac
  done
  gzip -f gpurun_out/launches_$TAG.csv
  du -sh gpurun_out
fi
