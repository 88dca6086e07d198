# ncu --set full of one kernel launch during bench (scratch driver): $1 tag, $2 kernel regex, $3 skip
mkdir -p gpurun_out
T=$1; K=$2; S=${3:-0}
GBEM_NO_GREEN=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  --kernel-name "regex:$K" -s $S -c 1 -o gpurun_out/prof_$T -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$T.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_$T.log
