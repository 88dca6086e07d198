#!/bin/bash
# factor time under the factorisation's scheduling knobs (experiments): factor_knobs.sh [config] ; KNOBS="VAR=val ..." overrides the list
mkdir -p gpurun_out
IFS='|' read -ra LIST <<< "${KNOBS:-A=1|GBEM_SUPERBLOCK=5|GBEM_SUPERBLOCK=10|GBEM_SB_SCHED=12:14000,8:9000,5:6000,3:3500,2:0|GBEM_SB_SCHED=12:12000,8:8000,5:5000,3:3000,2:0|GBEM_SB_SCHED=16:20000,12:12000,8:8000,5:5000,3:3000,2:0|GBEM_SB_SCHED=10:10000,6:6000,4:4000,2:0|GBEM_SB_SCHED=12:16000,10:12000,8:9000,6:7000,4:5000,3:3500,2:0}"
for v in "${LIST[@]}"; do
env $v GBEM_NO_CLOCKS=1 python bench.py --config ${1:-3} --steps 3 --warmup 2 --no-sharded --no-cpu-baseline > gpurun_out/knob.json 2> gpurun_out/knob.err; python -c "
import json; d=json.load(open('gpurun_out/knob.json')); print('$v', d['ms_per_step'], d['phases_ms']['factor_ms'], d['roofline']['achieved'], d['max_residual'])"
done | tee gpurun_out/factor_knobs.log
