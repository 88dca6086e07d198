#!/bin/bash
for d in 0 1 2 3; do
echo "GBEM_FACTOR_DBG=$d"
GBEM_FACTOR_DBG=$d GBEM_NO_CLOCKS=1 GBEM_FACTOR_PROFILE=1 python bench.py --config 3 --steps 1 --warmup 1 --no-sharded --no-cpu-baseline 2>&1 >/dev/null | grep -E "totals|sb   0|sb   8 " | head -6
done
