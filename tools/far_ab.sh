#!/bin/bash
# far-field timing on configs 2 and 3 (assembly phases of one instrumented extraction step)
for c in 2 3; do
  python bench.py --config $c --steps 3 --warmup 2 --no-sharded --no-cpu-baseline | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms']
r=d['roofline'] if d['roofline']['kernel']=='k_far' else d['roofline_secondary']
print('config', d['config']['panels'], 'step', round(d['ms_per_step'],2), 'far', round(p['far_ms'],3), 'near', round(p['near_ms'],3), 'classify', round(p['classify_ms'],3), 'factor', round(p['factor_ms'],2), 'solve', round(p['solve_ms'],3), 'resid', round(p['residual_ms'],3), 'far_frac', round(r['frac'],4))"
done
