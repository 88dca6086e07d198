python bench.py --config 2 --steps 3 --warmup 2 --no-sharded --no-cpu-baseline | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms']; print('step', round(d['ms_per_step'],2), 'factor', round(p['factor_ms'],2))"
