timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2 3; do python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), [round(x,2) for x in d['step_ms']], round(d['e2e']['seconds_per_extraction']*1e3,2), d['clocks']['samples_in_timed_region'])"; done
