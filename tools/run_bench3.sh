for i in 1 2 3; do GBEM_NO_CLOCKS=1 python bench.py 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['seconds_per_extraction'], d['phases_ms']['factor_ms'])"; done
python bench.py --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['seconds_per_extraction'], d['clocks'])"
