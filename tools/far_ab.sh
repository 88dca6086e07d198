# bench twice, far/assembly phases
for k in 1 2; do python bench.py --no-cpu-baseline --steps 8 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms']; print(round(d['ms_per_step'],3), round(p['far_ms'],3), round(p['assembly_ms'],3), round(p['factor_ms'],3))"; done
