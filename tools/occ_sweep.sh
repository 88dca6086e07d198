# sweep of GBEM_OCC_ROWS (rest-update occupancy cap near the end of the factor)
for r in 0 3000 6000 9000 12000 20000; do echo "occ_rows=$r"; GBEM_OCC_ROWS=$r python bench.py --no-cpu-baseline --steps 8 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d['phases_ms']['factor_ms'],3))"; done
