# combined band+rest update vs separate launches
for v in 0 1; do if [ $v = 1 ]; then export GBEM_NO_COMBINED=1; fi; echo "no_combined=$v"; python bench.py --no-cpu-baseline --steps 8 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d['phases_ms']['factor_ms'],3), d['max_residual'])"; done
