one() { timeout 600 python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu --no-check --e2e-skew $1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('skew $1', 'value', round(d['value']), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],1))"; }
for rep in 1 2; do one 64; one 32; one 48; done
