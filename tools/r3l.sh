timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 600 python tools/overhead_probe.py 16 1000 2>&1 | tail -8
timeout 600 python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2', 'value', round(d['value']), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']), d['check']['pass'])"
timeout 600 python bench.py --workload cholesky --gpus 1 --steps 3 --warmup 1 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', round(d['value']), round(d['roofline']['frac'],4), d['check']['pass'])"
