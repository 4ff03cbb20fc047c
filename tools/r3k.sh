timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
for i in 1 2; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2', 'value', round(d['value']), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']), d['check']['pass'], d['roofline']['kernel_paths']['multi_tile'])"
timeout 600 python bench.py --workload cholesky --gpus 1 --steps 3 --warmup 1 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', round(d['value']), round(d['roofline']['frac'],4), d['check']['pass'])"
done
timeout 900 python bench.py --workload cholesky --gpus 1 --n 65536 --steps 2 --warmup 1 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5', round(d['value']), round(d['roofline']['frac'],4), d['check']['pass'])"
