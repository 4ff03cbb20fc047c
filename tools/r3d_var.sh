for i in 1 2 3 4 5 6 7 8; do
timeout 900 python bench.py --workload cholesky --gpus 1 --steps 4 --warmup 2 --no-check 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', round(d['value']), d['rep_ms'])"
done
