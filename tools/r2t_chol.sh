for cg in 8 16 32; do
  timeout 900 python bench.py --workload cholesky --gpus 1 --chol-group $cg --steps 3 --warmup 2 --no-check 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chol-group $cg', round(d['value']), round(d['roofline']['frac'],4))"
done
