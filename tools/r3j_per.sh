for per in 2 3 4; do
export SFX_GEMM_TILES_PER_CTA=$per
timeout 600 python bench.py --workload cholesky --gpus 1 --steps 3 --warmup 1 --no-check 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('per $per C3', round(d['value']), round(d['roofline']['frac'],4))"
timeout 600 python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('per $per C2', 'value', round(d['value']), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']))"
done
