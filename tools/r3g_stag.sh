for st in 1 0 1 0; do
SFX_GEMM_STAGGER=$st timeout 900 python bench.py --workload cholesky --gpus 1 --steps 3 --warmup 1 --no-check 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stagger $st C3', round(d['value']), round(d['roofline']['frac'],4))"
done
for st in 1 0; do
SFX_GEMM_TILES_PER_CTA=2 SFX_GEMM_STAGGER=$st timeout 900 python bench.py --workload cholesky --gpus 1 --steps 3 --warmup 1 --no-check 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('per2 stagger $st C3', round(d['value']), round(d['roofline']['frac'],4))"
done
