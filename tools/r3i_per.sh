for per in 2 0 2 0; do
if [ $per = 0 ]; then unset SFX_GEMM_TILES_PER_CTA; else export SFX_GEMM_TILES_PER_CTA=$per; fi
timeout 600 python bench.py --workload cholesky --gpus 1 --steps 3 --warmup 1 --no-check 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('per $per C3', round(d['value']), round(d['roofline']['frac'],4))"
done
for per in 2 0; do
if [ $per = 0 ]; then unset SFX_GEMM_TILES_PER_CTA; else export SFX_GEMM_TILES_PER_CTA=$per; fi
timeout 900 python bench.py --workload cholesky --gpus 1 --n 65536 --steps 2 --warmup 1 --no-check 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('per $per C5', round(d['value']), round(d['roofline']['frac'],4))"
done
