for tp in 1 2 1 2 1 2; do
  SFX_GEMM_TRI_PER=$tp timeout 900 python bench.py --workload cholesky --gpus 1 --steps 3 --warmup 2 --no-check 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tri_per $tp', round(d['value']), round(d['roofline']['frac'],4))"
done
