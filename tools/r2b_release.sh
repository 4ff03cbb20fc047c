# A/B of the DGEMM stage release (SFX_GEMM_RELEASE: 0 = data-dependent arrive, 1 = fence)
for r in 0 1; do
  echo "== release $r"
  SFX_GEMM_RELEASE=$r STEPS=3 timeout 300 python tools/c2_check.py 2>&1 | grep "max rel\|bad"
  for rep in 1 2; do
  SFX_GEMM_RELEASE=$r timeout 600 python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('value', round(d['value']), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']))"
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -2
