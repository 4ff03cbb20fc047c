# A/B: staggered DMMA warpgroups (SFX_GEMM_STAGGER=1, default) vs together (0)
one() { timeout 600 python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', 'value', round(d['value']), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']))"; }
for rep in 1 2 3; do
  SFX_GEMM_STAGGER=1 one stagger; SFX_GEMM_STAGGER=0 one together
done
STEPS=2 timeout 300 python tools/c2_check.py 2>&1 | grep "max rel"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ops.py -x -q -p no:cacheprovider 2>&1 | tail -2
