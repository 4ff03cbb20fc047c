for r in 0 1 2 3; do
  echo "== release $r"
  SFX_GEMM_RELEASE=$r python tools/c2_check.py 2>&1 | grep "max rel"
  SFX_GEMM_RELEASE=$r STEPS=3 python tools/c2_check.py 2>&1 | grep "max rel"
  SFX_GEMM_RELEASE=$r python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'])"
done
