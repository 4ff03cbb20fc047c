# A/B: next-stage wait hoisted above the second half's DMMAs (current) vs previous HEAD
one() { timeout 600 python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', 'value', round(d['value']), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']))"; }
cp paper_2308_15964_b200/libsfx.so /tmp/libsfx_cur.so
for rep in 1 2; do
  cp /tmp/libsfx_cur.so paper_2308_15964_b200/libsfx.so; one cur
  cp variants/head/libsfx.so paper_2308_15964_b200/libsfx.so; one head
done
cp /tmp/libsfx_cur.so paper_2308_15964_b200/libsfx.so
STEPS=2 timeout 300 python tools/c2_check.py 2>&1 | grep "max rel"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -2
