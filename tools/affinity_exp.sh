for a in 1 0; do
  echo "== stream_affinity=$a"
  SFX_OPT_STREAM_AFFINITY=$a python tools/overhead_probe.py
  SFX_OPT_STREAM_AFFINITY=$a python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2 value', d['value'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'])"
  SFX_OPT_STREAM_AFFINITY=$a ORD=0 REPS=4 python tools/chol_multi_check.py | tail -3
done
