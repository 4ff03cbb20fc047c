# A/B: stages / C buffer / stagger depth
one() { timeout 600 python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', 'value', round(d['value']), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']))"; }
cp paper_2308_15964_b200/libsfx.so /tmp/libsfx_cur.so
for rep in 1 2; do
  cp /tmp/libsfx_cur.so paper_2308_15964_b200/libsfx.so
  SFX_GEMM_STAGGER=1 one "s3c1 lag1"; SFX_GEMM_STAGGER=2 one "s3c1 lag2"
  cp variants/s6c0/libsfx.so paper_2308_15964_b200/libsfx.so
  SFX_GEMM_STAGGER=1 one "s6c0 lag1"; SFX_GEMM_STAGGER=2 one "s6c0 lag2"; SFX_GEMM_STAGGER=3 one "s6c0 lag3"
  cp variants/s4c0/libsfx.so paper_2308_15964_b200/libsfx.so
  SFX_GEMM_STAGGER=1 one "s4c0 lag1"; SFX_GEMM_STAGGER=2 one "s4c0 lag2"
done
cp variants/s6c0/libsfx.so paper_2308_15964_b200/libsfx.so
STAGES=1 SFX_GEMM_STAGGER=3 timeout 300 python tools/c2_check.py 2>&1 | grep "max rel"
cp /tmp/libsfx_cur.so paper_2308_15964_b200/libsfx.so
SFX_GEMM_STAGGER=2 timeout 300 python tools/c2_check.py 2>&1 | grep "max rel"
