#!/bin/bash
export SFX_GEMM_TMA_STORE=1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ops.py tests/test_gpu_potrf_flow.py -q -x 2>&1 | tail -3
one() { timeout 400 python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', 'value', round(d['value']), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']), 'check', d['check']['pass'], d['e2e']['check']['pass'])" || echo "$* failed"; }
for rep in 1 2; do
SFX_GEMM_TMA_STORE=0 one
SFX_GEMM_TMA_STORE=1 one
done
