#!/bin/bash
one() { timeout 400 python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('per', '${SFX_GEMM_TILES_PER_CTA}', 'value', round(d['value']), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']), 'check', d['check']['pass'], d['e2e']['check']['pass'])" || echo "$* failed"; }
for rep in 1 2; do
for per in 3 4 6 8 12; do SFX_GEMM_TILES_PER_CTA=$per; export SFX_GEMM_TILES_PER_CTA; one; done
done
