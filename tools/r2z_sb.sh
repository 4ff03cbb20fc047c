#!/bin/bash
one() { timeout 400 python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu --no-check "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', 'value', round(d['value']), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],1))" || echo "$* failed"; }
for rep in 1 2; do
one --e2e-stage-stream 1 --e2e-skew 64 --e2e-skew-block 16
one --e2e-stage-stream 1 --e2e-skew 96 --e2e-skew-block 16
one --e2e-stage-stream 1 --e2e-skew 128 --e2e-skew-block 16
one --e2e-stage-stream 0 --e2e-skew 64 --e2e-skew-block 16
one --e2e-stage-stream 1 --e2e-skew 64 --e2e-skew-block 8
one --e2e-stage-stream 1 --e2e-skew 64 --e2e-skew-block 16 --e2e-flush-priority 100000
done
