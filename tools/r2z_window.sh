#!/bin/bash
# e2e A/B: staging window x copy stream x order
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_ops.py -q -x -k "stage_stream or copy_stream or small_arena" 2>&1 | tail -3
one() { timeout 400 python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu --no-check "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', 'value', round(d['value']), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],1))" || echo "$* failed"; }
for rep in 1 2; do
one --e2e-stage-stream 1
one --e2e-stage-stream 1 --e2e-stage-window 512
one --e2e-stage-stream 1 --e2e-stage-window 256
one --e2e-stage-stream 1 --e2e-stage-window 256 --e2e-tile-block 8
one --e2e-stage-stream 1 --e2e-stage-window 256 --e2e-skew 64
one --e2e-stage-stream 1 --e2e-stage-window 128 --e2e-tile-block 8
done
