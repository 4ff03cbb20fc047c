# rep outliers: Python GC during insertion? (2 logical devices, 10 timed reps each)
for ng in 0 1 0 1; do
SFX_BENCH_NOGC=$ng timeout 600 python bench.py --workload cholesky --gpus 2 --ordinals 0,0 --steps 10 --warmup 1 --no-check --no-secondary > gpurun_out/r4o_$ng.log 2>&1
grep '^{' gpurun_out/r4o_$ng.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('nogc=$ng', round(j['value']), j['rep_ms'])"
done
