# rep outliers vs the scratch pool backing (6 GiB): 2 logical devices twice, 1 device
for i in 1 2; do
timeout 600 python bench.py --workload cholesky --gpus 2 --ordinals 0,0 --steps 10 --warmup 1 --no-check --no-secondary > gpurun_out/r4p_x2_$i.log 2>&1
grep '^{' gpurun_out/r4p_x2_$i.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('x2 run $i', round(j['value']), j['rep_ms'])"
done
timeout 600 python bench.py --workload cholesky --gpus 1 --steps 10 --warmup 1 --no-check > gpurun_out/r4p_x1.log 2>&1
grep '^{' gpurun_out/r4p_x1.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('x1', round(j['value']), j['rep_ms'], round(j['e2e']['value']))"
