# C3 rep-time variance at HEAD (1 GPU, 2 logical devices)
for i in 1 2; do
timeout 600 python bench.py --workload cholesky --gpus 1 --steps 10 --warmup 2 --no-check > gpurun_out/r4k_c3_$i.log 2>&1
grep '^{' gpurun_out/r4k_c3_$i.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C3 1dev', round(j['value']), j['rep_ms'])"
done
timeout 600 python bench.py --workload cholesky --gpus 2 --ordinals 0,0 --steps 6 --warmup 1 --no-check > gpurun_out/r4k_c3x2.log 2>&1
grep '^{' gpurun_out/r4k_c3x2.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C3 2dev', round(j['value']), j['rep_ms'])"
