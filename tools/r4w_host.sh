# host-side runtime cost per task in the C2 value leg (is the box host-bound?)
nproc; uptime; lscpu | grep -i "model name\|MHz" | head -3
for r in 1 2; do
timeout 600 python bench.py --no-secondary --no-cpu > gpurun_out/r4w_$r.log 2>&1
grep '^{' gpurun_out/r4w_$r.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('run', round(j['value']), 'share', round(j['roofline']['kernel_share_of_step'],3), j['runtime_host_us_per_task'], 'e2e', round(j['e2e']['value']))"
done
