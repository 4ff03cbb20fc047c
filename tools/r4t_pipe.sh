# device-resident leg pipelined vs per step
for r in 1 2; do
timeout 600 python bench.py --no-secondary --no-cpu > gpurun_out/r4t_$r.log 2>&1; echo "exit $?" >> gpurun_out/r4t_$r.log
grep '^{' gpurun_out/r4t_$r.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('run $r value', round(j['value']), j['ms_per_step'], 'iso', round(j['isolated_step']['value']), 'frac', round(j['roofline']['frac'],4), 'share', round(j['roofline']['kernel_share_of_step'],4), 'e2e', round(j['e2e']['value']), j['check']['pass'], j['check']['expected'])"
done
