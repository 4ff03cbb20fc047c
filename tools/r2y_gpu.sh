timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2y_gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2y_gputests.log
tail -2 gpurun_out/r2y_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/r2y_bench.log 2>&1; echo "bench exit $?"
grep '^{' gpurun_out/r2y_bench.log | tail -1 > gpurun_out/r2y_bench_line.json
python -c "
import json
d=json.load(open('gpurun_out/r2y_bench_line.json'))
print('value', round(d['value']), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']), 'launches', d['gpu_launches'], d['check']['pass'], d['e2e']['check']['pass'])
s=d['secondary']; print('C1', round(s['dgemm_C1']['gflops']), 'C3', round(s['cholesky_C3']['gflops']), s['cholesky_C3']['check']['pass'], 'C4', s['particles_C4']['interactions_per_s'], s['particles_C4']['check']['pass'])
print([(r['D_s'], r['mode'], r['deps'], round(r['o_avg_us'],1), round(r['insertion_per_task_us'],2)) for r in s['runtime_overhead']['runs']])
print('cpu', d['cpu_baseline']['value'])
"
