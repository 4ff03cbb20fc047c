timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2l_gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2l_gputests.log
tail -3 gpurun_out/r2l_gputests.log
for w in "--n 32768" "--n 65536 --steps 2 --warmup 1"; do
timeout 900 python bench.py --workload cholesky --gpus 1 $w > gpurun_out/r2l_chol.log 2>&1
grep '^{' gpurun_out/r2l_chol.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['n'], round(d['value']), round(d['roofline']['frac'],4), d['check'])"
done
