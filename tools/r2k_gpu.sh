timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2k_gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2k_gputests.log
timeout 600 python tools/overhead_probe.py 16 1000 > gpurun_out/r2k_overhead.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2 value', round(d['value']), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']))"
tail -3 gpurun_out/r2k_gputests.log; cat gpurun_out/r2k_overhead.log
