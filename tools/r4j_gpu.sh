# Cholesky line: e2e leg + gpu_launches; full GPU suite + smoke at this HEAD
timeout 900 python bench.py --workload cholesky --gpus 2 --ordinals 0,0 --steps 2 --warmup 1 > gpurun_out/r4j_c3x2.log 2>&1; echo "exit $?" >> gpurun_out/r4j_c3x2.log
grep '^{' gpurun_out/r4j_c3x2.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C3x2', round(j['value']), j['e2e'], j['gpu_launches'], j['p2p'], j['scaling_reference'])"
tail -2 gpurun_out/r4j_c3x2.log | cut -c1-300
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r4j_gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r4j_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4j_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r4j_smoke.log
tail -2 gpurun_out/r4j_gputests.log; tail -2 gpurun_out/r4j_smoke.log
