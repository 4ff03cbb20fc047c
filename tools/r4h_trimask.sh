# TRI masking moved to the producer warpgroup: parity, lone-op latency, C3/C5
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "trsm or cholesky or potrf or fullinv or parity" > gpurun_out/r4h_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r4h_tests.log
tail -3 gpurun_out/r4h_tests.log
timeout 300 python tools/potrf_probe.py --sizes 1024,2048 > gpurun_out/r4h_probe.log 2>&1; tail -12 gpurun_out/r4h_probe.log
timeout 600 python tools/chol_sweep.py --help > /dev/null 2>&1
timeout 600 python bench.py --workload cholesky --gpus 1 --steps 3 --warmup 2 > gpurun_out/r4h_c3.log 2>&1; grep '^{' gpurun_out/r4h_c3.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C3', j['value'], j['check'], j['rep_ms'])"
timeout 600 python bench.py --workload cholesky --gpus 1 --n 65536 --steps 2 --warmup 1 > gpurun_out/r4h_c5.log 2>&1; grep '^{' gpurun_out/r4h_c5.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C5', j['value'], j['check'], j['rep_ms'])"
