timeout 900 python -m pytest tests/test_gpu_potrf_flow.py tests/test_gpu_ops.py tests/test_gpu_deterministic.py tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python tools/potrf_probe.py --sizes 512,1024,2048 | grep trsm
for i in 1 2; do
timeout 900 python bench.py --workload cholesky --gpus 1 --steps 3 --warmup 2 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', round(d['value']), round(d['roofline']['frac'],4), d['check']['pass'])"
done
timeout 900 python bench.py --workload cholesky --gpus 1 --n 65536 --steps 2 --warmup 1 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5', round(d['value']), round(d['roofline']['frac'],4), d['check']['pass'])"
