timeout 600 python tools/potrf_probe.py --sizes 1024 | grep trsm
for tp in 2 1 2 1; do
SFX_GEMM_TRI_PER=$tp timeout 900 python bench.py --workload cholesky --gpus 1 --steps 3 --warmup 1 --no-check 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tri_per $tp C3', round(d['value']), round(d['roofline']['frac'],4), d['rep_ms'])"
done
timeout 900 python -m pytest tests/test_gpu_potrf_flow.py tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -1
