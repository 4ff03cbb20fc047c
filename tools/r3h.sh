SFX_GEMM_TILES_PER_CTA=2 timeout 120 python tools/potrf_probe.py --sizes 1024 --reps 2 2>&1 | grep trsm
timeout 120 python tools/potrf_probe.py --sizes 512,1024 2>&1 | grep trsm
SFX_GEMM_TILES_PER_CTA=2 timeout 300 python bench.py --workload cholesky --gpus 1 --steps 2 --warmup 1 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('per2 C3', round(d['value']), d['check'])"
timeout 900 python -m pytest tests/test_gpu_potrf_flow.py tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -1
