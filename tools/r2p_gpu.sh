timeout 900 python -m pytest tests/test_gpu_potrf_flow.py tests/test_gpu_ops.py tests/test_gpu_deterministic.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python tools/potrf_probe.py --sizes 512,1024,2048 | grep trsm
