# dataflow POTRF: parity tests, then op latency (flow vs the round-1 cooperative kernel)
timeout 900 python -m pytest tests/test_gpu_potrf_flow.py tests/test_gpu_failures.py -x -q -p no:cacheprovider 2>&1 | tail -15
echo "== flow"; timeout 600 python tools/potrf_probe.py --sizes 512,1024,2048
echo "== coop"; SFX_POTRF=coop timeout 600 python tools/potrf_probe.py --sizes 512,1024,2048
