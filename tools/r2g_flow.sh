./tools/bin/flow_prof 1024 2 | sed -n "4,6p;20,21p"
timeout 900 python -m pytest tests/test_gpu_potrf_flow.py tests/test_gpu_failures.py -x -q -p no:cacheprovider 2>&1 | tail -5
timeout 600 python tools/potrf_probe.py --sizes 1024,2048
