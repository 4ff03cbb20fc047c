./tools/bin/flow_prof 1024 2 | grep -E "alone|k  1:|k 14"
SFX_POTRF_F=pivot ./tools/bin/flow_prof 1024 2 | grep -E "k  1:"
timeout 900 python -m pytest tests/test_gpu_potrf_flow.py tests/test_gpu_failures.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python tools/potrf_probe.py --sizes 512,1024,2048 | grep potrf
