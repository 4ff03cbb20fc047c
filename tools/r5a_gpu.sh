# paged tid table: burst probe + full GPU suite
timeout 600 python tools/burst_probe.py 20 4 > gpurun_out/r5a_burst.log 2>&1; tail -6 gpurun_out/r5a_burst.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r5a_gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r5a_gputests.log
tail -2 gpurun_out/r5a_gputests.log
