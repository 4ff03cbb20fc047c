# grouped noops: overhead protocol + full GPU suite
timeout 600 python tools/overhead_probe.py 16 1000 > gpurun_out/r4e_overhead.log 2>&1; echo "exit $?" >> gpurun_out/r4e_overhead.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r4e_gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r4e_gputests.log
cat gpurun_out/r4e_overhead.log | cut -c1-400; tail -3 gpurun_out/r4e_gputests.log
