# commutative guards passed at launch (1 device): overhead protocol + full GPU suite
timeout 600 python tools/overhead_probe.py 16 1000 > gpurun_out/r4m_overhead.log 2>&1; echo "exit $?" >> gpurun_out/r4m_overhead.log
cut -c1-200 gpurun_out/r4m_overhead.log | head -7
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r4m_gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r4m_gputests.log
tail -3 gpurun_out/r4m_gputests.log
