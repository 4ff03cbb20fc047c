# grouped spins: overhead protocol
timeout 600 python tools/overhead_probe.py 16 1000 > gpurun_out/r4g_overhead.log 2>&1; echo "exit $?" >> gpurun_out/r4g_overhead.log
cat gpurun_out/r4g_overhead.log | cut -c1-300
