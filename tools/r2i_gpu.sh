# full GPU suite, default bench, overhead probe, ncu of the panel-chain kernels
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2i_gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2i_gputests.log
timeout 900 python bench.py > gpurun_out/r2i_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/r2i_bench.log
timeout 600 python tools/overhead_probe.py 16 1000 > gpurun_out/r2i_overhead.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:potrf_flow -s 1 -c 1 -o gpurun_out/r2i_potrf_flow python tools/trsm_once.py 1024 > gpurun_out/r2i_ncu1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:dgemm_dmma -s 1 -c 1 -o gpurun_out/r2i_trsm_tri python tools/trsm_once.py 1024 > gpurun_out/r2i_ncu2.log 2>&1
tail -3 gpurun_out/r2i_gputests.log; tail -c 600 gpurun_out/r2i_bench.log; cat gpurun_out/r2i_overhead.log
