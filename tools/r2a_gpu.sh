set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2a_gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2a_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r2a_smoke.log
timeout 900 python bench.py > gpurun_out/r2a_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/r2a_bench.log
tail -3 gpurun_out/r2a_gputests.log; tail -2 gpurun_out/r2a_smoke.log; tail -c 3000 gpurun_out/r2a_bench.log
