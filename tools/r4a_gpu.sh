timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r4a_gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r4a_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4a_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r4a_smoke.log
timeout 1200 python bench.py > gpurun_out/r4a_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/r4a_bench.log
timeout 900 python bench.py --impl reference > gpurun_out/r4a_ref.log 2>&1; echo "ref exit $?" >> gpurun_out/r4a_ref.log
tail -2 gpurun_out/r4a_gputests.log; tail -2 gpurun_out/r4a_smoke.log; tail -1 gpurun_out/r4a_bench.log; tail -1 gpurun_out/r4a_ref.log
grep '^{' gpurun_out/r4a_bench.log | tail -1 > gpurun_out/r4a_bench_line.json
grep '^{' gpurun_out/r4a_ref.log | tail -1 > gpurun_out/r4a_ref_line.json
