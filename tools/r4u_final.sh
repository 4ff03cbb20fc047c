# closing run at HEAD: GPU suite, smoke, default bench, reference arm, Cholesky line on 2 logical devices
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r4u_gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r4u_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4u_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r4u_smoke.log
timeout 1200 python bench.py > gpurun_out/r4u_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/r4u_bench.log
timeout 900 python bench.py --impl reference > gpurun_out/r4u_ref.log 2>&1; echo "ref exit $?" >> gpurun_out/r4u_ref.log
timeout 900 python bench.py --workload cholesky --gpus 2 --ordinals 0,0 > gpurun_out/r4u_c3x2.log 2>&1; echo "c3x2 exit $?" >> gpurun_out/r4u_c3x2.log
tail -2 gpurun_out/r4u_gputests.log; tail -2 gpurun_out/r4u_smoke.log; tail -1 gpurun_out/r4u_bench.log; tail -1 gpurun_out/r4u_ref.log; tail -1 gpurun_out/r4u_c3x2.log
grep '^{' gpurun_out/r4u_bench.log | tail -1 > gpurun_out/r4u_bench_line.json
grep '^{' gpurun_out/r4u_ref.log | tail -1 > gpurun_out/r4u_ref_line.json
grep '^{' gpurun_out/r4u_c3x2.log | tail -1 > gpurun_out/r4u_c3x2_line.json
