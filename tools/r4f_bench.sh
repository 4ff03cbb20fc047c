timeout 1200 python bench.py > gpurun_out/r4f_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/r4f_bench.log
timeout 900 python bench.py --impl reference > gpurun_out/r4f_ref.log 2>&1; echo "ref exit $?" >> gpurun_out/r4f_ref.log
grep '^{' gpurun_out/r4f_bench.log | tail -1 > gpurun_out/r4f_bench_line.json
grep '^{' gpurun_out/r4f_ref.log | tail -1 > gpurun_out/r4f_ref_line.json
