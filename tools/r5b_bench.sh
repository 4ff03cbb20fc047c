# closing bench + reference lines; host load recorded
nproc > gpurun_out/r5b_host.log; uptime >> gpurun_out/r5b_host.log; free -g >> gpurun_out/r5b_host.log
timeout 1200 python bench.py > gpurun_out/r5b_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/r5b_bench.log
timeout 900 python bench.py --impl reference > gpurun_out/r5b_ref.log 2>&1; echo "ref exit $?" >> gpurun_out/r5b_ref.log
uptime >> gpurun_out/r5b_host.log
grep '^{' gpurun_out/r5b_bench.log | tail -1 > gpurun_out/r5b_bench_line.json
grep '^{' gpurun_out/r5b_ref.log | tail -1 > gpurun_out/r5b_ref_line.json
cat gpurun_out/r5b_host.log
