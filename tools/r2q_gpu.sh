timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/r2q_bench.log 2>&1; echo "bench exit $?"
timeout 900 python bench.py --impl reference > gpurun_out/r2q_ref.log 2>&1; echo "ref exit $?"
grep '^{' gpurun_out/r2q_bench.log | tail -1 > gpurun_out/r2q_bench_line.json
grep '^{' gpurun_out/r2q_ref.log | tail -1 > gpurun_out/r2q_ref_line.json
timeout 900 python bench.py --workload particles --gpus 2 --ordinals 0,0 --steps 2 --warmup 1 > gpurun_out/r2q_c4_l2.log 2>&1; echo "c4 l2 exit $?"
timeout 900 python bench.py --workload particles --gpus 1 --steps 2 --warmup 1 > gpurun_out/r2q_c4_1.log 2>&1; echo "c4 1 exit $?"
