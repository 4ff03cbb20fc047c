# C3 + the north-star C5 leg on 8 LOGICAL devices of one B200 (code path of the N=8 line; host-side costs only)
free -g | head -2 > gpurun_out/r4q_host.log; nproc >> gpurun_out/r4q_host.log
timeout 900 python bench.py --workload cholesky --gpus 8 --ordinals 0,0,0,0,0,0,0,0 --steps 2 --warmup 1 > gpurun_out/r4q_c5.log 2>&1; echo "exit $?" >> gpurun_out/r4q_c5.log
tail -3 gpurun_out/r4q_c5.log | cut -c1-3000
