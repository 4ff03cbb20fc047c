# trace SVG from a real CUDA run; C3/C5 over 2/4/8 LOGICAL devices on one B200 (host-side runtime costs)
timeout 300 python tools/trace_svg.py --n 16384 --b 1024 --out gpurun_out/r2_trace_chol16k.svg > gpurun_out/r2j_trace.log 2>&1
timeout 300 python tools/trace_svg.py --n 16384 --b 1024 --ordinals 0,0 --out gpurun_out/r2_trace_chol16k_2dev.svg > gpurun_out/r2j_trace2.log 2>&1
for N in 2 4 8; do
  ORD=$(python -c "print(','.join(['0']*$N))")
  timeout 600 python bench.py --workload cholesky --gpus $N --ordinals $ORD --steps 3 --warmup 2 > gpurun_out/r2j_c3_l$N.log 2>&1
done
ORD=0,0,0,0,0,0,0,0
timeout 900 python bench.py --workload cholesky --gpus 8 --ordinals $ORD --n 65536 --steps 2 --warmup 1 > gpurun_out/r2j_c5_l8.log 2>&1
timeout 900 python bench.py --workload cholesky --gpus 1 --n 65536 --steps 2 --warmup 1 > gpurun_out/r2j_c5_1.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2j_ref.log 2>&1
tail -2 gpurun_out/r2j_trace.log gpurun_out/r2j_trace2.log
for f in gpurun_out/r2j_c*.log; do echo $f; grep '^{' $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], round(d['value']), d['config']['grid'], d.get('check'), d['runtime_host_us_per_task'], d['p2p']['gbs'], d.get('scaling_reference'))"; done
tail -c 400 gpurun_out/r2j_ref.log
