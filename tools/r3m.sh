for N in 2 8; do
  ORD=$(python -c "print(','.join(['0']*$N))")
  timeout 600 python bench.py --workload cholesky --gpus $N --ordinals $ORD --steps 3 --warmup 2 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($N, round(d['value']), d['check']['pass'], {k: round(v,2) for k,v in d['runtime_host_us_per_task'].items()}, round(d['p2p']['gbs'],1), round(d['scaling_reference']['value']))"
done
timeout 900 python bench.py --workload cholesky --gpus 8 --ordinals 0,0,0,0,0,0,0,0 --n 65536 --steps 2 --warmup 1 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5 l8', round(d['value']), d['check']['pass'], {k: round(v,2) for k,v in d['runtime_host_us_per_task'].items()})"
