for i in 1 2 3 4; do
  timeout 900 python bench.py --workload cholesky --gpus 1 --steps 3 --warmup 2 --no-check 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('run $i', round(d['value']), round(d['roofline']['frac'],4), d['clocks'])"
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
