# Cholesky e2e: priorities of the host-staged factorization
for pr in auto true critical; do
SFX_CHOL_E2E_PRIO=$pr timeout 600 python bench.py --workload cholesky --gpus 1 --steps 2 --warmup 1 --no-check > gpurun_out/r4s_$pr.log 2>&1
grep '^{' gpurun_out/r4s_$pr.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('prio $pr', round(j['value']), 'e2e', round(j['e2e']['value']), j['e2e']['ms_per_step'])"
done
