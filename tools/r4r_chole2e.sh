# Cholesky e2e: staging FIFO on the copy stream or not
for st in 0 1; do
SFX_CHOL_E2E_STAGE_STREAM=$st timeout 600 python bench.py --workload cholesky --gpus 1 --steps 2 --warmup 1 --no-check > gpurun_out/r4r_$st.log 2>&1
grep '^{' gpurun_out/r4r_$st.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('stage_stream $st', round(j['value']), 'e2e', round(j['e2e']['value']), j['e2e']['ms_per_step'])"
done
