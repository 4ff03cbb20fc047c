# 2 logical devices: rep variance vs streams per device (hardware queue aliasing hypothesis)
for st in 32 12; do
timeout 600 python bench.py --workload cholesky --gpus 2 --ordinals 0,0 --streams $st --steps 6 --warmup 1 --no-check > gpurun_out/r4l_c3x2_$st.log 2>&1
grep '^{' gpurun_out/r4l_c3x2_$st.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C3 2dev streams $st', round(j['value']), j['rep_ms'], 'e2e', round(j['e2e']['value']), j['e2e']['h2d_bytes_per_step'], j['gpu_launches'])"
done
