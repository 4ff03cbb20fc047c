# A/B: NN column-permuted B operands (current) vs round-1 LDS.64 path (variants/nn0), and
# CUDA_DEVICE_MAX_CONNECTIONS 32 vs 8; plus one ncu --set full capture of each NN variant
one() { timeout 600 python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', 'value', round(d['value']), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']), 'conc', round(d['roofline']['launch_concurrency'],1))"; }
cp paper_2308_15964_b200/libsfx.so /tmp/libsfx_cur.so
for rep in 1 2; do
  cp /tmp/libsfx_cur.so paper_2308_15964_b200/libsfx.so
  one "cur conn32"; CUDA_DEVICE_MAX_CONNECTIONS=8 one "cur conn8"
  cp variants/nn0/libsfx.so paper_2308_15964_b200/libsfx.so
  one "nn0 conn32"; CUDA_DEVICE_MAX_CONNECTIONS=8 one "nn0 conn8"
done
cp variants/nn0/libsfx.so paper_2308_15964_b200/libsfx.so
STEPS=2 timeout 300 python tools/c2_check.py 2>&1 | grep "max rel"
ncu --set full --clock-control none --import-source on -k regex:dgemm_dmma -s 40 -c 1 -o gpurun_out/r2c_dgemm_nn0 python tools/prof_workload.py gemm --n 8192 --b 512 --reps 2 > gpurun_out/r2c_ncu_nn0.log 2>&1
cp /tmp/libsfx_cur.so paper_2308_15964_b200/libsfx.so
ncu --set full --clock-control none --import-source on -k regex:dgemm_dmma -s 40 -c 1 -o gpurun_out/r2c_dgemm_cur python tools/prof_workload.py gemm --n 8192 --b 512 --reps 2 > gpurun_out/r2c_ncu_cur.log 2>&1
tail -2 gpurun_out/r2c_ncu_*.log
