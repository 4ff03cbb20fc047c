set -x
for c in 8 32 8 32; do
  CUDA_DEVICE_MAX_CONNECTIONS=$c python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('conn $c C2 value', d['value'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'])"
done
ncu --set full --clock-control none --import-source on -k regex:dgemm_dmma -s 40 -c 1 -o gpurun_out/r2_dgemm_nn_c2 python tools/prof_workload.py gemm --n 8192 --b 512 --reps 2 > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -c 80 -o gpurun_out/r2_chol2k python tools/prof_workload.py cholesky --n 2048 --b 1024 --reps 1 > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/ncu1.log gpurun_out/ncu2.log
