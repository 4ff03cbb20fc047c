# launch list of C3 (serialised kernel times) and of the default bench
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2m_launches_c3.csv python bench.py --workload cholesky --gpus 1 --steps 1 --warmup 0 --no-check > gpurun_out/r2m_c3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2m_launches_bench.csv python bench.py --steps 1 --warmup 0 --no-secondary --no-cpu --no-check > gpurun_out/r2m_bench.log 2>&1
ls -la gpurun_out/r2m_*
