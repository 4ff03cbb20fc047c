# ncu evidence for the producer-masked TRI TRSM: lone (trsm_once) and grouped (first dgemm launch of a
# 8192/1024 Cholesky = panel 0's 7 grouped TRSMs), plus the C3 launch list
ncu --set full --import-source on --clock-control none -k regex:dgemm_dmma -s 1 -c 1 -o gpurun_out/r4i_trsm_lone python tools/trsm_once.py 1024 > gpurun_out/r4i_ncu1.log 2>&1; echo "ncu1 $?"
ncu --set full --import-source on --clock-control none -k regex:dgemm_dmma -c 1 -o gpurun_out/r4i_trsm_grouped python tools/prof_workload.py cholesky --n 8192 --b 1024 --reps 1 > gpurun_out/r4i_ncu2.log 2>&1; echo "ncu2 $?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4i_launches_c3.csv python bench.py --workload cholesky --gpus 1 --steps 1 --warmup 0 --no-check > gpurun_out/r4i_c3.log 2>&1; echo "ncu3 $?"
