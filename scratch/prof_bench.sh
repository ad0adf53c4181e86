CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/plain_b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 1500 --csv --log-file gpurun_out/launches_r01.csv $CMD > gpurun_out/ncu_l.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:"k_spmv|k_bond_assemble|k_element_assemble|k_pcg_update" -s 400 -c 8 -o gpurun_out/prof_bench_r01 $CMD > gpurun_out/ncu_b.log 2>&1; tail -2 gpurun_out/ncu_b.log
