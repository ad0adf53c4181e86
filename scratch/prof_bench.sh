CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-c5"
$CMD > gpurun_out/plain_b.log 2>&1 && true; \
ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 1500 --csv --log-file gpurun_out/launches_r01b.csv $CMD > gpurun_out/ncu_l.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:"k_spmv|k_bond_assemble|k_element_assemble|k_pcg_update|k_pcg_pupdate" -s 3000 -c 12 -o gpurun_out/prof_bench_r01b -f $CMD > gpurun_out/ncu_b.log 2>&1; tail -2 gpurun_out/ncu_b.log
ncu -i gpurun_out/prof_bench_r01b.ncu-rep --page raw --csv > gpurun_out/prof_bench_r01b_raw.csv
python profiles/summarize.py gpurun_out/prof_bench_r01b.ncu-rep > gpurun_out/prof_bench_r01b_summary.txt
