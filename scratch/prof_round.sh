# round profile set: plain run && ncu launch list; plain run && ncu --set full of the PCG/assembly kernels
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-c5"
$CMD > gpurun_out/plain_c.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 1500 --csv --log-file gpurun_out/launches_bench_r01c.csv $CMD > gpurun_out/ncu_lc.log 2>&1
$CMD > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_spmv|k_bond_assemble|k_element_assemble|k_pcg_update|k_pcg_pupdate|k_bond_energy" -s 3000 -c 14 -o gpurun_out/prof_bench_r01c -f $CMD > gpurun_out/ncu_bc.log 2>&1
ncu -i gpurun_out/prof_bench_r01c.ncu-rep --page raw --csv > gpurun_out/prof_bench_r01c_raw.csv
python profiles/summarize.py gpurun_out/prof_bench_r01c.ncu-rep > gpurun_out/prof_bench_r01c_summary.txt
