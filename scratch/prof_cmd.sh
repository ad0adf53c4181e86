CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:k_spmv -s 100 -c 2 -o gpurun_out/prof_spmv $CMD > gpurun_out/ncu2.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:k_bond_assemble -s 3 -c 1 -o gpurun_out/prof_asm $CMD > gpurun_out/ncu3.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:"k_pcg_update|k_element_assemble|k_bond_energy" -s 30 -c 3 -o gpurun_out/prof_misc $CMD > gpurun_out/ncu4.log 2>&1; \
ls -la gpurun_out; tail -3 gpurun_out/ncu*.log
